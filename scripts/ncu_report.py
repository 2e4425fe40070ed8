"""Summarize one-kernel `ncu --set full` captures into profiles/ (development tool, runs here:
ncu -i reads the .ncu-rep without a GPU).

    python scripts/ncu_report.py OUT_PREFIX REP [REP ...]

writes OUT_PREFIX.txt (per capture: launch shape, time, tensor/DRAM/L2 metrics, the top warp
stall reasons and the executed-instruction mix from the SASS source page) and OUT_PREFIX.json
(the numbers bench.py quotes: DRAM bytes and FP64 tensor ops per captured launch).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

NCU = os.environ.get("NCU", "/usr/local/cuda/bin/ncu")
KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_src_fp64.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3,
         "msecond": 1e-3, "nsecond": 1e-9, "Kbyte/block": 1e3, "byte/block": 1}


def ncu_csv(rep, *page):
    out = subprocess.run([NCU, "-i", rep, *page, "--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def to_num(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    return x * SCALE.get(unit, 1)


def summarize(rep):
    raw = ncu_csv(rep, "--page", "raw")
    hdr, units, vals = raw[0], raw[1], raw[2]
    col = {h: i for i, h in enumerate(hdr)}
    m = {k: (vals[col[k]], units[col[k]]) for k in KEYS if k in col}
    kname = vals[col["Kernel Name"]] if "Kernel Name" in col else "?"
    stalls = []
    for h, i in col.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            stalls.append((to_num(vals[i], "") or 0.0, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    stalls.sort(reverse=True)
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    i0 = [k for k, r in enumerate(src) if r and r[0] == "Address"][0]
    sh = src[i0]
    ci, si, so = sh.index("Instructions Executed"), sh.index("Warp Stall Sampling (All Samples)"), sh.index("Source")
    ex, smp = collections.Counter(), collections.Counter()
    for r in src[i0 + 1:]:
        if len(r) <= ci or not r[so]:
            continue
        toks = r[so].split()
        op = (toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
        ex[op] += int(float(r[ci] or 0))
        smp[op] += int(float(r[si] or 0))
    return kname, m, stalls, ex, smp


def main():
    prefix, reps = sys.argv[1], sys.argv[2:]
    lines, js = [], {}
    for rep in reps:
        kname, m, stalls, ex, smp = summarize(rep)
        tag = os.path.splitext(os.path.basename(rep))[0]
        lines.append(f"== {tag}: {kname}")
        lines.append(f"   source: {rep} (ncu --set full --clock-control none --import-source on, one launch)")
        for k, (v, u) in m.items():
            lines.append(f"   {k:80s} {v} {u}")
        lines.append("   top stall reasons (warps per issue-active cycle):")
        for v, name in stalls[:8]:
            lines.append(f"     {name:28s} {v:7.3f}")
        tot, tots = sum(ex.values()) or 1, sum(smp.values()) or 1
        lines.append("   executed SASS by opcode (share of instructions | share of stall samples):")
        for op, n in ex.most_common(14):
            lines.append(f"     {op:10s} {100 * n / tot:5.1f}% | {100 * smp[op] / tots:5.1f}%")
        g = lambda k: to_num(*m[k]) if k in m else None
        js[tag] = {"kernel": kname, "report": rep, "duration_s": g("gpu__time_duration.sum"),
                   "grid": g("launch__grid_size"), "dram_read_bytes": g("dram__bytes_read.sum"),
                   "dram_write_bytes": g("dram__bytes_write.sum"),
                   "fp64_tensor_flops": g("sm__ops_path_tensor_src_fp64.sum"),
                   "dmma_active_pct": g("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active")}
    with open(prefix + ".txt", "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(prefix + ".json", "w") as f:
        json.dump(js, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
