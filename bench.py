#!/usr/bin/env python
"""bench.py -- FP64 HT-reduction (HouseHT, arXiv 1710.08538) on B200.

One "step" = one complete Hessenberg-triangular reduction (all of SURVEY §8(a):
panels P1-P5 + absorption R1-L3, with Q and Z accumulated) of the BASELINE.json
headline workload (config 3: n = 8192, nb = 128, A ~ U(-1,1), B = R of QR(U(-1,1)),
seed 2), with A, B restored from a pristine device copy at the start of each step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C] [--n N]

N > 1 is launched with torch.distributed.run (one process per GPU, NCCL): all ranks
reduce ONE pencil together (paper_1710_08538_b200/mg.py): A, B replicated, Q and Z split
into row slabs and all-gathered at the end (strong scaling).
Prints ONE JSON line on rank 0.  `value` is GFLOP/s on the instrumented EXECUTED flop
count F_exec (per-launch formulas, the paper's interposition convention P:2161-2162;
SURVEY §8(d)); F_model (App. A) and GFLOP/s on it are in `detail`.  `ms_per_step` is the
wall time of one reduction (max over ranks).  `roofline_e2e` is T_roof / t with
T_roof = F_L3,exec / P64 + B_L2,exec / BW.  `configs` carries the other BASELINE.json
configs (1, 2, 4, 5) measured in the same run (fewer steps; --also none skips them).
`--gpus N` without WORLD_SIZE re-launches itself under torch.distributed.run.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import ht_inputs  # noqa: E402

METRIC = "FP64 HT-reduction wall time & GFLOP/s at n=8192, 1/2/4/8 B200"
WORKLOAD = {
    1: "cfg1: n=256 FP64 pencil, A~N(0,1), B=R of QR(N(0,1)), seed 0, nb=32, Q,Z accumulated",
    2: "cfg2: n=2048 FP64 pencil, A~N(0,1), B=triu(N(0,1))+sqrt(n)I, seed 1, nb=64, Q,Z accumulated",
    3: "cfg3: n=8192 FP64 pencil, A~U(-1,1), B=R of QR(U(-1,1)), seed 2, nb=128, Q,Z accumulated",
    4: "cfg4: n=8192 FP64 pencil, singular graded B (10% zero pivots), seed 3, nb=128, Q,Z accumulated",
    5: "cfg5: n=16384 FP64 pencil, A~N(0,1), B=triu(N(0,1))+sqrt(n)I, seed 4, nb=256, Q,Z accumulated",
}


from paper_1710_08538_b200.model import model_flops, roofline_seconds  # noqa: E402  (measurement logic)

ENV_KNOBS = ("HT_NO_TRSV4", "HT_NO_GREEN", "HT_GREEN_SMS", "HT_TRSV4_CLUSTER", "HT_L2PERSIST", "HT_SWEEP_RES_MB", "HT_NO_WAVE", "HT_WAVE_GROUP", "HT_SIDE_GRID_QZ", "HT_SERIAL", "HT_BATCH", "HT_SIDE_GRID", "HT_SB_GRID", "HT_PANEL_NOCLUSTER", "HT_PHASES",
             "HT_PROFILE", "HT_DEBUG_IR", "HT_TRACE_COL", "HT_FPROF", "HT_SYNC_CHECK")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 8 for i in range(4)
                          if r[4 + i].strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def dgemm_probe(torch, n=8192, reps=5):
    """cuBLAS DGEMM (torch.matmul float64) as the FP64 tensor-pipe measuring stick."""
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c = a @ b
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    del a, b, c
    torch.cuda.empty_cache()
    return 2.0 * n ** 3 / best / 1e12


def cpu_oracle_sample(A, B, budget_s: float):
    """Time Oracle-T (oracle/, as it stands) on the first j columns of the same pencil,
    j chosen to fill ~budget_s, and extrapolate to the full reduction with its own
    per-column flop model 39 m^2 + 40 n m (host-memory-bound, ~constant rate)."""
    import oracle
    n = A.shape[0]
    t0 = time.time()
    oracle.ht_T(A, B, jmax=2)
    t2 = time.time() - t0
    per_col = max(t2 / 2.0, 1e-4)
    j = int(max(2, min(n - 2, budget_s / per_col)))
    t0 = time.time()
    oracle.ht_T(A, B, jmax=j)
    ts = time.time() - t0
    f_s = oracle.flops_T(n, j)
    f_full = oracle.flops_T(n)
    t_full = ts * f_full / f_s
    return dict(t_sample=ts, cols=j, t_full_est=t_full, cores=oracle.num_threads(), gflops_oracle=f_s / ts / 1e9)


def run_reference(args, cfg, n, nb, rank, world):
    """--impl reference: the oracle (CPU) arm, rank 0 only."""
    if rank != 0:
        return 0
    A, B, _ = ht_inputs.config_pencil(cfg, n=n)
    Fm = model_flops(n, nb)
    budget = max(2.0, 30.0 / max(args.steps + args.warmup, 1))
    for _ in range(args.warmup):
        cpu_oracle_sample(A, B, budget / 4)
    tf = []
    last = None
    for _ in range(args.steps):
        last = cpu_oracle_sample(A, B, budget)
        tf.append(last["t_full_est"])
    t = float(np.mean(tf))
    val = Fm / t / 1e9
    line = {"metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": WORKLOAD.get(cfg, f"cfg{cfg}") + (f" (n={n})" if n != ht_inputs.CONFIGS[cfg]["n"] else ""),
                       "n": n, "nb": nb},
            "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": last["cores"], "kind": "oracle",
                             "sample": f"Oracle-T (oracle/ht_oracle.c) on columns 0..{last['cols'] - 1} of the "
                                       f"n={n} pencil, extrapolated by its flop model to a full reduction"},
            "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def relaunch_distributed(args) -> int:
    """`--gpus N` (N > 1) without a torch.distributed environment: run this script under
    torch.distributed.run, one process per GPU (the driver's own launch line)."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def env_knobs():
    """HT_* development switches present in the environment (recorded in the line)."""
    return {k: os.environ[k] for k in ENV_KNOBS if k in os.environ}


def measure_config(torch, ht, mg, cfg, n, nb, steps, warmup, stream, world, rank, dist, want_e2e=False, A_h=None, B_h=None,
                   comm=None, flags=0):
    """Time `steps` full reductions of config `cfg` after `warmup` untimed ones (device
    events on the caller's stream, max over ranks).  Returns a dict of measurements."""
    if A_h is None:
        A_h, B_h, _ = ht_inputs.config_pencil(cfg, n=n)
    to_dev = lambda M: torch.from_numpy(np.ascontiguousarray(M.T)).cuda()
    A0, B0 = to_dev(A_h), to_dev(B_h)
    A, B = torch.empty_like(A0), torch.empty_like(B0)
    Q, Z = torch.empty_like(A0), torch.empty_like(A0)

    def step():
        A.copy_(A0)  # pristine inputs each step (inputs larger than L2 at n >= 2048)
        B.copy_(B0)
        return mg.reduce_mg(A, B, Q, Z, nb=nb, comm=comm, rank=rank, world=world, stream=stream.cuda_stream,
                            flags=flags)

    f_single = None
    for i in range(warmup):
        if world > 1 and i == 0:
            # executed flops of the whole problem (F_exec of P = 1: replicated work is not credited twice)
            A.copy_(A0)
            B.copy_(B0)
            f_single = ht.reduce_device(A, B, Q, Z, nb=nb, stream=stream.cuda_stream, flags=flags)["flops"]
        else:
            step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = []
    e0.record(stream)
    for _ in range(steps):
        reps.append(step())
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    elapsed = e0.elapsed_time(e1) * 1e-3
    if dist:
        t = torch.tensor([elapsed], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    out = {"elapsed": elapsed, "t_step": elapsed / steps, "reps": reps, "f_single": f_single}
    if want_e2e:
        # end to end through the public API: host pencil -> device -> reduction -> H, T, Q, Z on the host.
        # The pencil and the result buffers live in pinned host memory (allocated once, outside
        # the timed region); each timed call copies A, B in and H, T, Q, Z out (ht_reduce_host).
        ts = []
        if world == 1:
            Ap, Bp = ht.pinned_empty(n), ht.pinned_empty(n)
            Ap[:], Bp[:] = A_h, B_h
            outs = tuple(ht.pinned_empty(n) for _ in range(4))
            ht.ht_reduce(Ap, Bp, nb=nb, out=outs)  # warm-up (device staging, pinned pages)
        for _ in range(max(1, min(steps, 2))):
            if dist:
                dist.barrier()
            t0 = time.time()
            if world == 1:
                ht.ht_reduce(Ap, Bp, nb=nb, out=outs)
            else:
                hA = torch.from_numpy(np.ascontiguousarray(A_h.T)).pin_memory()
                hB = torch.from_numpy(np.ascontiguousarray(B_h.T)).pin_memory()
                A.copy_(hA, non_blocking=True)
                B.copy_(hB, non_blocking=True)
                mg.reduce_mg(A, B, Q, Z, nb=nb, comm=comm, rank=rank, world=world, stream=stream.cuda_stream)
                [M.cpu() for M in (A, B, Q, Z)]
                torch.cuda.synchronize()
            te_ = time.time() - t0
            if dist:
                tt = torch.tensor([te_], dtype=torch.float64, device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                te_ = float(tt.item())
            ts.append(te_)
        out["e2e_s"] = float(np.mean(ts))
    del A0, B0, A, B, Q, Z
    torch.cuda.empty_cache()
    return out


def summarize(reps, steps):
    keys = ("t_panel", "t_gemm", "t_factor", "t_other", "panel_bytes", "flops", "flops_level3", "launches",
            "t_chain", "flops_chain", "chain_launches", "t_absorb_right", "t_absorb_left", "t_factor_exposed", "t_chain_busy")
    return {k: float(np.sum([r[k] for r in reps])) / steps for k in keys}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--nb", type=int, default=0)
    ap.add_argument("--also", default="1,2,4,5", help="other configs measured in the same run ('none' to skip)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = args.config
    n = args.n or ht_inputs.CONFIGS[cfg]["n"]
    nb = args.nb or ht_inputs.CONFIGS[cfg]["nb"]

    if args.impl == "reference":
        return run_reference(args, cfg, n, nb, rank, world)

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1710_08538_b200 as ht
    from paper_1710_08538_b200 import mg

    stream = torch.cuda.current_stream()
    comm = mg.init_comm()[0] if world > 1 else None
    A_h, B_h, _ = ht_inputs.config_pencil(cfg, n=n)
    clocks = ClockSampler(local)
    clocks.start()
    m = measure_config(torch, ht, mg, cfg, n, nb, args.steps, args.warmup, stream, world, rank, dist,
                       want_e2e=not args.no_e2e, A_h=A_h, B_h=B_h, comm=comm)
    clk = clocks.stop()
    elapsed, t_step, reps = m["elapsed"], m["t_step"], m["reps"]
    agg = summarize(reps, args.steps)
    rep0 = reps[-1]
    Fm = model_flops(n, nb)
    Fx = m["f_single"] if m["f_single"] else agg["flops"]
    value = Fx / t_step / 1e9  # executed flops of one pencil per second, whatever the number of GPUs

    # roofline of the dominant kernel class
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    fp64_peak = dgemm_probe(torch)
    # roofline of the dominant kernel by device time in the ncu launch list (profiles/): the
    # chained window applies on the FP64 tensor pipe.  Their launch durations are CUDA events on
    # their own (concurrent) streams, so `achieved` is a per-launch rate while sharing the GPU.
    ach = agg["flops_chain"] / max(agg["t_chain"], 1e-12) / 1e12
    roof = {"bound": "tensor", "kernel": "chain_apply_kernel (FP64 DMMA window applies, K8/K9)", "achieved": ach,
            "peak": fp64_peak, "unit": "TFLOP/s", "frac": ach / fp64_peak, "traffic": None,
            "peak_source": "cuBLAS DGEMM 8192^3 measured live (FP64 tensor pipe; no FP64 entry in MEASURED_PEAKS.json)",
            "launches_per_step": agg["chain_launches"],
            "flops_per_launch": agg["flops_chain"] / max(agg["chain_launches"], 1)}
    # the launches of this kernel overlap one another (A's and Q/Z's streams share an SM
    # partition, B's run next to them), so the sum of their durations counts the same wall time
    # several times: `concurrent` divides the same flops by the time during which at least one
    # launch was running (union of the event intervals, ht_report.t_chain_busy)
    if agg["t_chain_busy"] > 0:
        cach = agg["flops_chain"] / agg["t_chain_busy"] / 1e12
        roof["concurrent"] = {"achieved": cach, "frac": cach / fp64_peak, "unit": "TFLOP/s",
                              "busy_s": agg["t_chain_busy"], "sum_of_launch_durations_s": agg["t_chain"],
                              "note": "aggregate rate of the overlapping launches while the critical stream's "
                                      "factorization and band kernels hold the other SMs"}
    # the same kernel alone (full grid, no concurrent streams), on the shape of the first R2
    # update of B at this (n, nb): n rows, a chain of (n - 1 - 2nb)/nb windows of width 2nb.
    try:
        nwin = max(1, (n - 1 - 2 * nb) // nb)
        sec, fl = ht.ht_bench_chain_apply(n, 2 * nb, nwin, False, 5)
        st_ach = fl / sec / 1e12
        roof["standalone"] = {"achieved": st_ach, "frac": st_ach / fp64_peak, "unit": "TFLOP/s",
                              "shape": f"{n} rows x chain of {nwin} windows of {2 * nb}, full grid",
                              "seconds": sec, "flops": fl}
    except Exception as exc:  # measurement hook only; never affects the timed result
        roof["standalone"] = {"error": str(exc)}
    # DRAM traffic of one live launch of the same kernel at this config, from the committed
    # `ncu --set full` capture (profiles/r02/ncu_chain.json, scripts/gpu_ncu_chain.sh)
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "ncu_chain.json")) as f:
            nj = json.load(f)
        live = nj.get("chain_cfg3_live") if cfg == 3 else None
        if live:
            roof["traffic"] = live["dram_read_bytes"] + live["dram_write_bytes"]
            roof["traffic_launch"] = {"flops": live["fp64_tensor_flops"], "duration_s_under_ncu": live["duration_s"],
                                      "grid": live["grid"], "dmma_active_pct": live["dmma_active_pct"],
                                      "source": "profiles/r02/ncu_chain.txt (launch 301 of the cfg3 reduction)"}
        st = nj.get("chain_cfg3_standalone")
        if st and "standalone" in roof and "error" not in roof["standalone"]:
            roof["standalone"]["traffic"] = st["dram_read_bytes"] + st["dram_write_bytes"]
            roof["standalone"]["algorithmic_bytes"] = 2.0 * n * ((nwin - 1) * nb + 2 * nb) * 8
    except (OSError, ValueError, KeyError):
        pass
    panel_ach = agg["panel_bytes"] / max(agg["t_panel"], 1e-12) / 1e9
    roof_panel = {"bound": "hbm", "kernel": "panel_kernel (persistent panel)", "achieved": panel_ach, "peak": hbm,
                  "unit": "GB/s", "frac": panel_ach / hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    if cfg == 3 and n == 8192:
        # one launch under `ncu --set full` (profiles/r02s4/ncu_panel_s4.txt, scripts/gpu_s4_ncu_panel.sh:
        # the 21st panel of this reduction, s0 = 2560, 128 columns, no IR step); before the sweep's
        # evict-first reads the same launch moved 70.6 GB in 27.6 ms (profiles/r02s2/ncu_panel_s2.txt)
        M21 = 8192 - 2560 - 1
        roof_panel["traffic"] = 67.108145e9 + 0.092566e9
        roof_panel["traffic_launch"] = {"algorithmic_bytes": 8.0 * sum(
            M21 * (M21 + 1) / 2.0 + float(M21) * c + i * c + c * (c + 1) / 2.0
            for i, c in ((i, 8192 - 2560 - i - 1) for i in range(128))),
            "duration_s_under_ncu": 24.25e-3, "source": "profiles/r02s4/ncu_panel_s4.txt"}
    # whole-path roofline: level-3 flops at the FP64 tensor peak + panel bytes at HBM
    t_roof = roofline_seconds(agg["flops_level3"], agg["panel_bytes"], fp64_peak, hbm)
    roof_e2e = {"t_roof_s": t_roof, "t_s": t_step, "frac": t_roof / t_step,
                "flops_level3_exec": agg["flops_level3"], "panel_bytes_exec": agg["panel_bytes"],
                "p64_tflops": fp64_peak, "hbm_gbs": hbm}
    # WY-apply phase (SURVEY §8(d) "Phase definitions"): all chain applies + DMMA GEMMs
    wy_t = agg["t_chain"] + agg["t_gemm"]
    wy = {"tflops": agg["flops_level3"] / max(wy_t, 1e-12) / 1e12, "frac": agg["flops_level3"] / max(wy_t, 1e-12) / 1e12 / fp64_peak,
          "note": "sum of launch durations on concurrent streams (a per-launch rate while sharing the GPU)"}

    e2e = None
    if "e2e_s" in m:
        te = m["e2e_s"]
        e2e = {"value": Fx / te / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": 2 * n * n * 8,
               "d2h_bytes_per_step": 4 * n * n * 8, "s_per_step": te,
               "path": "ht_reduce_host (C-ABI) from pinned host buffers: H2D of A, B + reduction + D2H of H, T, Q, Z"
               if world == 1 else "H2D from pinned host memory + ht_reduce_mg + D2H of A, B, Q, Z"}

    # the other BASELINE.json configs, same binary, fewer steps (parity-tested sizes)
    others = {}
    if args.also != "none" and world >= 1:
        for c in [int(x) for x in args.also.split(",") if x.strip()]:
            if c == cfg or c not in ht_inputs.CONFIGS:
                continue
            nc, nbc = ht_inputs.CONFIGS[c]["n"], ht_inputs.CONFIGS[c]["nb"]
            st_, wu_ = (10, 3) if nc <= 2048 else (2, 1 if world == 1 else 2)
            mc = measure_config(torch, ht, mg, c, nc, nbc, st_, wu_, stream, world, rank, dist, comm=comm)
            ac = summarize(mc["reps"], st_)
            if mc["f_single"]:
                ac["flops"] = mc["f_single"]
            rc0 = mc["reps"][-1]
            others[f"cfg{c}"] = {"workload": WORKLOAD[c], "n": nc, "nb": nbc, "steps": st_, "warmup": wu_,
                                 "ms_per_step": mc["t_step"] * 1e3, "gflops_exec": ac["flops"] / mc["t_step"] / 1e9,
                                 "gflops_model": model_flops(nc, nbc) / mc["t_step"] / 1e9,
                                 "roofline_e2e_frac": roofline_seconds(ac["flops_level3"], ac["panel_bytes"], fp64_peak, hbm) / mc["t_step"],
                                 "t_panel_s": ac["t_panel"], "t_absorb_right_s": ac["t_absorb_right"],
                                 "t_absorb_left_s": ac["t_absorb_left"], "t_factor_exposed_s": ac["t_factor_exposed"],
                                 "ir_extra_columns": rc0["ir_extra_columns"], "ir_steps": rc0["ir_steps_total"],
                                 "ir_failed_columns": rc0["ir_failed_columns"],
                                 "premature_absorptions": rc0["premature_absorptions"],
                                 "desingularizations": rc0["desingularizations"]}

    # the paper's Test Suite 4 (saddle-point pencils, Table 4) at n = 4000, with and
    # without the sec. 3.5.1 preprocessing, and the QZ step-1 front end (general B) at this n
    extra = {}
    if args.also != "none":
        As, Bs = ht_inputs.pencil("saddle", 4000, 40)
        for tag, fl in (("suite4_saddle_n4000", 0), ("suite4_saddle_n4000_preprocessed", ht.HT_FLAG_DEFLATE_ZERO_COLUMNS)):
            me = measure_config(torch, ht, mg, 0, 4000, 128, 2, 1, stream, world, rank, dist, A_h=As, B_h=Bs,
                                comm=comm, flags=fl)
            r0 = me["reps"][-1]
            extra[tag] = {"n": 4000, "nb": 128, "ms_per_step": me["t_step"] * 1e3,
                          "pct_columns_extra_ir": 100.0 * r0["ir_extra_columns"] / 4000,
                          "pct_columns_failed_ir": 100.0 * r0["ir_failed_columns"] / 4000,
                          "avg_ir_steps_per_column": r0["ir_steps_total"] / 4000,
                          "premature_absorptions": r0["premature_absorptions"],
                          "deflated_columns": r0["deflated_columns"], "t_front_s": r0["t_front"]}
        Ag, Bg = ht_inputs.pencil("general", n, 41)
        me = measure_config(torch, ht, mg, 0, n, nb, 1, 1, stream, world, rank, dist, A_h=Ag, B_h=Bg, comm=comm,
                            flags=ht.HT_FLAG_GENERAL_B)
        extra[f"general_b_n{n}"] = {"n": n, "nb": nb, "ms_per_step": me["t_step"] * 1e3,
                                    "t_front_s": me["reps"][-1]["t_front"]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        s = cpu_oracle_sample(A_h, B_h, budget_s=15.0)
        cpu = {"value": Fx / s["t_full_est"] / 1e9, "unit": "GFLOP/s", "cores": s["cores"], "kind": "oracle",
               "sample": f"Oracle-T (oracle/ht_oracle.c, as it stands) on columns 0..{s['cols'] - 1} of the same "
                         f"n={n} pencil ({s['t_sample']:.1f} s), extrapolated by its flop model to "
                         f"{s['t_full_est']:.0f} s per full reduction",
               "full_run": full_oracle_run(cfg, n)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": WORKLOAD.get(cfg, f"cfg{cfg}") + (f" (n={n})" if n != ht_inputs.CONFIGS[cfg]["n"] else ""),
                           "n": n, "nb": nb, "seed": ht_inputs.CONFIGS[cfg]["seed"],
                           "l2": "inputs larger than L2 (A,B,Q,Z = 4 x %.0f MB)" % (n * n * 8 / 1e6),
                           "parallelism": (f"mg{world}: A row/column slabs + Q,Z row slabs, B/panel/factors replicated"
                                           if world > 1 else "single"),
                           "value_flops": "executed (instrumented per launch)", "env_knobs": env_knobs()},
                "roofline": roof, "roofline_panel": roof_panel, "roofline_e2e": roof_e2e, "wy_apply_phase": wy,
                "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(agg["launches"] * args.steps), "clocks": clk, "configs": others,
                "front_ends": extra,
                "detail": {"gflops_model": Fm / t_step / 1e9, "model_flops": Fm,
                           "executed_flops_per_step": Fx, "exec_over_model": Fx / Fm,
                           "t_panel_s": agg["t_panel"], "t_gemm_s": agg["t_gemm"],
                           "t_factor_s": agg["t_factor"], "t_factor_exposed_s": agg["t_factor_exposed"],
                           "t_absorb_right_s": agg["t_absorb_right"], "t_absorb_left_s": agg["t_absorb_left"],
                           "t_other_s": agg["t_other"], "t_chain_s": agg["t_chain"],
                           "gemm_tflops": (agg["flops_level3"] - agg["flops_chain"]) / max(agg["t_gemm"], 1e-9) / 1e12,
                           "panel_gbs": panel_ach, "fp64_dgemm_probe_tflops": fp64_peak,
                           "ir_steps": rep0["ir_steps_total"], "ir_extra_columns": rep0["ir_extra_columns"],
                           "ir_failed_columns": rep0["ir_failed_columns"],
                           "desingularizations": rep0["desingularizations"], "panels": rep0["panels"]}}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        ht.ht_nccl_comm_destroy(comm)
        dist.destroy_process_group()
    return 0


def full_oracle_run(cfg, n):
    """A full (not sampled) oracle run on this pencil, if one was recorded (tests/golden/, written by
    scripts/make_fullsize_golden.py on the build container's host: say so, it is another machine)."""
    for w in ("T", "G"):
        p = os.path.join(ROOT, "tests", "golden", f"fullsize_cfg{cfg}_{w}.npz")
        if os.path.exists(p):
            g = np.load(p)
            if int(g["n"]) == n:
                return {"oracle": f"Oracle-{w}", "seconds": float(g["seconds"]), "threads": int(g["threads"]),
                        "host": "build container (8 vCPU), not the GPU box"}
    return None


if __name__ == "__main__":
    sys.exit(main())
