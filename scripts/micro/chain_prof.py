"""Per-phase cycle split of chain_apply_kernel (development tool).  Needs the instrumented
library built by:  nvcc ... -DCHAIN_PROF -shared -o scripts/micro/libht_prof.so paper_1710_08538_b200/csrc/*.cu"""
import ctypes, os, sys
HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, sys.argv[1] if len(sys.argv) > 1 else "libht_prof.so"))
i64 = ctypes.c_int64
lib.ht_bench_chain_apply.argtypes = [i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
buf = (ctypes.c_ulonglong * (256 * 8))()
for rows, p, nwin, left in ((8192, 256, 61, 0), (8192, 256, 61, 1)):
    sec, fl = ctypes.c_double(), ctypes.c_double()
    lib.ht_bench_chain_apply(rows, p, nwin, left, 1, ctypes.byref(sec), ctypes.byref(fl))
    lib.ht_chain_prof_read(buf, 1)
    lib.ht_bench_chain_apply(rows, p, nwin, left, 1, ctypes.byref(sec), ctypes.byref(fl))
    lib.ht_chain_prof_read(buf, 0)
    lib.ht_chain_prof_read(buf, 1)
    ctas = [[buf[b * 8 + i] for i in range(8)] for b in range(256) if buf[b * 8 + 2]]
    nc = len(ctas)
    avg = [sum(c[i] for c in ctas) / nc / 2 for i in range(8)]  # 2 launches (warm-up + 1 rep)
    print(f"rows={rows} p={p} left={left}: {sec.value*1e3:.3f} ms {fl.value/sec.value/1e12:.2f} TF; ctas={nc}")
    print("  per CTA cycles: first-load %.0f  loop %.0f (barrier %.0f)  epilogue %.0f  transition %.0f" %
          (avg[0], avg[1], avg[4], avg[2] - avg[1], avg[3]))
    print("  per window: loop %.0f  barrier %.0f epi %.0f trans %.0f" % (avg[1] / nwin, avg[4] / nwin, (avg[2] - avg[1]) / nwin, avg[3] / nwin))
