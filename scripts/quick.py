"""Quick GPU sanity run: small cases with diagnostics (development helper)."""
import sys, os, time, traceback
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np
import torch
import ht_inputs, htcheck as C, oracle
import paper_1710_08538_b200 as ht
from test_gpu import gpu_reduce

cases = [("shifted", 3, 1), ("shifted", 5, 2), ("shifted", 8, 2), ("qrnormal", 12, 3), ("qrnormal", 30, 4),
         ("qrnormal", 64, 8), ("shifted", 130, 32), ("qruniform", 300, 32), ("singular", 120, 16)]
if len(sys.argv) > 1:
    cases = [(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))]
for kind, n, nb in cases:
    A, B = ht_inputs.pencil(kind, n, 7)
    try:
        t0 = time.time()
        H, T, Q, Z, rep = gpu_reduce(A, B, nb=nb)
        dt = time.time() - t0
        e = C.backward_errors(A, B, H, T, Q, Z)
        Hr, Tr, _, _ = (oracle.ht_G if kind == "singular" else oracle.ht_T)(A, B)
        print(f"{kind} n={n} nb={nb}: struct={C.structure_ok(H,T)} resA={e[0]:.2e} resB={e[1]:.2e} "
              f"oQ={e[2]:.2e} oZ={e[3]:.2e} |H|={C.abs_diff(H,Hr,C.fro(A)):.2e} |T|={C.abs_diff(T,Tr,C.fro(B)):.2e} "
              f"tol={C.tol_ns(n):.1e} t={dt:.3f}s ir={rep['ir_steps_total']} fail={rep['ir_failed_columns']} "
              f"resc={rep['solve_rescales']}", flush=True)
    except Exception:
        traceback.print_exc()
