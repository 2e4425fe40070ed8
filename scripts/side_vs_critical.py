"""Diagnosis: is the cfg3 absorption bound by the critical stream or by the side streams?
Times one reduction with Q and Z, with Q only, and with neither (less side work, same critical
chain).  Usage: python scripts/side_vs_critical.py [CFG]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ht_inputs  # noqa: E402
import paper_1710_08538_b200 as ht  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
A, B, nb = ht_inputs.config_pencil(cfg)
to_dev = lambda M: torch.from_numpy(np.ascontiguousarray(M.T)).cuda()
A0, B0 = to_dev(A), to_dev(B)
dA, dB = torch.empty_like(A0), torch.empty_like(B0)
dQ, dZ = torch.empty_like(A0), torch.empty_like(A0)
for label, q, z in (("QZ", dQ, dZ), ("Q only", dQ, None), ("none", None, None), ("QZ again", dQ, dZ)):
    ts = []
    for _ in range(2):
        dA.copy_(A0)
        dB.copy_(B0)
        rep = ht.reduce_device(dA, dB, q, z, nb=nb)
        torch.cuda.synchronize()
        ts.append(rep["seconds"])
    print(f"{label:9s}: {min(ts):.4f} s  panel {rep['t_panel']:.3f}  factor_exposed {rep['t_factor_exposed']:.3f}  "
          f"absorb R {rep['t_absorb_right']:.3f} L {rep['t_absorb_left']:.3f}", flush=True)
