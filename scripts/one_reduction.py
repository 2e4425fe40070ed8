"""One HT reduction of a BASELINE config (for ncu launch lists / captures).  Usage:
    python scripts/one_reduction.py CFG [N] [REPS]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ht_inputs  # noqa: E402
import paper_1710_08538_b200 as ht  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
A, B, nb = ht_inputs.config_pencil(cfg, n=n)
to_dev = lambda M: torch.from_numpy(np.ascontiguousarray(M.T)).cuda()
A0, B0 = to_dev(A), to_dev(B)
dA, dB = torch.empty_like(A0), torch.empty_like(B0)
dQ, dZ = torch.empty_like(A0), torch.empty_like(A0)
for _ in range(reps):
    dA.copy_(A0)
    dB.copy_(B0)
    rep = ht.reduce_device(dA, dB, dQ, dZ, nb=nb)
    torch.cuda.synchronize()
print({k: rep[k] for k in ("seconds", "launches", "panels", "ir_steps_total")})
