"""IR trace of one full reduction (development helper): columns with IR and failures."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np, torch, ht_inputs
import paper_1710_08538_b200 as ht
from test_gpu import to_dev
cfg = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
A, B, nb = ht_inputs.config_pencil(cfg, n=n or None)
dA, dB = to_dev(A), to_dev(B); dQ = torch.empty_like(dA); dZ = torch.empty_like(dA)
A0, B0 = dA.clone(), dB.clone()
reps = int(os.environ.get("REPS", "1"))
for it in range(reps):
    dA.copy_(A0); dB.copy_(B0)
    tr = np.zeros(A.shape[0], dtype=np.int32)
    rep = ht.reduce_device(dA, dB, dQ, dZ, nb=nb, ir_trace=tr)
    torch.cuda.synchronize()
    print("rep", it, {k: rep[k] for k in ("seconds", "panels", "ir_steps_total", "ir_failed_columns")}, "sum|H| %.17g" % dA.abs().sum().item())
cols = np.nonzero(tr)[0]
print("ir columns:", len(cols), "first:", [(int(c), int(tr[c])) for c in cols[:12]], "failed:", [int(c) for c in cols if tr[c] >= 1000][:10])
print({k: rep[k] for k in ("seconds", "panels", "ir_steps_total", "ir_extra_columns", "ir_failed_columns")})
h = np.asfortranarray(dA.cpu().numpy().T); print("sum|H| %.17g" % np.abs(h).sum())
