import sys, os, numpy as np, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import torch, ht_inputs, htcheck as C, oracle
import paper_1710_08538_b200 as ht
from test_gpu import to_dev, from_dev
os.makedirs("gpurun_out", exist_ok=True)
cases = [("singular", n, nb, 7) for n, nb in [(20, 4), (40, 8), (64, 8), (66, 8), (100, 16), (130, 16)]]
out = {}
for kind, n, nb, seed in cases:
    A, B = ht_inputs.pencil(kind, n, seed)
    tr = np.zeros(n, dtype=np.int32)
    dA, dB = to_dev(A), to_dev(B); dQ = torch.empty_like(dA); dZ = torch.empty_like(dA)
    rep = ht.reduce_device(dA, dB, dQ, dZ, nb=nb, ir_trace=tr)
    torch.cuda.synchronize()
    H = from_dev(dA); Hg = oracle.ht_G(A, B)[0]
    d = C.abs_diff(H, Hg, C.fro(A))
    out[f"{n}_{nb}"] = dict(trace=tr.tolist(), diff=d)
    print(kind, n, nb, "diff %.2e" % d, tr[:40].tolist())
json.dump(out, open("gpurun_out/traces.json", "w"))
