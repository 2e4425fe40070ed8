import sys, os, numpy as np, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import torch, ht_inputs, htcheck as C, oracle
import paper_1710_08538_b200 as ht
from test_gpu import to_dev, from_dev
cases = [("qrnormal", 130, 32, 1162)]
if len(sys.argv) > 4: cases = [(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))]
for kind, n, nb, seed in cases:
    A, B = ht_inputs.pencil(kind, n, seed)
    tr = np.zeros(n, dtype=np.int32)
    dA, dB = to_dev(A), to_dev(B); dQ = torch.empty_like(dA); dZ = torch.empty_like(dA)
    rep = ht.reduce_device(dA, dB, dQ, dZ, nb=nb, ir_trace=tr)
    torch.cuda.synchronize()
    print(kind, n, nb, tr[:48].tolist())
