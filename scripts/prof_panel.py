import sys, os, numpy as np, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import torch, ht_inputs
import paper_1710_08538_b200 as ht
from test_gpu import to_dev
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
A, B, nb = ht_inputs.config_pencil(cfg, n=n or None)
dA, dB = to_dev(A), to_dev(B); dQ = torch.empty_like(dA); dZ = torch.empty_like(dA)
A0, B0 = dA.clone(), dB.clone()
for i in range(2):
    dA.copy_(A0); dB.copy_(B0)
    if i == 1: os.environ["HT_PROFILE"] = "1"
    rep = ht.reduce_device(dA, dB, dQ, dZ, nb=nb)
    torch.cuda.synchronize()
print({k: round(v, 4) if isinstance(v, float) else v for k, v in rep.items()})
