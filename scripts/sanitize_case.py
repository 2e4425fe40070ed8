import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import torch, ht_inputs
import paper_1710_08538_b200 as ht
from test_gpu import to_dev
cfg, n, nb = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
A, B, _ = ht_inputs.config_pencil(cfg, n=n)
dA, dB = to_dev(A), to_dev(B); dQ = torch.empty_like(dA); dZ = torch.empty_like(dA)
rep = ht.reduce_device(dA, dB, dQ, dZ, nb=nb)
torch.cuda.synchronize()
print("ok", rep["seconds"])
