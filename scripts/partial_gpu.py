import sys, os, numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import torch, ht_inputs
import paper_1710_08538_b200 as ht
from test_gpu import to_dev, from_dev
os.makedirs("gpurun_out", exist_ok=True)
for kind, force in [("qruniform", (1,)), ("qruniform", (2,)), ("qruniform", (5,))]:
    A, B = ht_inputs.pencil(kind, 130, 7)
    for mp in [1, 2]:
        dA, dB = to_dev(A), to_dev(B); dQ = torch.empty_like(dA); dZ = torch.empty_like(dA)
        ht.reduce_device(dA, dB, dQ, dZ, nb=16, max_panels=mp, force_ir_fail=force)
        torch.cuda.synchronize()
        np.savez(f"gpurun_out/partialF_{force[0]}_{mp}.npz", A=from_dev(dA), B=from_dev(dB), Q=from_dev(dQ), Z=from_dev(dZ))
print("ok")
