"""Development check: HT_SERIAL=1 (everything on one stream) vs the multi-stream path."""
import sys, os, subprocess, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
if len(sys.argv) > 1 and sys.argv[1] == "run":
    import numpy as np, torch, ht_inputs
    import paper_1710_08538_b200 as ht
    from test_gpu import to_dev, from_dev
    A, B, nb = ht_inputs.config_pencil(3, n=1100)
    dA, dB = to_dev(A), to_dev(B); dQ = torch.empty_like(dA); dZ = torch.empty_like(dA)
    ht.reduce_device(dA, dB, dQ, dZ, nb=128, force_ir_fail=(300, 301))
    torch.cuda.synchronize()
    np.save(sys.argv[2], np.stack([from_dev(dA), from_dev(dB), from_dev(dQ), from_dev(dZ)]))
    sys.exit(0)
import numpy as np
env = dict(os.environ)
subprocess.run([sys.executable, __file__, "run", "/tmp/multi.npy"], check=True, env=env)
env["HT_SERIAL"] = "1"
subprocess.run([sys.executable, __file__, "run", "/tmp/serial.npy"], check=True, env=env)
a, b = np.load("/tmp/multi.npy"), np.load("/tmp/serial.npy")
print("max |multi - serial| over H, T, Q, Z:", float(np.max(np.abs(a - b))), "bitwise equal:", bool(np.array_equal(a, b)))
