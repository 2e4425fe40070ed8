"""Standalone chain-apply rate via the C-ABI measurement hook (ht_bench_chain_apply)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1710_08538_b200 as ht
for rows, p, nwin, left in ((8192, 256, 61, 0), (8192, 256, 61, 1), (16384, 512, 62, 0), (2048, 128, 30, 0)):
    sec, fl = ht.ht_bench_chain_apply(rows, p, nwin, left, 5)
    print(f"rows={rows} p={p} nwin={nwin} left={left}: {sec*1e3:.3f} ms  {fl/sec/1e12:.2f} TFLOP/s")
