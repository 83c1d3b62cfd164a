"""Time stored-cost LSE variants on C5 (32768 x 16384, cost materialised on device)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
inst = G.config("C5")
p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon)  # d=64 -> stored cost
cells = inst.n * inst.m
for v in range(100, 108):
    ms = sk.tune_variant(p, v, passes=5)
    print(f"variant {v}: {ms:7.3f} ms {cells/ms/1e6:8.1f} GCells/s {8*cells/ms/1e6:8.1f} GB/s", flush=True)
