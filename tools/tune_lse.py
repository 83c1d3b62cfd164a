"""Time launch variants of the d=2 LSE sum kernel at C4 (see tile_kernels.cu tune_variant)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

inst = G.config("C4")
p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon)
cells = inst.n * inst.m
print("fp64 peak (TFLOP/s, ms):", sk.bench_fp64_peak())
variants = [int(a) for a in sys.argv[1:]] or list(range(20))
for v in variants:
    ms = sk.tune_variant(p, v, passes=5)
    print(f"variant {v:2d}: {ms:7.3f} ms  {cells/ms/1e6:8.1f} GCells/s", flush=True)
