"""ncu target (dev tool): a few restricted-derivative passes with r fused (sknr_bench_pass
which=4) at C4 on the tensor-core path (or the FP64 DMMA path with argv[1] == 'fp64')."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

sk.set_tensor_block_pass(not (len(sys.argv) > 1 and sys.argv[1] == "fp64"))
name = sys.argv[2] if len(sys.argv) > 2 else "C4"
inst = G.config(name)
p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon, inst.cost_scale)
ms, kms = sk.bench_pass(p, 4, inst.ell, 3)
print(f"{name} block RS pass: {ms:.3f} ms ({kms:.3f} kernel)", flush=True)
