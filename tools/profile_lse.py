"""ncu target: the C4 column-LSE sum tile kernel (and the ell-wide block pass).
Usage: python tools/profile_lse.py [which] [bits]   which=2 LSE sum kernel, 3 block pass, 4 fused S / r block pass (Newton step);
bits=32 profiles the opt-in fp32 sum kernel (set_precision(32)); a third argument "cull"
turns culling on (use which=0: the full column LSE, whose sum pass is then pts_cull_kernel)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

which = int(sys.argv[1]) if len(sys.argv) > 1 else 2
inst = G.config("C4")
p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon)
if len(sys.argv) > 2 and int(sys.argv[2]) == 32:
    p.set_precision(32)
if len(sys.argv) > 3 and sys.argv[3] == "cull":
    p.set_culling(60.0)
ms, kms = sk.bench_pass(p, which, inst.ell, passes=2)
print(f"which={which} pass {ms:.3f} ms kernel {kms:.3f} ms")
