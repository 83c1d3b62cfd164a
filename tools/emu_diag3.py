import ctypes, sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
NN = 601
inst = G.config("C1", n=NN, m=433)
a = np.full(NN, 1 / NN); b = np.full(433, 1 / 433)
mk = lambda: sk.PointProblem(inst.x, inst.y, a, b, inst.epsilon)
L = sk.lib()
L.sknr_debug_sums.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]
def run(p):
    sk.solve(p, tol=1e-9, max_iter=1)
    out = np.zeros(16)
    L.sknr_debug_sums(p.handle, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return out
res = sk.run_emulated_shards(mk, 8, run)
np.set_printoptions(precision=17)
for r, o in enumerate(res):
    print(r, o[:6].tolist())
