"""C4 SK-NR(32) main solve (stable accept test) from the shared warm start and basis
(c4_full_inputs/inputs.npz): unsharded vs R emulated row shards on one GPU, each shard
running the tensor-core Newton pass on its rows. Writes gpurun_out/c4_shard_parity_r02.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
c = G.config("C4")
d = np.load(os.path.join(ROOT, "c4_full_inputs", "inputs.npz"))
mk = lambda: sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.epsilon, c.cost_scale)
V = np.asfortranarray(d["V"])
basis = sk.SpectralBasis(V, V, d["rhos"], c.basis_eps)
init = (d["warm_f"], d["warm_g"])
rel = lambda a, b: float(np.max(np.abs(a - b)) / np.max(np.abs(b)))
run = lambda p: sk.solve(p, tol=1e-9, max_iter=5000, ell=c.ell, basis=basis, init=init, trace=True, accept="stable")
t0 = time.perf_counter()
ref = run(mk())
t_ref = time.perf_counter() - t0
t0 = time.perf_counter()
res = sk.run_emulated_shards(mk, R, run)
t_sh = time.perf_counter() - t0
acc = lambda r: [bool(t.newton_accepted) for t in r.trace]
out = {"config": "C4 n=m=65536 d=2 eps=5e-4 ell=32 tol=1e-9, SK-NR main solve, stable accept, tensor-core Newton pass",
       "R": R, "tensor_block_pass": bool(sk.lib().sknr_get_tensor_block_pass()),
       "unsharded": {"iterations": ref.iterations, "accepts": int(sum(acc(ref))), "s": t_ref},
       "sharded": {"iterations": [r.iterations for r in res], "accepts": int(sum(acc(res[0]))), "s": t_sh,
                   "same_accepts": acc(res[0]) == acc(ref), "rel_f": rel(res[0].f, ref.f),
                   "rel_g": rel(res[0].g, ref.g),
                   "ranks_identical": all(np.array_equal(r.g, res[0].g) for r in res)}}
print(json.dumps(out), flush=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "c4_shard_parity_r02.json"), "w"), indent=1)
