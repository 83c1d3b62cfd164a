"""Tensor-core Newton block pass vs the FP64 DMMA pass (dev tool): device ms per
restricted-derivative pass (sknr_bench_pass which=3) and per SK-NR(ell) iteration on a
BASELINE config, and the agreement of the restricted derivatives at a random iterate.
Usage: python tools/i8_probe.py [C4|C3|C2] [passes]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G
from support import smooth_basis

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 10
inst = G.config(name)
p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon, inst.cost_scale)
V = np.asfortranarray(smooth_basis(inst.x, inst.alpha, inst.ell))
basis = sk.SpectralBasis(V, V, np.zeros(inst.ell), inst.epsilon)
out = {"config": name, "n": inst.n, "m": inst.m, "ell": inst.ell}
res = {}
for on in (True, False):
    sk.set_tensor_block_pass(on)
    tag = "tensor_i8" if on else "fp64_dmma"
    ms, kms = sk.bench_pass(p, 3, inst.ell, passes)
    it_ms, kpi = sk.bench_iterations(p, inst.ell, basis, iters=5, warmup=2)
    r = sk.solve(p, tol=1e-9, max_iter=8, trace=False)  # an iterate with a real anchor
    t0 = time.perf_counter()
    gr, H = sk.restricted_derivatives(p, r.f, basis)
    res[tag] = (gr, H)
    out[tag] = {"pass_ms": ms, "pass_kernel_ms": kms, "sknr_iteration_ms": it_ms, "kernels_per_iteration": kpi,
                "gcells_per_s": inst.n * inst.m / kms / 1e6}
    print(tag, json.dumps(out[tag]), flush=True)
gt, Ht = res["tensor_i8"]
gf, Hf = res["fp64_dmma"]
out["rel_grad"] = float(np.max(np.abs(gt - gf)) / np.max(np.abs(gf)))
out["rel_H"] = float(np.max(np.abs(Ht - Hf)) / np.max(np.abs(Hf)))
print(json.dumps({k: v for k, v in out.items() if not isinstance(v, dict)}), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"i8_probe_{name.lower()}.json"), "w"), indent=1)
