"""fp32 variant at C4: launch variants of the fp32 sum kernel, the MUFU ceiling, the SK
iteration rate, and SK to 1e-9 against the fp64 solve (iterations, potentials)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2506_14780_b200 as sk
from paper_2506_14780_b200 import generators as G

inst = G.config("C4")
cells = inst.n * inst.m
out = {}
gex2, _ = sk.bench_mufu_peak()
out["mufu_peak_gex2_per_s"] = gex2
p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon)
p.set_precision(32)
for v in [int(a) for a in sys.argv[1:]] or [300, 301, 302, 303, 304, 305]:
    ms = sk.tune_variant(p, v, passes=5)
    out[f"variant_{v}"] = {"ms": ms, "gcells_per_s": cells / ms / 1e6, "frac_mufu": cells / ms / 1e6 / gex2}
    print(v, out[f"variant_{v}"], flush=True)
ms_pass, ms_k = sk.bench_pass(p, 2, 0, passes=10)
out["column_lse_f32"] = {"pass_ms": ms_pass, "kernel_ms": ms_k, "kernel_gcells_per_s": cells / ms_k / 1e6}
ms_it, kpi = sk.bench_iterations(p, 0, None, iters=20, warmup=3, flush_l2=True)
out["sk_iteration_f32"] = {"ms": ms_it, "gcells_per_s": 2 * cells / ms_it / 1e6}
print(json.dumps(out), flush=True)
t0 = time.perf_counter()
r32 = sk.solve(p, tol=1e-9, trace=False)
t32 = time.perf_counter() - t0
p64 = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon)
t0 = time.perf_counter()
r64 = sk.solve(p64, tol=1e-9, trace=False)
t64 = time.perf_counter() - t0
rel = lambda a, b: float(np.max(np.abs(a - b)) / np.max(np.abs(b)))
out["c4_sk_ttt"] = {"f32": {"iterations": r32.iterations, "converged": r32.converged, "s": t32},
                    "f64": {"iterations": r64.iterations, "converged": r64.converged, "s": t64},
                    "rel_f": rel(r32.f, r64.f), "rel_g": rel(r32.g, r64.g)}
print(json.dumps(out["c4_sk_ttt"]), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "fp32_probe.json"), "w"), indent=1)
