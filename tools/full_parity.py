"""Full-size main-solve parity at BASELINE C3 / C4 against the oracle's OWN trajectory.

Both sides start from the same inputs -- the eps' warm potentials and the top_modes
basis in {c3,c4}_full_inputs/inputs.npz (made once on the GPU by
tools/c4_full_parity.py gpu) -- and each runs the SK-NR(ell) main solve to tolerance
on its own iterates (solver.cpp:104-151), in one accept mode:

  literal  the reference's Q(f') > Q(f) (solver.cpp:46-47)
  stable   the same predicate as dQ > 0, evaluated directly (sknr_config.accept_test)

  SKNR_PARITY_CFG=C4 python tools/full_parity.py gpu              # B200: both modes
  SKNR_PARITY_CFG=C4 python tools/full_parity.py oracle stable    # host cores, resumable
  SKNR_PARITY_CFG=C4 python tools/full_parity.py merge            # profiles/c4_full_parity_r02.json

The oracle runs in chunks of CHUNK iterations, each resumed from the previous chunk's
f (a solve iteration recomputes g from f first, so the chunks are one trajectory);
its state is checkpointed after every chunk.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

from paper_2506_14780_b200 import generators as G

CFG = os.environ.get("SKNR_PARITY_CFG", "C4").upper()
TAG = CFG.lower()
INPUTS = os.path.join(ROOT, f"{TAG}_full_inputs", "inputs.npz")
OUT = os.path.join(ROOT, "gpurun_out", f"{TAG}_r02")
# oracle checkpoints: beside the inputs here; under gpurun_out/ on the GPU box's host
STATE = os.environ.get("SKNR_PARITY_STATE", os.path.join(ROOT, f"{TAG}_full_inputs"))
CHUNK = int(os.environ.get("SKNR_PARITY_CHUNK", "5"))
MAX_ITER = 5000


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def run_gpu():
    import paper_2506_14780_b200 as sk

    c = G.config(CFG)
    d = np.load(INPUTS)
    os.makedirs(OUT, exist_ok=True)
    p = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.epsilon, c.cost_scale)
    basis = sk.SpectralBasis(np.asfortranarray(d["V"]), np.asfortranarray(d["V"]), d["rhos"], c.basis_eps)
    init = (d["warm_f"], d["warm_g"])
    res = {}
    for mode in ("literal", "stable"):
        t0 = time.perf_counter()
        r = sk.solve(p, tol=1e-9, max_iter=MAX_ITER, ell=c.ell, basis=basis, init=init, trace=True, accept=mode)
        secs = time.perf_counter() - t0
        np.savez(os.path.join(OUT, f"gpu_{mode}.npz"), f=r.f, g=r.g, iterations=r.iterations,
                 converged=r.converged, marginal_error=np.array([t.marginal_error for t in r.trace]),
                 semi_dual_value=np.array([t.semi_dual_value for t in r.trace]),
                 accepted=np.array([bool(t.newton_accepted) for t in r.trace]))
        res[mode] = {"iterations": r.iterations, "converged": r.converged, "s": secs,
                     "accepts": int(sum(t.newton_accepted for t in r.trace))}
        print(mode, json.dumps(res[mode]), flush=True)
    json.dump(res, open(os.path.join(OUT, "gpu_info.json"), "w"), indent=1)


def run_oracle(mode):
    import oracle_ref as O

    c = G.config(CFG)
    d = np.load(INPUTS)
    op = O.Instance(c.alpha, c.beta, c.epsilon, x=c.x, y=c.y, cost_div=1.0 / c.cost_scale)
    os.makedirs(STATE, exist_ok=True)
    path = os.path.join(STATE, f"oracle_{mode}.npz")
    if os.path.exists(path):
        s = np.load(path)
        f, g, done, secs = s["f"], s["g"], int(s["done"]), float(s["secs"])
        trace = [tuple(t) for t in s["trace"]]
    else:
        f, g, done, trace, secs = d["warm_f"], d["warm_g"], 0, [], 0.0
    print(f"oracle {CFG} {mode}: threads {O.max_threads()}, resuming at {done}", flush=True)
    converged = bool(trace) and trace[-1][0] < 1e-9
    with O.accept_mode(mode):
        while not converged and done < MAX_ITER:
            t0 = time.time()
            r = O.solve(op, tol=1e-9, max_iter=CHUNK, ell=c.ell, V=d["V"], init=(f, g), trace=True)
            secs += time.time() - t0
            f, g = r["f"], r["g"]
            trace += r["trace"]
            done += r["iterations"]
            converged = r["converged"]
            np.savez(path + ".tmp.npz", f=f, g=g, done=done, trace=np.array(trace, dtype=float), secs=secs,
                     converged=converged)
            os.replace(path + ".tmp.npz", path)
            print(f"iter {done}: err {trace[-1][0]:.4e} accepts {int(sum(t[4] for t in trace))} "
                  f"({secs:.0f} s)", flush=True)


def merge():
    c = G.config(CFG)
    out = {"config": f"{CFG} n={c.n} m={c.m} d={c.x.shape[1]} eps={c.epsilon} ell={c.ell} tol=1e-9: SK-NR({c.ell}) "
                     f"main solve from the shared eps'={c.basis_eps} warm potentials and top_modes basis "
                     f"({os.path.relpath(INPUTS, ROOT)}); each side on its own iterates to tolerance",
           "modes": {}}
    for mode in ("literal", "stable"):
        gp = os.path.join(OUT, f"gpu_{mode}.npz")
        op = os.path.join(STATE, f"oracle_{mode}.npz")
        if not (os.path.exists(gp) and os.path.exists(op)):
            continue
        g, o = np.load(gp), np.load(op)
        tr = o["trace"]
        acc_g = [bool(a) for a in g["accepted"]]
        acc_o = [bool(t[4]) for t in tr]
        me_g, me_o = g["marginal_error"], tr[:, 0]
        k = min(len(me_g), len(me_o))
        diff = [i + 1 for i, (a, b) in enumerate(zip(acc_g, acc_o)) if a != b]
        fscale = float(np.max(np.abs(o["f"])))
        row = {"iterations": {"gpu": int(g["iterations"]), "oracle": int(o["done"])},
               "converged": {"gpu": bool(g["converged"]), "oracle": bool(o["converged"])},
               "oracle_complete": bool(o["converged"]),
               "oracle_s": float(o["secs"]),
               "accepts": {"gpu": int(sum(acc_g)), "oracle": int(sum(acc_o))},
               "differing_accept_iterations": diff,
               "differing_accepts_above_noise_floor": [i for i in diff if tr[i - 1][6] > 1e-10 * fscale],
               "max_rel_marginal_error_diff": float(np.max(np.abs(me_g[:k] - me_o[:k]) / me_o[:k])),
               "oracle_newton_step_max": [float(t[6]) for t in tr],
               "oracle_newton_gain": [float(t[5]) for t in tr],
               "marginal_error_gpu": [float(v) for v in me_g], "marginal_error_oracle": [float(v) for v in me_o],
               "accepted_gpu": acc_g, "accepted_oracle": acc_o}
        # potentials at each side's stopping iteration (the same iteration when the counts agree)
        row["same_iteration_count"] = int(o["done"]) == int(g["iterations"])
        row["rel_f"] = rel(g["f"], o["f"])
        row["rel_g"] = rel(g["g"], o["g"])
        out["modes"][mode] = row
    gi = os.path.join(OUT, "gpu_info.json")
    if os.path.exists(gi):
        out["gpu"] = json.load(open(gi))
    json.dump(out, open(os.path.join(ROOT, "profiles", f"{TAG}_full_parity_r02.json"), "w"), indent=1)
    for mode, row in out["modes"].items():
        print(mode, json.dumps({k: v for k, v in row.items() if not isinstance(v, list)}))


if __name__ == "__main__":
    if sys.argv[1] == "gpu":
        run_gpu()
    elif sys.argv[1] == "oracle":
        run_oracle(sys.argv[2])
    else:
        merge()
