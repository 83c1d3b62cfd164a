#!/usr/bin/env python
"""bench.py -- SK-NR(ell) hot path on B200 (driver contract).

Workload (BASELINE.json configs[3], "C4"): n = m = 65536 points uniform in
[0,1]^2, squared-Euclidean cost evaluated on the fly, uniform marginals, fp64,
eps = 5e-4, ell = 32. A "step" is one Sinkhorn-Knopp iteration of the device
solve loop (row LSE + column LSE over all n*m cells, gauge, on-device marginal
stopping test); `value` counts the 2*n*m LSE cell-passes of that sweep per
second (GCells/s of LSE sweeps). One SK-NR(32) iteration (adds the restricted
Newton step: one more LSE pair + the ell-wide V^T P~ pass) and SK / SK-NR
time-to-tolerance on C1 are reported beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the CPU oracle (the reference restated in C++,
oracle/, since the reference itself needs the absent Eigen3) on all host
cores, on a bounded column sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
if int(os.environ.get("WORLD_SIZE", "1")) > 1:
    # NCCL's INFO log lets the driver confirm the communicator spans every rank
    os.environ.setdefault("NCCL_DEBUG", "INFO")

import numpy as np  # noqa: E402

METRIC = "GCells/s of LSE sweeps (C4 Sinkhorn sweep = 2 LSE passes over n*m cells)"
UNIT = "GCells/s"
# FP64 pipe instructions per cell of the on-the-fly d=2 LSE sum kernel (pts_sum12_kernel):
# exponent 1 DADD + 2 DFMA; exp2 3 DADD (Cody-Waite) + 3 DFMA (degree-3 polynomial, 4096-entry
# table) + 1 DFMA (table x poly fused with the accumulate) = 10 issue slots, counted as 2
# flops each (FMA-equivalent).
FP64_SLOTS_PER_CELL = 10
SUM_KERNEL = "pts_sum12_kernel<2,8,512,4> (column LSE, on-the-fly d=2, 4096-entry exp2 table)"
SUM_KERNEL_PROFILE = "ncu_lse_sum12_r02.json"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C4")
    ap.add_argument("--no-ttt", action="store_true", help="skip the time-to-tolerance and batch legs")
    ap.add_argument("--no-c4-ttt", action="store_true", help="skip the C4 time-to-tolerance leg (~1 min)")
    return ap.parse_args()


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms",
                 "100", "-i", str(self.gpu)], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None
        time.sleep(0.15)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        os.unlink(self.path)
        busy = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------- distributed
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def dist_init(world):
    if world <= 1:
        return None
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    return dist


def dist_max(dist, v: float) -> float:
    if dist is None:
        return v
    import torch

    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ---------------------------------------------------------------------------- helpers
def load_oracle():
    """CPU oracle: the cpu_baseline / --impl reference legs only."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ref

    return oracle_ref


def column_sample(inst, ms):
    y = np.asfortranarray(inst.y[:ms])
    b = inst.beta[:ms] / inst.beta[:ms].sum()
    return y, b


def oracle_sweep_rate(O, inst, ms, threads, reps, warm=0):
    """GCells/s of one reference SK iteration (solve with max_iter=1: column LSE,
    row LSE, gauge, plan_marginals) on the n x ms column sample."""
    O.set_threads(threads)
    y, b = column_sample(inst, ms)
    P = O.Instance(inst.alpha, b, inst.epsilon, x=inst.x, y=y, cost_div=1.0 / inst.cost_scale)
    for _ in range(warm):
        O.solve(P, tol=1e-300, max_iter=1, trace=False)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.solve(P, tol=1e-300, max_iter=1, trace=False)
        times.append(time.perf_counter() - t0)
    t = statistics.mean(times)
    return 2.0 * inst.n * ms / t / 1e9, t, times


def read_profile_traffic(name=SUM_KERNEL_PROFILE):
    path = os.path.join(ROOT, "profiles", name)
    if os.path.exists(path):
        try:
            return json.load(open(path)).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            return None
    return None


# ---------------------------------------------------------------------------- arms
REF_BUDGET_S = float(os.environ.get("SKNR_REF_BUDGET_S", "240"))


def run_reference(args, world, rank):
    """The reference's CPU implementation of the path (the oracle restatement, all host
    cores, output-parallel and bitwise equal to one thread) on the SAME workload as our
    arm: each step is one full C4 SK iteration of solve() (column LSE, row LSE, gauge,
    plan_marginals over all 65536^2 cells; solver.cpp:104-123). A full iteration takes
    tens of seconds on the host, so the number of timed steps is capped by a time budget
    (SKNR_REF_BUDGET_S, default 240 s) after one untimed warm-up step; the line reports
    the steps it actually timed."""
    if rank != 0:
        return
    from paper_2506_14780_b200 import generators as G

    O = load_oracle()
    inst = G.config(args.config)
    threads = O.max_threads()
    O.set_threads(threads)
    P = O.Instance(inst.alpha, inst.beta, inst.epsilon, x=inst.x, y=inst.y, cost_div=1.0 / inst.cost_scale)
    f = np.zeros(inst.n)
    g = np.zeros(inst.m)
    t_start = time.perf_counter()
    warm = min(max(args.warmup, 0), 1)
    t_first = None
    for _ in range(warm):
        t0 = time.perf_counter()
        r = O.solve(P, tol=1e-300, max_iter=1, init=(f, g), trace=False)
        t_first = time.perf_counter() - t0
        f, g = r["f"], r["g"]
    times = []
    while len(times) < max(args.steps, 1):
        t0 = time.perf_counter()
        r = O.solve(P, tol=1e-300, max_iter=1, init=(f, g), trace=False)
        times.append(time.perf_counter() - t0)
        f, g = r["f"], r["g"]
        est = statistics.mean(times)
        if sum(times) + est > REF_BUDGET_S:
            break
    t = statistics.mean(times)
    cells = float(inst.n) * inst.m
    rate = 2.0 * cells / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(times), "steps_requested": args.steps, "warmup": warm, "ms_per_step": t * 1e3,
        "step_ms": [v * 1e3 for v in times], "warmup_ms": None if t_first is None else t_first * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64, BASELINE C4)",
        "same_config": True,
        "config": {"workload": f"{args.config}: n=m={inst.n}, d=2, eps={inst.epsilon}; step = one full SK "
                               "iteration of the reference solve loop over all n*m cells",
                   "n": inst.n, "m": inst.m, "epsilon": inst.epsilon},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{len(times)} full {args.config} SK iterations (column LSE, row LSE, gauge, "
                                   "plan_marginals: 6 sweeps of n*m cells, 2 of them counted as the metric's "
                                   "LSE cell-passes) after 1 untimed, capped by a "
                                   f"{REF_BUDGET_S:.0f} s budget; oracle/sknr_oracle.cpp output-parallel "
                                   "restatement (the reference needs the absent Eigen3)"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t_start,
    }
    print(json.dumps(line), flush=True)


def cpu_time_to_tol(O):
    """The reference's solve to tolerance on the host, beside the GPU numbers (BASELINE.md
    section 3): C1 SK and SK-NR(10) end to end (eps' warm solve + top_modes + main solve) on
    1 core and on all cores; the C2 anneal on all cores."""
    from paper_2506_14780_b200 import generators as G

    out = {"cores_all": O.max_threads()}
    c = G.config("C1")
    P = O.Instance(c.alpha, c.beta, c.epsilon, x=c.x, y=c.y)
    Pw = P.with_epsilon(c.basis_eps)
    for label, threads in (("cores_1", 1), ("cores_all", O.max_threads())):
        O.set_threads(threads)
        t0 = time.perf_counter()
        r_sk = O.solve(P, tol=1e-9, trace=False)
        t_sk = time.perf_counter() - t0
        t0 = time.perf_counter()
        w = O.solve(Pw, tol=1e-9, trace=False)
        b = O.top_modes(Pw, w["f"], w["g"], c.ell)
        t_b = time.perf_counter() - t0
        r_nr = O.solve(P, tol=1e-9, ell=c.ell, V=b["vectors"], init=(w["f"], w["g"]), trace=False)
        t_nr = time.perf_counter() - t0 - t_b
        out.setdefault("C1", {})[label] = {
            "threads": threads, "sk": {"iterations": r_sk["iterations"], "ms": t_sk * 1e3},
            "sknr": {"iterations": r_nr["iterations"], "ms_main_solve": t_nr * 1e3,
                     "ms_end_to_end": (t_b + t_nr) * 1e3, "warm_iterations": w["iterations"]}}
    O.set_threads(O.max_threads())
    c2 = G.config("C2")
    P2 = O.Instance(c2.alpha, c2.beta, c2.epsilons[0], x=c2.x, y=c2.y, cost_div=1.0 / c2.cost_scale)
    t0 = time.perf_counter()
    st = O.anneal(P2, list(c2.epsilons), warm="spectral", ell=c2.ell)
    out["C2_anneal"] = {"threads": O.max_threads(), "ms_total": (time.perf_counter() - t0) * 1e3,
                        "iterations": [s_["iterations"] for s_ in st]}
    return out


def run_ours(args, world, rank, local):
    gpu = local
    if world > 1:
        # one process per GPU: this rank's GPU is the only one the library sees (set before
        # anything can initialise CUDA in this process)
        os.environ["CUDA_VISIBLE_DEVICES"] = str(local)
    import paper_2506_14780_b200 as sk
    from paper_2506_14780_b200 import generators as G

    dist = dist_init(world)
    inst = G.config(args.config)
    n, m = inst.n, inst.m
    cells = float(n) * m
    if world > 1:
        # row sharding: NCCL communicator over NVLink, id shared via gloo
        import torch

        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            uid = torch.tensor(list(sk.comm_unique_id()), dtype=torch.uint8)
        dist.broadcast(uid, src=0)
        sk.comm_init(rank, world, bytes(uid.tolist()), 0)

    def make_problem():
        p = sk.PointProblem(inst.x, inst.y, inst.alpha, inst.beta, inst.epsilon, inst.cost_scale)
        if world > 1:
            sk.shard(p, rank, world)
        return p

    prob = make_problem()
    rb, re_ = sk.row_partition(n, world, rank)
    cells_local = float(re_ - rb) * m

    # ---- value: SK iterations, device-resident, L2 flushed between timed steps
    clocks = ClockSampler(gpu)
    barrier(dist)
    if world > 1:
        sk.comm_stats(reset=True)
    clocks.start()
    warm_steps = max(args.warmup, 3)
    ms_iter, kpi = sk.bench_iterations(prob, 0, None, iters=args.steps, warmup=warm_steps,
                                       flush_l2=True)
    clk = clocks.stop()
    comm = None
    if world > 1:
        calls, nbytes = sk.comm_stats(reset=True)
        comm = {"sk_iteration": {"calls": calls / (warm_steps + args.steps),
                                 "bytes": nbytes / (warm_steps + args.steps)}}
    barrier(dist)
    ms_iter_max = dist_max(dist, ms_iter)
    value = 2.0 * cells / (ms_iter_max * 1e-3) / 1e9  # whole job: all rows of C4 per step

    # ---- dominant kernel: the column-LSE sum tile kernel alone, CUDA events on its stream
    ms_pass, ms_kernel = sk.bench_pass(prob, 2, 0, passes=10)
    peak_dfma, _ = sk.bench_fp64_peak()
    sm_mhz = 1965.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            sm_mhz = float(json.load(fh)["sm_max_mhz"])
    except (OSError, KeyError, ValueError):
        pass
    peak_nominal = 148 * 64 * 2 * sm_mhz * 1e6 / 1e12  # FP64 FMA lanes x 2 flops at the max SM clock
    achieved = FP64_SLOTS_PER_CELL * 2.0 * cells_local / (ms_kernel * 1e-3) / 1e12
    gcells_kernel = cells_local / (ms_kernel * 1e-3) / 1e9
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak_nominal, "unit": "TFLOP/s",
                "frac": achieved / peak_nominal, "traffic": read_profile_traffic(),
                "kernel": SUM_KERNEL,
                "kernel_ms": ms_kernel, "kernel_gcells_per_s": gcells_kernel,
                "algorithmic_per_cell": f"{FP64_SLOTS_PER_CELL} FP64 issue slots (x2 flops)",
                "peak_source": "nominal FP64 pipe: 148 SM x 64 FMA/clk x 2 flops x sm_max_mhz "
                               "(MEASURED_PEAKS.json has no FP64 entry, B200_PROFILING.md no FP64 fallback)",
                "peak_measured_dfma": peak_dfma, "frac_vs_measured_dfma": achieved / peak_dfma,
                "survey_8d_ceiling_gcells_per_s": 886.0,
                "frac_vs_survey_8d": gcells_kernel / 886.0,
                "survey_8d_note": "SURVEY 8(d) counts 21 FP64 slots per cell (exp pinned at 12); this kernel "
                                  f"spends {FP64_SLOTS_PER_CELL} (table-driven exp2), so its 21-slot reading exceeds 1"}

    # ---- row LSE separately (K1 vs K2)
    ms_row_pass, ms_row_kernel = sk.bench_pass(prob, 1, 0, passes=5)

    # ---- stored-cost roofline (HBM): C5 (32768 x 16384, d = 64) with the cost built once on device,
    # column LSE streaming 8 B per cell with 128-bit loads
    stored = None
    if world == 1 and not args.no_ttt:
        c5 = G.config("C5")
        p5 = sk.PointProblem(c5.x, c5.y, c5.alpha, c5.beta, c5.epsilon, cost_mode="stored")
        ms5, k5 = sk.bench_pass(p5, 2, 0, passes=10)
        cells5 = float(c5.n) * c5.m
        hbm_peak = 6552.0
        try:
            with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as fh:
                hbm_peak = float(json.load(fh)["hbm_gbs"])
        except (OSError, KeyError, ValueError):
            pass
        gbs = 8.0 * cells5 / (k5 * 1e-3) / 1e9
        stored = {"workload": "C5 stored cost: n=32768, m=16384, d=64, column LSE sum kernel (dense_v2)",
                  "kernel_ms": k5, "gcells_per_s": cells5 / (k5 * 1e-3) / 1e9, "bound": "hbm",
                  "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                  "algorithmic_per_cell": "8 B (the fp64 cost element, read once)",
                  "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured; a STREAM copy, so a read-only "
                                 "stream can land slightly above 1.0)"}
        del p5

    # ---- SK-NR(ell) iteration (restricted Newton step included)
    rng = np.random.default_rng(0)
    V = np.linalg.qr(rng.standard_normal((n, inst.ell)))[0] * np.sqrt(n)
    basis = sk.SpectralBasis(np.asfortranarray(V), np.asfortranarray(V), np.zeros(inst.ell), inst.epsilon)
    ms_nr, kpi_nr = sk.bench_iterations(prob, inst.ell, basis, iters=max(3, args.steps // 10), warmup=1,
                                        flush_l2=True)
    if world > 1:
        sk.comm_stats(reset=True)
    ms_nr_st, kpi_nr_st = sk.bench_iterations(prob, inst.ell, basis, iters=max(3, args.steps // 10), warmup=1,
                                              flush_l2=True, accept="stable")
    if world > 1:
        calls, nbytes = sk.comm_stats(reset=True)
        comm["sknr_iteration_stable"] = {"calls": calls / (1 + max(3, args.steps // 10)),
                                         "bytes": nbytes / (1 + max(3, args.steps // 10))}

    # ---- the Newton derivative pass alone (S = V^T P~, r = P~ beta): tensor-core slices vs FP64 DMMA
    newton_pass = None
    if world == 1 and inst.ell <= 32:
        ms_i8, k_i8 = sk.bench_pass(prob, 4, inst.ell, passes=5)
        prev = sk.set_tensor_block_pass(False)
        try:
            ms_f64, k_f64 = sk.bench_pass(prob, 4, inst.ell, passes=5)
        finally:
            sk.set_tensor_block_pass(prev)
        slots = 14.0  # FP64 issue slots per cell of pts_i8w_kernel (DESIGN 4.1)
        newton_pass = {"ell": inst.ell,
                       "tensor_core": {"kernel": "pts_i8w_kernel (tcgen05.mma.kind::i8 over exact byte slices)",
                                       "pass_ms": ms_i8, "kernel_ms": k_i8,
                                       "gcells_per_s": cells / (k_i8 * 1e-3) / 1e9,
                                       "fp64_slots_per_cell": slots,
                                       "int8_macs_per_cell": 1120,
                                       "frac_of_nominal_fp64": slots * 2 * cells / (k_i8 * 1e-3) / 1e12 / peak_nominal,
                                       "int8_tmacs_per_s": 1120 * cells / (k_i8 * 1e-3) / 1e12},
                       "fp64_dmma": {"kernel": "pts_mma2_kernel<.., RS> (mma.sync m8n8k4 f64)",
                                     "pass_ms": ms_f64, "kernel_ms": k_f64,
                                     "gcells_per_s": cells / (k_f64 * 1e-3) / 1e9}}

    # ---- e2e: public C ABI with host buffers (problem upload + solve + potentials download)
    # Five complete runs (each: new problem from host arrays, K iterations, download);
    # the median is reported, all five are listed (host-side allocation jitter).
    k_e2e = max(args.steps, 1)
    runs = []
    for _ in range(5):
        barrier(dist)
        t0 = time.perf_counter()
        p2 = make_problem()
        res = sk.solve(p2, tol=1e-300, max_iter=k_e2e, trace=False)
        t_run = time.perf_counter() - t0
        assert res.iterations == k_e2e
        runs.append(dist_max(dist, t_run))
        del p2
    t_e2e = statistics.median(runs)
    h2d = (inst.x.nbytes + inst.y.nbytes + inst.alpha.nbytes + inst.beta.nbytes) / k_e2e
    d2h = (res.f.nbytes + res.g.nbytes) / k_e2e
    e2e = {"value": 2.0 * cells * k_e2e / t_e2e / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "steps": k_e2e, "runs_s": runs, "statistic": "median of 5 runs",
           "path": "PointProblem(host arrays) + sknr_solve(max_iter=K) + f,g download, wall clock"}

    # ---- time to tolerance: C1 (reference basis method) and C3 (Chebyshev-filtered basis)
    ttt = None

    kept = {}

    def ttt_case(name, method, cull=0.0, degree=8):
        # SK and SK-NR(ell) to marginal error 1e-9 from inputs resident on the device;
        # SK-NR end to end = warm SK solve at eps' + top_modes basis + main solve.
        # Under torchrun every rank holds its row shard and each time is the max over ranks.
        c = G.config(name)
        p1 = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.epsilon, c.cost_scale)
        p1w = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.basis_eps, c.cost_scale)
        if world > 1:
            sk.shard(p1, rank, world)
            sk.shard(p1w, rank, world)
        if cull:
            p1.set_culling(cull)
            p1w.set_culling(cull)

        def timed(fn):
            barrier(dist)
            t0 = time.perf_counter()
            out = fn()
            return out, dist_max(dist, time.perf_counter() - t0)

        r_sk, t_sk = timed(lambda: sk.solve(p1, tol=1e-9, trace=False))
        if not cull:
            kept[name] = r_sk
        warm, t_warm = timed(lambda: sk.solve(p1w, tol=1e-9, trace=False))
        b1, t_basis = timed(lambda: sk.top_modes(p1w, warm.f, warm.g, c.ell, method=method, degree=degree,
                                                 max_power_iters=200000))
        r_nr, t_nr = timed(lambda: sk.solve(p1, tol=1e-9, ell=c.ell, basis=b1, init=(warm.f, warm.g),
                                            trace=False))
        r_st, t_st = timed(lambda: sk.solve(p1, tol=1e-9, ell=c.ell, basis=b1, init=(warm.f, warm.g),
                                            trace=False, accept="stable"))
        if not cull:
            kept[name + "_nr"] = r_nr
        return {"n": c.n, "m": c.m, "d": c.x.shape[1], "epsilon": c.epsilon, "tol": 1e-9,
                "culling": cull or None, "ranks": world,
                "sk": {"iterations": r_sk.iterations, "converged": r_sk.converged, "ms": t_sk * 1e3},
                "sknr": {"ell": c.ell, "iterations": r_nr.iterations, "converged": r_nr.converged,
                         "ms_main_solve": t_nr * 1e3,
                         "ms_end_to_end": (t_warm + t_basis + t_nr) * 1e3,
                         "warm_eps": c.basis_eps, "warm_iterations": warm.iterations,
                         "warm_ms": t_warm * 1e3, "basis_method": f"{method}({degree})",
                         "basis_operator_applications": b1.sweeps, "basis_ms": t_basis * 1e3},
                "sknr_stable_accept": {"iterations": r_st.iterations, "converged": r_st.converged,
                                       "ms_main_solve": t_st * 1e3,
                                       "ms_end_to_end": (t_warm + t_basis + t_st) * 1e3}}

    cull_note = ("opt-in culling (sknr_problem_set_culling, T=60): terms below e^-60 of their output's "
                 "total skipped under rigorous group bounds")
    # C4 basis: restarted block Lanczos (12 blocks per cycle; 26 operator applications vs 81
    # for Chebyshev(16))
    if not args.no_ttt and world > 1 and not args.no_c4_ttt:
        # north-star time-to-tolerance at R GPUs: C4 row-sharded over all ranks (NCCL)
        ttt = {"C4": ttt_case("C4", "lanczos", degree=12),
               "C4_culled": ttt_case("C4", "lanczos", cull=60.0, degree=12)}
        ttt["C4_culled"]["note"] = cull_note
    if not args.no_ttt and world == 1:
        ttt = {"C1": ttt_case("C1", "subspace"), "C3": ttt_case("C3", "chebyshev")}
        # C2 (BASELINE configs[1]): the reference's anneal driver, eps 0.1 -> 0.001 halving,
        # spectral warm start, ell = 16, refresh_basis = false (solver.hpp:44)
        c2 = G.config("C2")
        p2c = sk.PointProblem(c2.x, c2.y, c2.alpha, c2.beta, c2.epsilons[0], c2.cost_scale)
        t0 = time.perf_counter()
        stages = sk.anneal(p2c, list(c2.epsilons), warm="spectral", ell=c2.ell)
        t_an = time.perf_counter() - t0
        ttt["C2_anneal"] = {"n": c2.n, "m": c2.m, "epsilons": list(c2.epsilons), "ell": c2.ell, "tol": 1e-9,
                            "warm": "spectral", "ms_total": t_an * 1e3,
                            "iterations": [s.iterations for s in stages],
                            "converged": all(s.converged for s in stages)}
        del p2c
        if not args.no_c4_ttt:
            ttt["C4"] = ttt_case("C4", "lanczos", degree=12)
            ttt["C4_culled"] = ttt_case("C4", "lanczos", cull=60.0, degree=12)
            ttt["C4_culled"]["note"] = cull_note

    # ---- opt-in fp32 variant (sknr_problem_set_precision(32), north star "1e-5 if an fp32
    # variant is offered"): LSE sum passes with fp32 exponents on the MUFU ex2 unit
    fp32 = None
    if world == 1 and not args.no_ttt:
        p32 = make_problem()
        p32.set_precision(32)
        gex2, _ = sk.bench_mufu_peak()
        ms32_pass, ms32_k = sk.bench_pass(p32, 2, 0, passes=10)
        ms32_it, _ = sk.bench_iterations(p32, 0, None, iters=args.steps, warmup=max(args.warmup, 3),
                                         flush_l2=True)
        g32 = cells / (ms32_k * 1e-3) / 1e9
        fp32 = {"sweep_gcells_per_s": 2.0 * cells / (ms32_it * 1e-3) / 1e9, "ms_per_step": ms32_it,
                "roofline": {"bound": "mufu", "kernel": "pts_f32_kernel<2,8,512,2> (column LSE, fp32 exponent, "
                                                        "ex2.approx)",
                             "kernel_ms": ms32_k, "achieved": g32, "peak": gex2, "unit": "G ex2/s",
                             "frac": g32 / gex2, "algorithmic_per_cell": "1 MUFU ex2 + 7 FP32 ops",
                             "traffic": read_profile_traffic("ncu_lse_f32_kernel_r01.json"),
                             "peak_source": "measured ex2-only kernel on this GPU (sknr_bench_mufu_peak)"}}
        if "C4" in kept:
            ref = kept["C4"]
            t0 = time.perf_counter()
            r32 = sk.solve(p32, tol=1e-9, trace=False)
            t32 = time.perf_counter() - t0
            fp32["C4_sk_ttt"] = {"iterations": r32.iterations, "converged": r32.converged, "ms": t32 * 1e3,
                                 "fp64_iterations": ref.iterations,
                                 "rel_f_vs_fp64": float(np.max(np.abs(r32.f - ref.f)) / np.max(np.abs(ref.f))),
                                 "rel_g_vs_fp64": float(np.max(np.abs(r32.g - ref.g)) / np.max(np.abs(ref.g)))}
        # SK-NR(ell) end to end with only the eps' warm solve in fp32: the basis and the main
        # solve are the fp64 path, from a warm start that differs at the fp32 level (C4 dense
        # and culled on every pass, Lanczos basis; C3 with the Chebyshev basis of its fp64 leg)
        cases = [("C4_sknr_fp32_warm", "C4", 0.0, "lanczos", 12), ("C4_sknr_fp32_warm_culled", "C4", 60.0, "lanczos", 12),
                 ("C3_sknr_fp32_warm", "C3", 0.0, "chebyshev", 8)]
        for key, name, cull, method, degree in cases:
            if name + "_nr" not in kept:
                continue
            c = G.config(name)
            ref = kept[name + "_nr"]
            pw = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.basis_eps, c.cost_scale)
            pm = sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.epsilon, c.cost_scale)
            if cull:
                pw.set_culling(cull)
                pm.set_culling(cull)
            pw.set_precision(32)
            t0 = time.perf_counter()
            w32 = sk.solve(pw, tol=1e-9, trace=False)
            t_w = time.perf_counter() - t0
            pw.set_precision(64)
            b32 = sk.top_modes(pw, w32.f, w32.g, c.ell, method=method, degree=degree, max_power_iters=200000)
            t_b = time.perf_counter() - t0 - t_w
            t0 = time.perf_counter()
            rm = sk.solve(pm, tol=1e-9, ell=c.ell, basis=b32, init=(w32.f, w32.g), trace=False)
            t_m = time.perf_counter() - t0
            fp32[key] = {
                "culling": cull or None, "warm_iterations": w32.iterations, "warm_ms": t_w * 1e3,
                "basis_ms": t_b * 1e3, "basis_method": f"{method}({degree})",
                "basis_operator_applications": b32.sweeps, "main_iterations": rm.iterations,
                "main_converged": rm.converged, "main_ms": t_m * 1e3,
                "ms_end_to_end": (t_w + t_b + t_m) * 1e3,
                "fp64_pipeline_main_iterations": ref.iterations,
                "rel_f_vs_fp64_pipeline": float(np.max(np.abs(rm.f - ref.f)) / np.max(np.abs(ref.f))),
                "note": f"eps'={c.basis_eps} warm SK solve in fp32, basis and main SK-NR({c.ell}) solve in fp64"}
            del pw, pm
        del p32

    # ---- batched small problems: 32 C1 instances, SK to 1e-9
    batch = None
    if not args.no_ttt and world == 1:
        probs = []
        for s in range(32):
            c = G.config("C1", seed=1 + s)
            probs.append(sk.PointProblem(c.x, c.y, c.alpha, c.beta, c.epsilon))
        sk.solve_batch(probs[:2], tol=1e-9)
        t0 = time.perf_counter()
        rb = sk.solve_batch(probs, tol=1e-9)
        t_b = time.perf_counter() - t0
        t0 = time.perf_counter()
        r1 = [sk.solve(p, tol=1e-9, trace=False) for p in probs[:8]]
        t_1 = (time.perf_counter() - t0) / 8
        # one CTA per problem, whole SK loop in one kernel (sknr_solve_small_batch): 148 instances
        tup = []
        for s in range(148):
            c = G.config("C1", seed=1 + s)
            tup.append((c.x, c.y, c.alpha, c.beta, c.epsilon))
        sk.solve_small_batch(tup[:2], tol=1e-9)
        t0 = time.perf_counter()
        rsm = sk.solve_small_batch(tup, tol=1e-9)
        t_sm = time.perf_counter() - t0
        # the same kernel on ONE problem: a cooperative group of CTAs (low-latency single solve)
        sk.solve_small_batch(tup[:1], tol=1e-9)
        t1s = []
        for _ in range(3):
            t0 = time.perf_counter()
            r_one = sk.solve_small_batch(tup[:1], tol=1e-9)[0]
            t1s.append(time.perf_counter() - t0)
        small = {"problems": len(tup), "ms": t_sm * 1e3, "solves_per_s": len(tup) / t_sm,
                 "all_converged": all(r.converged for r in rsm),
                 "iterations_equal_first32": all(a.iterations == b.iterations for a, b in zip(rsm, rb)),
                 "single_problem_ms": min(t1s) * 1e3, "single_problem_iterations": r_one.iterations,
                 "single_problem_note": "C1 seed 1 alone: a group of CTAs with two group barriers per "
                                        "iteration, host arrays in and potentials out (min of 3)"}
        batch = {"problems": len(probs), "config": "C1 seeds 1..32, SK (ell=0) to marginal error 1e-9",
                 "small_problem_kernel": small,
                 "ms_batch": t_b * 1e3, "solves_per_s": len(probs) / t_b, "ms_per_solve_one_by_one": t_1 * 1e3,
                 "speedup_vs_one_by_one": t_1 * len(probs) / t_b,
                 "all_converged": all(r.converged for r in rb),
                 "bitwise_equal_first8": all(np.array_equal(a.f, b.f) for a, b in zip(rb[:8], r1))}
        del probs

    # ---- CPU baseline: oracle, 1 core (the reference is single-threaded by design)
    cpu = None
    cpu_ttt = None
    if rank == 0 and world == 1 and not args.no_ttt:
        cpu_ttt = cpu_time_to_tol(load_oracle())
    if rank == 0:
        O = load_oracle()
        ms_s = 256
        rate, t, _ = oracle_sweep_rate(O, inst, ms_s, 1, reps=2)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"n={n} x m={ms_s} columns of C4, one reference SK iteration (column LSE, row "
                         "LSE, gauge, plan_marginals) per rep, 2 reps, oracle/sknr_oracle.cpp"}

    launches = int(kpi * args.steps)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_iter_max, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded SplitMix64 point clouds, BASELINE C4)",
            "config": {"workload": "C4: n=m=65536, d=2 uniform [0,1]^2, on-the-fly squared-Euclidean cost, "
                                   "uniform marginals, eps=5e-4; step = one SK iteration of the device loop",
                       "n": n, "m": m, "d": 2, "epsilon": inst.epsilon,
                       "l2": "flushed between timed steps (256 MiB memset, untimed)",
                       "parallelism": f"row-sharded x{world} (NCCL)" if world > 1 else "single GPU"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "kernels_per_step": kpi,
            "clocks": clk,
            "sknr_iteration": {"ell": inst.ell, "ms": ms_nr, "kernels": kpi_nr,
                               "cell_passes": 4, "gcells_per_s": 4 * cells / (ms_nr * 1e-3) / 1e9,
                               "note": "2 sweep LSEs + fused V^T P~ / P~ beta pass + candidate column LSE",
                               "stable_accept": {"ms": ms_nr_st, "kernels": kpi_nr_st,
                                                 "note": "candidate column LSE replaced by the anchor pass "
                                                         "s, t, u = P~^T (1, expm1(d/eps), exp(d/eps))"}},
            "newton_pass": newton_pass,
            "collectives": comm,
            "cpu_time_to_tol": cpu_ttt,
            "pass_ms": {"column_lse_full": ms_pass, "row_lse_full": ms_row_pass,
                        "row_lse_kernel_gcells_per_s": cells_local / (ms_row_kernel * 1e-3) / 1e9},
            "roofline_stored": stored,
            "fp32_variant": fp32,
            "time_to_tol": ttt,
            "batch_c1": batch,
            "library": sk.version(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        sk.comm_destroy()
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
