"""Row sharding on CPU (gloo, world size 2): the merge the GPU path performs
across ranks -- each rank's column sums under its OWN shift (its local exact max, or a
local bound), one all-gather of (shift_r, S_r) and the fixed rank-order merge
L_j = M_j + log(sum_r S_rj exp(shift_rj - M_j)) (engine.cu lse(), k_lse_merge) --
reproduces the unsharded column transform, and the row transform is local.
Uses the oracle on each rank's row block as the per-rank compute."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_ref as O
from paper_2506_14780_b200 import generators as G
from paper_2506_14780_b200 import row_partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _column_partials(x, y, a, f, eps, shift):
    """S_j = sum_i a_i exp((f_i - C_ij)/eps - shift_j) over this rank's rows."""
    C = ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)
    return np.exp(np.log(a)[:, None] + (f[:, None] - C) / eps - shift[None, :]).sum(0)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    inst = G.config("C1", n=96, m=80)
    eps = 0.05
    f = np.linspace(-0.1, 0.1, inst.n)
    b0, b1 = row_partition(inst.n, world, rank)
    xs, as_, fs = inst.x[b0:b1], inst.alpha[b0:b1], f[b0:b1]
    # rank-local shift (this rank's exact column max; a looser local bound works the same)
    C = ((xs[:, None, :] - inst.y[None, :, :]) ** 2).sum(-1)
    shift_r = (np.log(as_)[:, None] + (fs[:, None] - C) / eps).max(0)
    if rank == 1:
        shift_r = shift_r + 3.0  # a loose bound on one rank: the merge must not care
    S_r = _column_partials(xs, inst.y, as_, fs, eps, shift_r)
    row = torch.from_numpy(np.concatenate([shift_r, S_r]))
    rows = [torch.zeros_like(row) for _ in range(world)]
    dist.all_gather(rows, row)
    X = np.stack([r_.numpy() for r_ in rows])  # [R][2m], rank order
    m = inst.m
    M = X[:, :m].max(0)
    T = np.zeros(m)
    for r in range(world):  # fixed rank order
        T += X[r, m:] * np.exp(X[r, :m] - M)
    g = -eps * (M + np.log(T))
    # row transform of the local block is independent of the other ranks
    P = O.Instance(as_ / as_.sum(), inst.beta, eps, x=xs, y=inst.y)
    f_local = O.ctransform_of_g(P, g)
    gathered = [torch.zeros(n, dtype=torch.float64) for n in [row_partition(inst.n, world, r)[1] - row_partition(inst.n, world, r)[0]
                                         for r in range(world)]]
    dist.all_gather(gathered, torch.from_numpy(f_local))
    if rank == 0:
        q.put((g, np.concatenate([t.numpy() for t in gathered])))
    dist.destroy_process_group()


def test_two_rank_column_merge_matches_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    g_sharded, f_sharded = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    inst = G.config("C1", n=96, m=80)
    P = O.Instance(inst.alpha, inst.beta, 0.05, x=inst.x, y=inst.y)
    f = np.linspace(-0.1, 0.1, inst.n)
    g_ref = O.ctransform_of_f(P, f)
    assert np.max(np.abs(g_sharded - g_ref)) <= 1e-13 * np.max(np.abs(g_ref))
    f_ref = O.ctransform_of_g(P, g_ref)
    assert np.max(np.abs(f_sharded - f_ref)) <= 1e-12 * np.max(np.abs(f_ref))


def test_row_partition_is_contiguous_and_complete():
    for n in (1, 7, 512, 65536):
        for world in (1, 2, 3, 8):
            blocks = [row_partition(n, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            for (b0, e0), (b1, _) in zip(blocks, blocks[1:]):
                assert e0 == b1 and b0 <= e0


def _newton_worker(rank, world, port, q):
    """Newton exchange (engine_solver.cuh): each rank forms its partial
    S_r = V_r^T P~_r (m x ell) over its rows, writes it rank-blocked (block q = target rows
    [q mb, (q+1) mb), mb = ceil(m/R), zero-padded: k_block_finalize blk_rows), one
    reduce-scatter leaves rank q the summed block q, the rank adds its rows of
    cross = S diag(b) S^T to its partial G1 = V_r^T diag(r_r) V_r and grad, and ONE
    allreduce of [G1 | cross | grad] completes the ell x ell system on every rank."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, m, ell, eps = 90, 77, 5, 0.05
    inst = G.config("C1", n=n, m=m)
    rng = np.random.default_rng(3)
    f = 0.05 * rng.standard_normal(n)
    V = rng.standard_normal((n, ell))
    P = O.Instance(inst.alpha, inst.beta, eps, x=inst.x, y=inst.y)
    h = O.ctransform_of_f(P, f)
    C = ((inst.x[:, None, :] - inst.y[None, :, :]) ** 2).sum(-1)
    Pt = inst.alpha[:, None] * np.exp((f[:, None] + h[None, :] - C) / eps)  # P~ (n x m)
    b0, b1 = row_partition(n, world, rank)
    S_r = Pt[b0:b1].T @ V[b0:b1]                      # m x ell, this rank's rows
    r_r = Pt[b0:b1] @ inst.beta                       # r = P~ beta on this rank's rows
    mb = (m + world - 1) // world
    blocked = np.zeros((world, ell, mb))              # rank-blocked send buffer
    for j in range(m):
        blocked[j // mb, :, j % mb] = S_r[j]
    send = torch.from_numpy(blocked.reshape(-1).copy())
    recv = torch.zeros(ell * mb, dtype=torch.float64)
    # gloo has no reduce_scatter: an all-reduce then this rank's block is the same sum
    dist.all_reduce(send)
    recv.copy_(send[rank * ell * mb:(rank + 1) * ell * mb])
    S_loc = recv.numpy().reshape(ell, mb).T           # mb x ell, ld = mb
    j0 = min(m, rank * mb)
    rows = min(m, j0 + mb) - j0
    G1 = V[b0:b1].T @ (r_r[:, None] * V[b0:b1])
    cross = S_loc[:rows].T @ (inst.beta[j0:j0 + rows, None] * S_loc[:rows])
    grad = V[b0:b1].T @ (inst.alpha[b0:b1] - r_r)
    buf = torch.from_numpy(np.concatenate([G1.ravel(), cross.ravel(), grad]))
    dist.all_reduce(buf)
    if rank == 0:
        q.put((buf.numpy(), Pt, V, inst.alpha, inst.beta))
    dist.destroy_process_group()


def test_two_rank_newton_exchange_matches_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_newton_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    buf, Pt, V, a, b = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ell = V.shape[1]
    r = Pt @ b
    S = Pt.T @ V
    ref = np.concatenate([(V.T @ (r[:, None] * V)).ravel(), (S.T @ (b[:, None] * S)).ravel(), V.T @ (a - r)])
    assert np.max(np.abs(buf - ref)) <= 1e-13 * np.max(np.abs(ref))
    assert buf.size == 2 * ell * ell + ell
