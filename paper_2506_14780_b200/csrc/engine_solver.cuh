// engine_solver.cuh -- the SK-NR(ell) solve loop: one iteration as a captured graph body, device-side WHILE loop, batches
// Part of the libsknr_b200 translation unit: included once, in order, by engine.cu
// (shares its types, static helpers and kernels; not a standalone header).
#pragma once

// ============================================================ solve
struct SolveState {
    DBuf f, g, gnext, h, fcand, hcand, rowres, colres, am, r, Lr, V, Wv, S, delta, G;
    DBuf trace_raw;  // sknr_record array (as doubles)
};

struct SolveOut {
    std::vector<double> f, g;
    int64_t iterations = 0;
    bool converged = false;
    std::vector<sknr_record> trace;
};

// Enqueue one SK-NR(ell) iteration (solver.cpp:104-151).
static void enqueue_iteration(Problem& P, SolveState& S, int64_t ell, bool trace_enabled,
                              int64_t trace_cap, bool exact_marginals = false,
                              cudaGraphConditionalHandle loop = 0) {
    const int64_t n = P.n, m = P.m;
    cudaStream_t s = P.stream;
    const bool newton = ell > 0;
    count_launch();
    k_iter_begin<<<1, 32, 0, s>>>(P.st);
    // sk_sweep: g = f^{C,eps} (computed at the end of the previous iteration), f = g^{C,eps}
    count_launch();
    k_copy<<<grid_for(m), AUX_NT, 0, s>>>(S.g.p, S.gnext.p, m, P.st, G_DONE);
    lse(P, 1, S.g.p, S.f.p, G_DONE);
    // gauge (solver.cpp:108-112): c = alpha . f
    {
        RedArgs ra;
        ra.T[0] = n;
        ra.nterms = 1;
        ra.x[0] = P.src.w.p;
        ra.y[0] = S.f.p;
        ra.op[0] = RED_DOT;
        ra.out = P.sums.p + 8;
        ra.part = P.gram_part.p;
        ra.counter = &P.st->counters[6];
        ra.epilogue = P.shard ? EPI_NONE : EPI_GAUGE;
        ra.st = P.st;
        ra.guard = G_DONE;
        count_launch();
        k_reduce<<<reduce_blocks(n), AUX_NT, 0, s>>>(ra);
        if (P.shard) {
            allreduce(P, P.sums.p + 8, 1, ncclSum);
            count_launch();
            k_epilogue<<<1, 32, 0, s>>>(P.st, EPI_GAUGE, 0, P.sums.p + 8, G_DONE);
        }
    }
    count_launch();
    k_gauge_apply<<<grid_for(n + m), AUX_NT, 0, s>>>(S.f.p, P.L[1].p, P.src.w.p, n, S.g.p, m,
                                                     P.inv_eps(), S.rowres.p, P.st);
    // h = f^{C,eps}: the column marginal and the next sweep's g
    lse(P, 0, S.f.p, S.h.p, G_DONE);
    if (exact_marginals) {
        // reference-faithful plan_marginals (core.cpp:120-143): explicit row and
        // column sums of a_i b_j exp((f_i + g_j - C_ij)/eps) at the gauged (f, g)
        PassSpec pr;
        pr.dir = 1;
        pr.in_v = S.g.p;
        pr.in_lw = P.tgt.lw.p;
        pr.out_v = S.f.p;
        pr.out_lw = P.src.lw.p;
        pr.out = S.rowres.p;
        pr.guard = G_DONE;
        plan_pass(P, pr);
        PassSpec pc;
        pc.dir = 0;
        pc.in_v = S.f.p;
        pc.in_lw = P.src.lw.p;
        pc.out_v = S.g.p;
        pc.out_lw = P.tgt.lw.p;
        pc.out = S.colres.p;
        pc.guard = G_DONE;
        plan_pass(P, pc);
        count_launch();
        k_axpby<<<grid_for(n), AUX_NT, 0, s>>>(S.rowres.p, P.src.w.p, n, 1.0, -1.0, S.rowres.p);
        count_launch();
        k_axpby<<<grid_for(m), AUX_NT, 0, s>>>(S.colres.p, P.tgt.w.p, m, 1.0, -1.0, S.colres.p);
    } else {
        count_launch();
        k_colres<<<grid_for(m), AUX_NT, 0, s>>>(S.g.p, S.h.p, P.tgt.w.p, m, P.inv_eps(), S.colres.p, P.st,
                                                G_DONE);
    }
    double* sums = P.sums.p;
    // marginal_gap (core.cpp:145-150) + Q0 = a.f + b.h, stopping test on device
    {
        RedArgs ra;
        ra.T[0] = n;
        ra.T[1] = m;
        ra.nterms = 6;
        // layout: |row-a|^2, a.f, max|row-a| (sharded rows) | |col-b|^2, max|col-b|, b.h
        const double* xs[6] = {S.rowres.p, P.src.w.p, S.rowres.p, S.colres.p, S.colres.p, P.tgt.w.p};
        const double* ys[6] = {nullptr, S.f.p, nullptr, nullptr, nullptr, S.h.p};
        const int ops[6] = {RED_SQ, RED_DOT, RED_MAXABS, RED_SQ, RED_MAXABS, RED_DOT};
        for (int t = 0; t < 6; ++t) {
            ra.x[t] = xs[t];
            ra.y[t] = ys[t];
            ra.op[t] = ops[t];
            ra.seg[t] = t < 3 ? 0 : 1;
        }
        ra.out = sums;
        ra.part = P.gram_part.p;
        ra.counter = &P.st->counters[6];
        ra.epilogue = P.shard ? EPI_NONE : EPI_CHECK;
        ra.newton = newton ? 1 : 0;
        ra.st = P.st;
        ra.guard = G_DONE;
        count_launch();
        k_reduce<<<reduce_blocks(n + m), AUX_NT, 0, s>>>(ra);
        if (P.shard) {
            allreduce(P, sums, 2, ncclSum);
            allreduce(P, sums + 2, 1, ncclMax);
            count_launch();
            k_epilogue<<<1, 32, 0, s>>>(P.st, EPI_CHECK, newton ? 1 : 0, sums, G_DONE);
        }
    }
    if (newton) {
        const unsigned gn = G_DONE | G_NEWTON;
        const int l = static_cast<int>(ell);
        const bool cull_nr = cull_block_active(P, 0) && cull_active(P, 1);
        const bool fuse_r = block_rs_fusable(P) && !cull_nr;
        if (!fuse_r) {
            // r = P~ beta at (f, h): alpha - r = -a expm1(f/eps + L_row(h))
            lse(P, 1, S.h.p, nullptr, gn);
            count_launch();
            k_newton_r<<<grid_for(n), AUX_NT, 0, s>>>(S.f.p, P.L[1].p, P.src.w.p, n, P.inv_eps(), S.am.p,
                                                      S.r.p, P.st, gn);
        }
        // S = V^T P~ (m x ell), P~_ij = a_i e^{(f_i + h_j - C_ij)/eps}; with fuse_r the
        // same cells also give r = P~ beta (objective.cpp:127-128) in this pass
        PassSpec sp;
        sp.dir = 0;
        sp.in_v = S.f.p;
        sp.in_lw = P.src.lw.p;
        sp.out_v = S.h.p;
        sp.W = S.Wv.p;
        sp.k = l;
        sp.kt = block_kt_for(l);
        sp.out = S.S.p;
        sp.rsum_out = fuse_r ? S.r.p : nullptr;
        sp.cull = cull_nr;  // P~ columns sum to 1 at h = f^{C,eps}: no normalisation needed
        sp.guard = gn;
        plan_pass(P, sp);
        if (fuse_r) {
            count_launch();
            k_axpby<<<grid_for(n), AUX_NT, 0, s>>>(P.src.w.p, S.r.p, n, 1.0, -1.0, S.am.p);
        }
        // (plan_pass has already summed S = V^T P~ over the row shards)
        double* G1 = S.G.p;
        double* cross = G1 + l * l;
        double* grad = cross + l * l;
        gram(P, n, l, l, S.V.p, n, S.V.p, n, S.r.p, G1, gn);
        gram(P, m, l, l, S.S.p, m, S.S.p, m, P.tgt.w.p, cross, gn);
        gram(P, n, l, 1, S.V.p, n, S.am.p, n, nullptr, grad, gn);
        allreduce(P, G1, static_cast<size_t>(l) * l, ncclSum);
        allreduce(P, grad, l, ncclSum);
        count_launch();
        k_newton_solve<<<1, 256, sizeof(double) * l * l, s>>>(G1, cross, grad, l, P.inv_eps(), S.delta.p,
                                                            P.st, gn);
        count_launch();
        k_fcand<<<grid_for(n), AUX_NT, 0, s>>>(S.f.p, S.V.p, n, l, S.delta.p, S.fcand.p, P.st, gn);
        lse(P, 0, S.fcand.p, S.hcand.p, gn);
        {
            RedArgs ra;
            ra.T[0] = n;
            ra.T[1] = m;
            ra.nterms = 2;
            ra.x[0] = P.src.w.p;
            ra.y[0] = S.fcand.p;
            ra.x[1] = P.tgt.w.p;
            ra.y[1] = S.hcand.p;
            ra.op[0] = ra.op[1] = RED_DOT;
            ra.seg[1] = 1;
            ra.out = sums + 6;
            ra.part = P.gram_part.p;
            ra.counter = &P.st->counters[6];
            ra.epilogue = P.shard ? EPI_NONE : EPI_ACCEPT;
            ra.st = P.st;
            ra.guard = gn;
            count_launch();
            k_reduce<<<reduce_blocks(n + m), AUX_NT, 0, s>>>(ra);
            if (P.shard) {
                allreduce(P, sums + 6, 1, ncclSum);
                count_launch();
                k_epilogue<<<1, 32, 0, s>>>(P.st, EPI_ACCEPT, 0, sums + 6, gn);
            }
        }
        count_launch();
        k_select<<<grid_for(n + m), AUX_NT, 0, s>>>(S.f.p, S.fcand.p, n, S.gnext.p, S.h.p, S.hcand.p, m,
                                                    P.st);
    } else {
        count_launch();
        k_copy<<<grid_for(m), AUX_NT, 0, s>>>(S.gnext.p, S.h.p, m, P.st, G_DONE);
    }
    count_launch();
    k_record<<<1, 32, 0, s>>>(P.st, reinterpret_cast<sknr_record*>(S.trace_raw.p), trace_cap,
                              trace_enabled ? 1 : 0, loop);
    CK(cudaGetLastError());
}

static void prepare_solve(Problem& P, SolveState& S, int64_t ell, const double* basis_host,
                          const double* init_f, int64_t max_iter, double tol, int64_t trace_cap) {
    const int64_t n = P.n, m = P.m;
    cudaStream_t s = P.stream;
    S.f.ensure(n);
    S.g.ensure(m);
    S.gnext.ensure(m);
    S.h.ensure(m);
    S.fcand.ensure(n);
    S.hcand.ensure(m);
    S.rowres.ensure(n);
    S.colres.ensure(m);
    S.am.ensure(n);
    S.r.ensure(n);
    S.delta.ensure(64);
    S.G.ensure(3 * 64 * 64);
    S.trace_raw.ensure(std::max<int64_t>(trace_cap, 1) * (sizeof(sknr_record) / sizeof(double)));
    P.misc.ensure(256);
    if (ell > 0) {
        const int kt = block_kt_for(static_cast<int>(ell));
        S.V.ensure(n * ell);
        S.Wv.ensure(n * kt);
        S.S.ensure(m * ell);
        upload_rows(P, S.V.p, basis_host, ell);
        count_launch();
        k_pack_w<<<grid_for(n * kt), AUX_NT, 0, s>>>(S.V.p, n, n, static_cast<int>(ell), kt, nullptr,
                                                     S.Wv.p);
        // pre-size the block-pass partials outside graph capture
        const bool cull_nr = cull_block_active(P, 0) && cull_active(P, 1);
        plan_for(P, 0, cull_nr ? MODE_BLOCK_CULL : (block_rs_fusable(P) ? MODE_BLOCK_RS : MODE_BLOCK), kt, 8);
    }
    plan_for(P, 0, MODE_SUM, 0);
    plan_for(P, 1, MODE_SUM, 0);
    plan_for(P, 0, MODE_MAX, 0);
    plan_for(P, 1, MODE_MAX, 0);
    for (int dir = 0; dir < 2; ++dir)
        if (sum_mode(P, dir) != MODE_SUM) plan_for(P, dir, sum_mode(P, dir), 0);
    if (init_f)
        upload_rows(P, S.f.p, init_f);
    else {
        count_launch();
        k_fill<<<grid_for(n), AUX_NT, 0, s>>>(S.f.p, n, 0.0);
    }
    count_launch();
    k_state_init<<<1, 32, 0, s>>>(P.st, max_iter, tol);
    // first sweep's g = f0^{C,eps} (exact shift: no reference state yet)
    lse(P, 0, S.f.p, S.gnext.p, G_NONE);
    CK(cudaGetLastError());
}

static bool poll_done(Problem& P) {
    CK(cudaMemcpyAsync(P.st_host, P.st, sizeof(DevState), cudaMemcpyDeviceToHost, P.stream));
    CK(cudaStreamSynchronize(P.stream));
    return P.st_host->done != 0;
}

static SolveOut run_solve(Problem& P, double tol, int64_t max_iter, int64_t ell, const double* basis,
                          const double* init_f, bool trace_enabled, int64_t trace_cap_hint,
                          bool exact_marginals = false) {
    if (!(tol > 0.0)) throw InvalidArgument("solve: tol_omega must be positive");
    if (max_iter < 1) throw InvalidArgument("solve: max_iter must be >= 1");
    if (ell > 64) throw InvalidArgument("solve: ell > 64 is not supported by sknr_b200");
    const int64_t trace_cap = trace_enabled ? std::min<int64_t>(max_iter, std::max<int64_t>(trace_cap_hint, 1)) : 1;
    if (!P.solve_cache) P.solve_cache = std::make_shared<SolveState>();
    SolveState& S = *P.solve_cache;
    prepare_solve(P, S, ell, basis, init_f, max_iter, tol, trace_cap);
    cudaStream_t s = P.stream;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    // SKNR_HOST_LOOP=1: one graph per iteration, host-polled (profilers such as ncu do not
    // see kernels inside conditional-node bodies)
    static const bool host_loop = std::getenv("SKNR_HOST_LOOP") != nullptr;
    const bool polled = P.shard || host_loop;
    if (!polled) {
        // the whole solve as one graph: a WHILE node whose body is one iteration;
        // k_record clears the loop condition once the stopping test (or max_iter) hits
        CK(cudaGraphCreate(&graph, 0));
        cudaGraphConditionalHandle loop = 0;
        CK(cudaGraphConditionalHandleCreate(&loop, graph, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = loop;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        enqueue_iteration(P, S, ell, trace_enabled, trace_cap, exact_marginals, loop);
        CK(cudaStreamEndCapture(s, &body));
        make_programmatic(body);
        CK(cudaGraphInstantiate(&exec, graph, 0));
        CK(cudaGraphLaunch(exec, s));
        CK(cudaStreamSynchronize(s));
    } else if (!P.emu) {
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        enqueue_iteration(P, S, ell, trace_enabled, trace_cap, exact_marginals);
        CK(cudaStreamEndCapture(s, &graph));
        make_programmatic(graph);
        CK(cudaGraphInstantiate(&exec, graph, 0));
    }
    int64_t batch = 1;
    int64_t launched = 0;
    while (polled) {  // sharded (NCCL in the graph), emulated shards, SKNR_HOST_LOOP: host-polled batches
        for (int64_t b = 0; b < batch; ++b) {
            if (exec)
                CK(cudaGraphLaunch(exec, s));
            else  // emulated shards: the same kernels and collectives, launched eagerly
                enqueue_iteration(P, S, ell, trace_enabled, trace_cap, exact_marginals);
            ++launched;
        }
        if (poll_done(P)) break;
        if (launched >= max_iter + 2) break;
        batch = std::min<int64_t>(batch * 2, 64);
    }
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    SolveOut out;
    out.f.resize(P.n_global);
    out.g.resize(P.m);
    gather_rows(P, S.f.p, out.f.data());
    download(out.g.data(), S.g.p, P.m, s);
    CK(cudaMemcpyAsync(P.st_host, P.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    out.iterations = P.st_host->iter;
    out.converged = P.st_host->conv != 0;
    if (trace_enabled) {
        const int64_t len = std::min<int64_t>(out.iterations, trace_cap);
        out.trace.resize(len);
        CK(cudaMemcpyAsync(out.trace.data(), S.trace_raw.p, sizeof(sknr_record) * len,
                           cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    return out;
}

// Batched solve: B independent problems in one CUDA graph,
// each as its own device-side WHILE loop (conditional node) over its iteration
// body, so the loops run concurrently and each stops at its own stopping test.
// Problems may differ in size and cost kind; every body issues exactly the
// kernels of run_solve, so per-problem results are bitwise identical to solving
// the problems one by one.
struct BatchItem {
    Problem* P = nullptr;
    const double* basis = nullptr;
    const double* init_f = nullptr;
};

static std::vector<SolveOut> run_solve_batch(std::vector<BatchItem>& items, double tol, int64_t max_iter,
                                             int64_t ell, bool exact_marginals) {
    if (!(tol > 0.0)) throw InvalidArgument("solve: tol_omega must be positive");
    if (max_iter < 1) throw InvalidArgument("solve: max_iter must be >= 1");
    if (ell > 64) throw InvalidArgument("solve: ell > 64 is not supported by sknr_b200");
    const size_t B = items.size();
    std::vector<SolveState*> Sp(B);
    for (size_t b = 0; b < B; ++b) {
        Problem& P = *items[b].P;
        if (!P.solve_cache) P.solve_cache = std::make_shared<SolveState>();
        Sp[b] = P.solve_cache.get();
    }
    auto S = [&](size_t b) -> SolveState& { return *Sp[b]; };
    for (size_t b = 0; b < B; ++b) {
        prepare_solve(*items[b].P, S(b), ell, items[b].basis, items[b].init_f, max_iter, tol, 1);
        CK(cudaStreamSynchronize(items[b].P->stream));
    }
    cudaStream_t s0 = nullptr;
    CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::vector<SolveOut> out(B);
    try {
        // one graph, one independent device-side WHILE loop per problem (conditional
        // nodes without dependencies between them): each problem iterates until its own
        // stopping test, none waits for the others
        CK(cudaGraphCreate(&graph, 0));
        for (size_t b = 0; b < B; ++b) {
            Problem& P = *items[b].P;
            cudaGraphConditionalHandle loop = 0;
            CK(cudaGraphConditionalHandleCreate(&loop, graph, 1, cudaGraphCondAssignDefault));
            cudaGraphNodeParams cp = {};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = loop;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            cudaGraphNode_t node;
            CK(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
            cudaGraph_t body = cp.conditional.phGraph_out[0];
            CK(cudaStreamBeginCaptureToGraph(P.stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
            enqueue_iteration(P, S(b), ell, false, 1, exact_marginals, loop);
            CK(cudaStreamEndCapture(P.stream, &body));
            make_programmatic(body);
        }
        CK(cudaGraphInstantiate(&exec, graph, 0));
        CK(cudaGraphLaunch(exec, s0));
        CK(cudaStreamSynchronize(s0));
        for (size_t b = 0; b < B; ++b) {
            Problem& P = *items[b].P;
            out[b].f.resize(P.n_global);
            out[b].g.resize(P.m);
            download(out[b].f.data(), S(b).f.p, P.n, P.stream);
            download(out[b].g.data(), S(b).g.p, P.m, P.stream);
            CK(cudaMemcpyAsync(P.st_host, P.st, sizeof(DevState), cudaMemcpyDeviceToHost, P.stream));
        }
        for (size_t b = 0; b < B; ++b) {
            Problem& P = *items[b].P;
            CK(cudaStreamSynchronize(P.stream));
            out[b].iterations = P.st_host->iter;
            out[b].converged = P.st_host->conv != 0;
        }
    } catch (...) {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        cudaStreamDestroy(s0);
        throw;
    }
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    cudaStreamDestroy(s0);
    return out;
}
