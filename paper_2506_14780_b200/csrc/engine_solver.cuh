// engine_solver.cuh -- the SK-NR(ell) solve loop: one iteration as a captured graph body, device-side WHILE loop, batches
// Part of the libsknr_b200 translation unit: included once, in order, by engine.cu
// (shares its types, static helpers and kernels; not a standalone header).
#pragma once

// ============================================================ solve
struct SolveState {
    DBuf f, g, gnext, h, fcand, hcand, rowres, colres, am, r, Lr, V, Wv, S, delta, G;
    DBuf Sloc;  // sharded: this rank's reduce-scattered block of S (scatter_rows x ell)
    DBuf dvec, Wst, ST, dh;  // stable accept test: d = f' - f, anchor-pass weights/sums, h' - h
    DBuf trace_raw;  // sknr_record array (as doubles)
};

struct SolveOut {
    std::vector<double> f, g;
    int64_t iterations = 0;
    bool converged = false;
    std::vector<sknr_record> trace;
};

// Largest max_i |f'_i - f_i| / eps the stable accept test evaluates (expm1 stays finite).
constexpr double kStableSpan = 600.0;

// Enqueue one SK-NR(ell) iteration (solver.cpp:104-151).
// accept: 0 literal Q1 > Q0 (the reference), 1 stable dQ > 0 (ACCEPT_STABLE below).
static void enqueue_iteration(Problem& P, SolveState& S, int64_t ell, bool trace_enabled,
                              int64_t trace_cap, bool exact_marginals = false,
                              cudaGraphConditionalHandle loop = 0, int accept = 0) {
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
        sp.scatter_out = P.shard ? S.Sloc.p : nullptr;
        sp.rsum_out = fuse_r ? S.r.p : nullptr;
        sp.w_static = true;
        sp.cull = cull_nr;  // P~ columns sum to 1 at h = f^{C,eps}: no normalisation needed
        sp.guard = gn;
        plan_pass(P, sp);
        if (fuse_r) {
            count_launch();
            k_axpby<<<grid_for(n), AUX_NT, 0, s>>>(P.src.w.p, S.r.p, n, 1.0, -1.0, S.am.p);
        }
        double* G1 = S.G.p;
        double* cross = G1 + l * l;
        double* grad = cross + l * l;
        gram(P, n, l, l, S.V.p, n, S.V.p, n, S.r.p, G1, gn);
        if (P.shard) {
            // S = V^T P~ was reduce-scattered: this rank holds target rows
            // [q mb, q mb + rows) and adds its part of cross = S diag(b) S^T; one allreduce
            // sums [G1 | cross | grad] (contiguous) over the shards
            const int64_t mb = scatter_rows(P);
            const int64_t j0 = std::min<int64_t>(m, mb * P.rank), rows = std::min<int64_t>(m, j0 + mb) - j0;
            if (rows > 0)
                gram(P, rows, l, l, S.Sloc.p, mb, S.Sloc.p, mb, P.tgt.w.p + j0, cross, gn);
            else {
                count_launch();
                k_fill<<<1, AUX_NT, 0, s>>>(cross, static_cast<int64_t>(l) * l, 0.0);
            }
            gram(P, n, l, 1, S.V.p, n, S.am.p, n, nullptr, grad, gn);
            allreduce(P, G1, static_cast<size_t>(2 * l * l + l), ncclSum);
        } else {
            gram(P, m, l, l, S.S.p, m, S.S.p, m, P.tgt.w.p, cross, gn);
            gram(P, n, l, 1, S.V.p, n, S.am.p, n, nullptr, grad, gn);
        }
        count_launch();
        k_newton_solve<<<1, 256, sizeof(double) * l * l, s>>>(G1, cross, grad, l, P.inv_eps(), S.delta.p,
                                                            P.st, gn);
        // accept test. Literal (solver.cpp:45-47): Q1 = a.f' + b.f'^{C,eps} from a full
        // column LSE of the candidate, accept iff Q1 > Q0. Stable (accept = 1): the same
        // predicate as dQ = Q1 - Q0 > 0 evaluated directly -- one anchor pass at (f, h)
        // gives s_j = sum_i P~_ij, t_j = sum_i P~_ij expm1(d_i/eps) and u_j = sum_i P~_ij
        // exp(d_i/eps), d = f' - f, and h'_j - h_j = -eps log(u_j/s_j) = -eps log1p(t_j/s_j)
        // (exact algebra; k_dh picks the form that does not cancel), so dQ = a.d + b.(h' - h) rounds
        // at the size of the step instead of at ulp(Q) (oracle stable_delta_q). Steps with
        // max|d| > 600 eps take the literal path (guard bits G_LIT / G_NOLIT).
        const bool stable = accept == 1;
        const unsigned glit = stable ? (gn | G_LIT) : gn;
        if (stable) {
            const unsigned gst = gn | G_NOLIT;
            count_launch();
            const int akt = anchor_kt(P);
            k_fcand_step<<<grid_for(n), AUX_NT, 0, s>>>(S.f.p, S.V.p, n, l, S.delta.p, P.inv_eps(), S.fcand.p,
                                                        S.dvec.p, S.Wst.p, akt, P.st, gn);
            {
                RedArgs ra;
                ra.T[0] = n;
                ra.nterms = 2;
                ra.x[0] = P.src.w.p;
                ra.y[0] = S.dvec.p;
                ra.op[0] = RED_DOT;
                ra.x[1] = S.dvec.p;
                ra.op[1] = RED_MAXABS;
                ra.out = sums + 10;
                ra.part = P.gram_part.p;
                ra.counter = &P.st->counters[6];
                ra.epilogue = P.shard ? EPI_NONE : EPI_STEP;
                ra.st = P.st;
                ra.guard = gn;
                count_launch();
                k_reduce<<<reduce_blocks(n), AUX_NT, 0, s>>>(ra);
                if (P.shard) {
                    allreduce(P, sums + 10, 1, ncclSum);
                    allreduce(P, sums + 11, 1, ncclMax);
                    count_launch();
                    k_epilogue<<<1, 32, 0, s>>>(P.st, EPI_STEP, 0, sums + 10, gn);
                }
            }
            PassSpec tp;
            tp.dir = 0;
            tp.in_v = S.f.p;
            tp.in_lw = P.src.lw.p;
            tp.out_v = S.h.p;
            tp.W = S.Wst.p;
            tp.k = 3;
            tp.kt = akt;
            tp.out = S.ST.p;
            tp.guard = gst;
            plan_pass(P, tp);  // sums over the row shards
            count_launch();
            k_dh<<<grid_for(m), AUX_NT, 0, s>>>(S.ST.p, S.h.p, m, P.eps, S.dh.p, S.hcand.p, P.st, gst);
            RedArgs ra;
            ra.T[1] = m;
            ra.nterms = 1;
            ra.x[0] = P.tgt.w.p;
            ra.y[0] = S.dh.p;
            ra.op[0] = RED_DOT;
            ra.seg[0] = 1;  // replicated on every rank: same layout, no exchange
            ra.out = sums + 12;
            ra.part = P.gram_part.p;
            ra.counter = &P.st->counters[6];
            ra.epilogue = EPI_ACCEPT_DQ;
            ra.st = P.st;
            ra.guard = gst;
            count_launch();
            k_reduce<<<reduce_blocks(m), AUX_NT, 0, s>>>(ra);
        } else {
            count_launch();
            k_fcand<<<grid_for(n), AUX_NT, 0, s>>>(S.f.p, S.V.p, n, l, S.delta.p, S.fcand.p, P.st, gn);
        }
        lse(P, 0, S.fcand.p, S.hcand.p, glit);
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
            ra.guard = glit;
            count_launch();
            k_reduce<<<reduce_blocks(n + m), AUX_NT, 0, s>>>(ra);
            if (P.shard) {
                allreduce(P, sums + 6, 1, ncclSum);
                count_launch();
                k_epilogue<<<1, 32, 0, s>>>(P.st, EPI_ACCEPT, 0, sums + 6, glit);
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
                          const double* init_f, int64_t max_iter, double tol, int64_t trace_cap,
                          int accept = 0) {
    own_stream(P.stream);
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
        if (P.shard) {
            S.S.ensure(P.world * scatter_rows(P) * ell);  // rank-blocked, padded rows stay 0
            S.Sloc.ensure(scatter_rows(P) * ell);
        } else {
            S.S.ensure(m * ell);
        }
        upload_rows(P, S.V.p, basis_host, ell);
        count_launch();
        k_pack_w<<<grid_for(n * kt), AUX_NT, 0, s>>>(S.V.p, n, n, static_cast<int>(ell), kt, nullptr,
                                                     S.Wv.p);
        // pre-size the block-pass partials outside graph capture
        const bool cull_nr = cull_block_active(P, 0) && cull_active(P, 1);
        const TilePlan bp =
            plan_for(P, 0, cull_nr ? MODE_BLOCK_CULL : (block_rs_fusable(P) ? MODE_BLOCK_RS : MODE_BLOCK), kt, 8);
        P.vsl_src = nullptr;
        if (bp.i8) {  // the basis is fixed for the solve: its int8 digit tiles are made once, here
            launch_i8_vprep(S.Wv.p, kt, n, reinterpret_cast<uint8_t*>(P.vsl.p),
                            reinterpret_cast<unsigned*>(P.vexp.p), P.st, 0, s);
            P.vsl_src = S.Wv.p;
        }
        if (accept == 1) {  // stable accept test: anchor pass with W = (1, expm1(d/eps))
            const int akt = anchor_kt(P);
            S.dvec.ensure(n);
            S.Wst.ensure(n * akt);
            S.ST.ensure(3 * m);
            S.dh.ensure(m);
            plan_for(P, 0, MODE_BLOCK, akt, anchor_in_blocks(akt));
        }
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
    k_state_init<<<1, 32, 0, s>>>(P.st, max_iter, tol, kStableSpan * P.eps);
    // first sweep's g = f0^{C,eps} (exact shift: no reference state yet)
    lse(P, 0, S.f.p, S.gnext.p, G_NONE);
    CK(cudaGetLastError());
}

static bool poll_done(Problem& P) {
    CK(cudaMemcpyAsync(P.st_host, P.st, sizeof(DevState), cudaMemcpyDeviceToHost, P.stream));
    CK(cudaStreamSynchronize(P.stream));
    return P.st_host->done != 0;
}

// Device trace capacity per chunk: long solves pause the device loop when it fills, the
// host drains it and relaunches (the host copy grows with the iterations actually run,
// like the reference's push_back, never with max_iter).
constexpr int64_t kTraceChunk = 1 << 14;

// Ends a pending stream capture on unwind (an exception between Begin/EndCapture would
// otherwise leave the handle's stream in capture mode) and frees the graph objects.
struct GraphGuard {
    cudaStream_t s = nullptr;
    bool capturing = false;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    ~GraphGuard() {
        if (capturing) {
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(s, &g);
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
        }
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
    }
};

static SolveOut run_solve(Problem& P, double tol, int64_t max_iter, int64_t ell, const double* basis,
                          const double* init_f, bool trace_enabled, int64_t trace_cap_hint,
                          bool exact_marginals = false, int accept = 0) {
    if (!(tol > 0.0)) throw InvalidArgument("solve: tol_omega must be positive");
    if (max_iter < 1) throw InvalidArgument("solve: max_iter must be >= 1");
    if (ell > 64) throw InvalidArgument("solve: ell > 64 is not supported by sknr_b200");
    (void)trace_cap_hint;
    const int64_t trace_cap = trace_enabled ? std::min<int64_t>(max_iter, kTraceChunk) : 1;
    if (!P.solve_cache) P.solve_cache = std::make_shared<SolveState>();
    SolveState& S = *P.solve_cache;
    prepare_solve(P, S, ell, basis, init_f, max_iter, tol, trace_cap, accept);
    cudaStream_t s = P.stream;
    GraphGuard gg;
    gg.s = s;
    SolveOut out;
    // copies the device trace records of iterations (trace_base, iter] to the host
    auto drain = [&]() {
        if (!trace_enabled) return;
        CK(cudaMemcpyAsync(P.st_host, P.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const int64_t len = std::min<int64_t>(P.st_host->iter - P.st_host->trace_base, trace_cap);
        if (len > 0) {
            const size_t old = out.trace.size();
            out.trace.resize(old + static_cast<size_t>(len));
            CK(cudaMemcpyAsync(out.trace.data() + old, S.trace_raw.p, sizeof(sknr_record) * len,
                               cudaMemcpyDeviceToHost, s));
        }
        count_launch();
        k_trace_rebase<<<1, 32, 0, s>>>(P.st);
        CK(cudaStreamSynchronize(s));
    };
    // SKNR_HOST_LOOP=1: one graph per iteration, host-polled (profilers such as ncu do not
    // see kernels inside conditional-node bodies)
    static const bool host_loop = std::getenv("SKNR_HOST_LOOP") != nullptr;
    const bool polled = P.shard || host_loop;
    if (!polled) {
        // the whole solve as one graph: a WHILE node whose body is one iteration;
        // k_record clears the loop condition once the stopping test (or max_iter) hits,
        // or pauses it when the device trace chunk is full
        CK(cudaGraphCreate(&gg.graph, 0));
        cudaGraphConditionalHandle loop = 0;
        CK(cudaGraphConditionalHandleCreate(&loop, gg.graph, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = loop;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, gg.graph, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        gg.capturing = true;
        enqueue_iteration(P, S, ell, trace_enabled, trace_cap, exact_marginals, loop, accept);
        gg.capturing = false;
        CK(cudaStreamEndCapture(s, &body));
        make_programmatic(body);
        CK(cudaGraphInstantiate(&gg.exec, gg.graph, 0));
        while (true) {
            CK(cudaGraphLaunch(gg.exec, s));
            if (!trace_enabled) {
                CK(cudaStreamSynchronize(s));
                break;
            }
            drain();  // pauses only to drain a full trace chunk
            if (P.st_host->done) break;
        }
    } else if (!P.emu) {
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        gg.capturing = true;
        enqueue_iteration(P, S, ell, trace_enabled, trace_cap, exact_marginals, 0, accept);
        gg.capturing = false;
        CK(cudaStreamEndCapture(s, &gg.graph));
        make_programmatic(gg.graph);
        CK(cudaGraphInstantiate(&gg.exec, gg.graph, 0));
    }
    int64_t batch = 1;
    int64_t launched = 0;
    double gap_prev = 0.0;
    int64_t iter_prev = 0;
    while (polled) {  // sharded (NCCL in the graph), emulated shards, SKNR_HOST_LOOP: host-polled batches
        // batches never outrun the trace chunk: they are drained at every poll
        for (int64_t b = 0; b < batch; ++b) {
            if (gg.exec)
                CK(cudaGraphLaunch(gg.exec, s));
            else  // emulated shards: the same kernels and collectives, launched eagerly
                enqueue_iteration(P, S, ell, trace_enabled, trace_cap, exact_marginals, 0, accept);
            ++launched;
        }
        const bool done = poll_done(P);
        const double gap = P.st_host->gap_l2;
        const int64_t it = P.st_host->iter;
        drain();
        if (done) break;
        if (launched >= max_iter + 2) break;
        // Launches past the stop are guard-skipped no-ops, but their collectives still run:
        // size the next batch from the observed contraction of the marginal error, so the
        // batch that crosses tol overshoots by a few iterations instead of up to 63.
        int64_t next = std::min<int64_t>(batch * 2, 64);
        if (gap_prev > 0.0 && gap > 0.0 && gap < gap_prev && it > iter_prev) {
            const double rate = std::log(gap / gap_prev) / static_cast<double>(it - iter_prev);  // < 0
            const double remaining = std::log(tol / gap) / rate;
            if (std::isfinite(remaining))
                next = std::min<int64_t>(next, std::max<int64_t>(1, static_cast<int64_t>(remaining) + 1));
        }
        gap_prev = gap;
        iter_prev = it;
        batch = std::min<int64_t>(next, std::max<int64_t>(trace_cap, 1));
    }
    out.f.resize(P.n_global);
    out.g.resize(P.m);
    gather_rows(P, S.f.p, out.f.data());
    download(out.g.data(), S.g.p, P.m, s);
    CK(cudaMemcpyAsync(P.st_host, P.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    out.iterations = P.st_host->iter;
    out.converged = P.st_host->conv != 0;
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
                                             int64_t ell, bool exact_marginals, int accept = 0) {
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
        prepare_solve(*items[b].P, S(b), ell, items[b].basis, items[b].init_f, max_iter, tol, 1, accept);
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
            enqueue_iteration(P, S(b), ell, false, 1, exact_marginals, loop, accept);
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
