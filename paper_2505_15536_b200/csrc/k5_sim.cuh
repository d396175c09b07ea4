// k5_sim.cuh - K5: 1F1B discrete-event simulation, one thread per timing / candidate.
#pragma once
#include "k2_eval.cuh"

// ----------------------------------------------------------------------------
// K5: 1F1B discrete-event simulation, one thread per timing
// (PipelineEngine.run, Policy.ONE_F_ONE_B, constant trace, no adapter;
//  src/engine.py:154-431, src/nettrace.py:57-76).
//
// Bounded state instead of the reference's dicts and heap:
//  * every chunk is min(m, B - i*m) for the i-th chunk of an iteration, so
//    FIFO contents (W queue, link queues) are index ranges, not lists;
//  * a stage is never more than one iteration ahead of its neighbours'
//    credits, so per stage two iteration slots (tagged) hold the pools;
//  * at most one op per stage and one transfer per link direction are in
//    flight: <= 3S-2 pending events, popped by a linear (time, seq) scan.
// ----------------------------------------------------------------------------
struct SimPool {
    long long fwd_avail, fwd_taken, fwd_done, bwd_avail, bwd_taken, bwd_done, w_done;
    int it_tag;         // iteration held by this slot
    int wq_head, wq_tail;   // W queue = backward chunk indices [head, tail)
    int flags;          // bit0 sync_done, bit1 opt_done
};

struct SimEv {
    double t;
    unsigned long long seq;
    int code;           // kind<<31 | s<<20 | op<<16 | it
    int size;
};

__device__ __forceinline__ SimPool& sim_pool(SimPool* P, int s, int it) {
    SimPool& p = P[s * 2 + (it & 1)];
    if (p.it_tag != it) {
        p.fwd_avail = p.fwd_taken = p.fwd_done = p.bwd_avail = p.bwd_taken = p.bwd_done = 0;
        p.w_done = 0;
        p.wq_head = p.wq_tail = 0;
        p.flags = 0;
        p.it_tag = it;
    }
    return p;
}

// NetworkTrace.multiplier (src/nettrace.py:36-43): last breakpoint <= t
__device__ __forceinline__ double trace_mult(const gp_trace* tr, int link, double t) {
    const int np = (int)tr->n_points[link];
    double m = 1.0;
    for (int i = 0; i < np; ++i)
        if (tr->t[link][i] <= t) m = tr->mult[link][i];
    return m;
}

// transfer_end_time (src/nettrace.py:57-76)
__device__ double transfer_end(double start, double bytes, double base_bw, double latency,
                               const gp_trace* tr, int link) {
    double t = start, remaining = bytes;
    if (tr) {
        const int np = (int)tr->n_points[link];
        for (int i = 0; i < np; ++i) {
            const double bp_t = tr->t[link][i];
            if (!(bp_t > start)) continue;
            const double bw = base_bw * trace_mult(tr, link, t);
            const double span = bp_t - t;
            if (remaining <= bw * span) return (t + remaining / bw) + latency;
            remaining -= bw * span;
            t = bp_t;
        }
    }
    const double bw = base_bw * (tr ? trace_mult(tr, link, t) : 1.0);
    return (t + remaining / bw) + latency;
}

// _ready_op (src/engine.py:157-215): candidates F, B, W, SYNC, OPT in this
// order; the lowest priority wins, the earliest on ties.  `size` is the
// stage's current micro-batch (the adapter's, or m), `m` the configured one
// that sets the warm-up quota.  Returns the op kind (-1: none) and its size.
__device__ __forceinline__ int ready_op(int policy, int S, int s, long long B, long long m,
                                        long long size, long long fwd_avail, long long fwd_taken,
                                        long long fwd_done, long long bwd_avail, long long bwd_taken,
                                        long long bwd_done, long long w_done, bool wq_any,
                                        long long wq_head_size, bool sync_done, bool opt_done,
                                        long long* out_size) {
    const bool zbc = policy == GP_POLICY_ZB_COMPACT, zbo = policy == GP_POLICY_ZB_ORIGINAL;
    const bool gpipe = policy == GP_POLICY_GPIPE;
    int best_pr = 100, best_k = -1;
    long long best_sz = 0;
    const long long fwd_rem = B - fwd_taken;
    if (fwd_rem > 0) {
        const long long chunk = size < fwd_rem ? size : fwd_rem;
        if (fwd_avail - fwd_taken >= chunk) {
            int pr = -1;
            if (zbc || gpipe) {
                pr = zbc ? 0 : 1;
            } else {
                const long long quota = (long long)(S - s) * m;
                if (fwd_taken < quota) pr = zbo ? 0 : 1;
                else if (fwd_taken + chunk <= quota + bwd_done) pr = zbo ? 3 : 2;
            }
            if (pr >= 0) { best_pr = pr; best_k = 0; best_sz = chunk; }
        }
    }
    const long long bwd_rem = B - bwd_taken;
    if (bwd_rem > 0 && (!gpipe || fwd_done == B)) {
        const long long chunk = size < bwd_rem ? size : bwd_rem;
        long long av = (bwd_avail < fwd_done ? bwd_avail : fwd_done) - bwd_taken;
        if (s == S - 1) av = fwd_done - bwd_taken;
        const int pr = (zbc || zbo) ? 1 : 2;
        if (av >= chunk && pr < best_pr) { best_pr = pr; best_k = 1; best_sz = chunk; }
    }
    if (wq_any) {
        const int pr = (gpipe || policy == GP_POLICY_1F1B) ? 0 : 2;
        if (pr < best_pr) { best_pr = pr; best_k = 2; best_sz = wq_head_size; }
    }
    if (w_done == B && !wq_any && !sync_done && 8 < best_pr) { best_pr = 8; best_k = 3; best_sz = 0; }
    if (sync_done && !opt_done && 9 < best_pr) { best_pr = 9; best_k = 4; best_sz = 0; }
    *out_size = best_sz;
    return best_k;
}

__device__ int sim_dev(const gp_timing& T, int policy, int iterations, const gp_trace* trace,
                       double* makespan) {
    const int S = (int)T.n_stages;
    if (S < 1 || S > GP_MAX_STAGES || iterations < 1 || T.microbatch <= 0) return GP_ERR_TIMING;
    const long long B = T.batch, m = T.microbatch;
    const long long nchunk = (B + m - 1) / m;  // chunks per iteration
    SimPool P[2 * GP_MAX_STAGES];
    for (int i = 0; i < 2 * S; ++i) P[i].it_tag = -1;
    int cur[GP_MAX_STAGES];
    bool busy[GP_MAX_STAGES];
    // links: 2 per boundary (fwd, bwd): transfers enqueued / started / busy
    long long l_enq[2 * GP_MAX_STAGES], l_start[2 * GP_MAX_STAGES];
    bool l_busy[2 * GP_MAX_STAGES];
    SimEv ev[3 * GP_MAX_STAGES];
    int nev = 0;
    unsigned long long seq = 0;
    for (int s = 0; s < S; ++s) {
        cur[s] = 0;
        busy[s] = false;
        SimPool& p = sim_pool(P, s, 0);
        if (s == 0) p.fwd_avail = B;
    }
    for (int l = 0; l < 2 * (S - 1); ++l) { l_enq[l] = 0; l_start[l] = 0; l_busy[l] = false; }
    auto chunk_size = [&](long long j) -> long long {  // j-th chunk of an iteration
        long long r = B - (j % nchunk) * m;
        return r < m ? r : m;
    };
    auto try_start = [&](double tnow, int bnd, int dir) {
        const int l = 2 * bnd + dir;
        if (l_busy[l] || l_start[l] >= l_enq[l]) return;
        const long long j = l_start[l]++;
        l_busy[l] = true;
        const long long sz = chunk_size(j);
        const int it = (int)(j / nchunk);
        const double per = dir == 0 ? T.act[bnd] : T.grad[bnd];
        SimEv& e = ev[nev++];
        e.t = transfer_end(tnow, per * (double)sz, T.bw[bnd], T.lat[bnd], trace, bnd);
        e.seq = seq++;
        e.code = (int)(1u << 31) | (bnd << 20) | (dir << 16) | it;
        e.size = (int)sz;
    };
    double now = 0.0;
    for (;;) {
        // dispatch(now) (src/engine.py:335-341)
        bool progress = true;
        while (progress) {
            progress = false;
            for (int s = 0; s < S; ++s) {
                if (busy[s]) continue;
                const int it = cur[s];
                if (it >= iterations) continue;
                SimPool& p = sim_pool(P, s, it);
                long long best_sz;
                const int best_k = ready_op(policy, S, s, B, m, m, p.fwd_avail, p.fwd_taken,
                                            p.fwd_done, p.bwd_avail, p.bwd_taken, p.bwd_done,
                                            p.w_done, p.wq_head < p.wq_tail,
                                            p.wq_head < p.wq_tail ? chunk_size(p.wq_head) : 0,
                                            (p.flags & 1) != 0, (p.flags & 2) != 0, &best_sz);
                if (best_k < 0) continue;
                double dur;
                switch (best_k) {
                    case 0: dur = T.fwd[s] * (double)best_sz; p.fwd_taken += best_sz; break;
                    case 1: dur = T.bwd[s] * (double)best_sz; p.bwd_taken += best_sz; break;
                    case 2: dur = T.wgt[s] * (double)best_sz; p.wq_head++; break;
                    case 3: dur = T.sync[s]; break;
                    default: dur = T.opt[s]; break;
                }
                busy[s] = true;
                SimEv& e = ev[nev++];
                e.t = now + dur;
                e.seq = seq++;
                e.code = (s << 20) | (best_k << 16) | it;
                e.size = (int)best_sz;
                progress = true;
            }
        }
        if (nev == 0) break;
        // pop the (time, seq) minimum
        int bi = 0;
        for (int i = 1; i < nev; ++i)
            if (ev[i].t < ev[bi].t || (ev[i].t == ev[bi].t && ev[i].seq < ev[bi].seq)) bi = i;
        const SimEv e = ev[bi];
        ev[bi] = ev[--nev];
        now = e.t;
        const int it = e.code & 0xffff, sb = (e.code >> 20) & 0x7ff, op = (e.code >> 16) & 0xf;
        if (e.code >= 0) {
            // finish_op (src/engine.py:343-378)
            const int s2 = sb;
            SimPool& p = sim_pool(P, s2, it);
            busy[s2] = false;
            if (op == 0) {
                p.fwd_done += e.size;
                if (s2 < S - 1) { l_enq[2 * s2]++; try_start(now, s2, 0); }
            } else if (op == 1) {
                p.bwd_done += e.size;
                p.wq_tail++;
                if (s2 > 0) { l_enq[2 * (s2 - 1) + 1]++; try_start(now, s2 - 1, 1); }
            } else if (op == 2) {
                p.w_done += e.size;
            } else if (op == 3) {
                p.flags |= 1;
            } else {
                p.flags |= 2;
                cur[s2] = it + 1;
                if (it + 1 < iterations) {
                    SimPool& q = sim_pool(P, s2, it + 1);
                    if (s2 == 0) q.fwd_avail = B;
                }
            }
        } else {
            // finish_transfer (src/engine.py:380-396)
            l_busy[2 * sb + op] = false;
            if (op == 0) sim_pool(P, sb + 1, it).fwd_avail += e.size;
            else sim_pool(P, sb, it).bwd_avail += e.size;
            try_start(now, sb, op);
        }
    }
    *makespan = now;
    for (int s = 0; s < S; ++s)
        if (cur[s] < iterations) return GP_ERR_SCHEDULING;
    return GP_OK;
}

// ----------------------------------------------------------------------------
// Register-resident specialisation of sim_dev for S <= SMAX stages, one
// iteration and a constant trace (the common case: ranking candidate plans
// by their simulated 1F1B makespan).  The event list becomes fixed slots -
// one pending op per stage, one pending transfer per link direction - so the
// (time, seq) pop is an unrolled comparison over 3*SMAX-2 slots, every loop
// over stages is unrolled with compile-time indices, and the state (counters
// as 32-bit ints, event times) lives in registers instead of a 5 KB local
// frame.  Event order, dispatch order and every floating-point operation are
// sim_dev's (src/engine.py:230-406), so makespans are bit-identical.
// ----------------------------------------------------------------------------
template <int SMAX>
__device__ int sim_regs(const gp_timing& T, int policy, double* makespan) {
    const int S = (int)T.n_stages;
    const long long B = T.batch, m = T.microbatch;
    const long long nchunk = (B + m - 1) / m;
    constexpr int L = 2 * (SMAX - 1) > 0 ? 2 * (SMAX - 1) : 1;
    long long fa[SMAX], ft[SMAX], fd[SMAX], ba[SMAX], bt[SMAX], bd[SMAX], wd[SMAX];
    int wh[SMAX], wtl[SMAX];
    bool syncd[SMAX], optd[SMAX], busy[SMAX];
    double ot[SMAX];
    unsigned oseq[SMAX];
    int ok[SMAX];
    long long osz[SMAX];
    long long lenq[L], lst[L], xsz[L];
    bool lbusy[L];
    double xt[L];
    unsigned xseq[L];
    double fwd[SMAX], bwd[SMAX], wgt[SMAX], syn[SMAX], opt[SMAX];
#pragma unroll
    for (int s = 0; s < SMAX; ++s) {
        fa[s] = ft[s] = fd[s] = ba[s] = bt[s] = bd[s] = wd[s] = 0;
        wh[s] = wtl[s] = 0;
        syncd[s] = optd[s] = false;
        busy[s] = s >= S;  // absent stages never dispatch
        ot[s] = INFINITY;
        oseq[s] = 0u;
        ok[s] = 0;
        osz[s] = 0;
        fwd[s] = T.fwd[s]; bwd[s] = T.bwd[s]; wgt[s] = T.wgt[s]; syn[s] = T.sync[s]; opt[s] = T.opt[s];
    }
    fa[0] = B;
#pragma unroll
    for (int l = 0; l < L; ++l) { lenq[l] = lst[l] = xsz[l] = 0; lbusy[l] = false; xt[l] = INFINITY; xseq[l] = 0u; }
    unsigned seq = 0u;
    auto chunk_size = [&](long long j) -> long long {
        long long r = B - (j % nchunk) * m;
        return r < m ? r : m;
    };
    // try_start_link (src/engine.py:271-289), boundary bnd and direction dir
    // compile-time after unrolling
    auto try_start = [&](double tnow, int bnd, int dir) {
        const int l = 2 * bnd + dir;
        if (lbusy[l] || lst[l] >= lenq[l]) return;
        const long long j = lst[l]++;
        lbusy[l] = true;
        const long long sz = chunk_size(j);
        const double per = dir == 0 ? T.act[bnd] : T.grad[bnd];
        const double bytes = per * (double)sz;
        const double bw = T.bw[bnd] * 1.0;
        xt[l] = (tnow + bytes / bw) + T.lat[bnd];
        xseq[l] = seq++;
        xsz[l] = sz;
    };
    double now = 0.0;
    for (;;) {
        bool progress = true;
        while (progress) {
            progress = false;
#pragma unroll
            for (int s = 0; s < SMAX; ++s) {
                if (busy[s] || optd[s]) continue;
                const bool wq_any = wh[s] < wtl[s];
                long long best_sz;
                const int best_k = ready_op(policy, S, s, B, m, m, fa[s], ft[s], fd[s], ba[s], bt[s],
                                            bd[s], wd[s], wq_any, wq_any ? chunk_size(wh[s]) : 0,
                                            syncd[s], optd[s], &best_sz);
                if (best_k < 0) continue;
                double dur;
                switch (best_k) {
                    case 0: dur = fwd[s] * (double)best_sz; ft[s] += best_sz; break;
                    case 1: dur = bwd[s] * (double)best_sz; bt[s] += best_sz; break;
                    case 2: dur = wgt[s] * (double)best_sz; wh[s]++; break;
                    case 3: dur = syn[s]; break;
                    default: dur = opt[s]; break;
                }
                busy[s] = true;
                ot[s] = now + dur;
                oseq[s] = seq++;
                ok[s] = best_k;
                osz[s] = best_sz;
                progress = true;
            }
        }
        // pop the (time, seq) minimum over the pending slots
        double bt_ = INFINITY;
        unsigned bs_ = ~0u;
        int slot = -1;
#pragma unroll
        for (int s = 0; s < SMAX; ++s)
            if (s < S && busy[s] && !optd[s] && (ot[s] < bt_ || (ot[s] == bt_ && oseq[s] < bs_))) {
                bt_ = ot[s]; bs_ = oseq[s]; slot = s;
            }
#pragma unroll
        for (int l = 0; l < L; ++l)
            if (lbusy[l] && (xt[l] < bt_ || (xt[l] == bt_ && xseq[l] < bs_))) {
                bt_ = xt[l]; bs_ = xseq[l]; slot = SMAX + l;
            }
        if (slot < 0) break;
        now = bt_;
#pragma unroll
        for (int s = 0; s < SMAX; ++s) {
            if (slot != s) continue;
            // finish_op (src/engine.py:343-378)
            busy[s] = false;
            const long long sz = osz[s];
            switch (ok[s]) {
                case 0:
                    fd[s] += sz;
                    if (s < SMAX - 1 && s < S - 1) { lenq[2 * s]++; try_start(now, s, 0); }
                    break;
                case 1:
                    bd[s] += sz;
                    wtl[s]++;
                    if (s > 0) { lenq[2 * (s - 1) + 1]++; try_start(now, s - 1, 1); }
                    break;
                case 2: wd[s] += sz; break;
                case 3: syncd[s] = true; break;
                default: optd[s] = true; busy[s] = true; break;  // iteration done: never dispatch
            }
        }
#pragma unroll
        for (int l = 0; l < L; ++l) {
            if (slot != SMAX + l) continue;
            // finish_transfer (src/engine.py:380-396)
            lbusy[l] = false;
            const int bnd = l / 2, dir = l % 2;
            if (dir == 0) fa[bnd + 1] += xsz[l];
            else ba[bnd] += xsz[l];
            try_start(now, bnd, dir);
        }
    }
    *makespan = now;
#pragma unroll
    for (int s = 0; s < SMAX; ++s)
        if (s < S && !optd[s]) return GP_ERR_SCHEDULING;
    return GP_OK;
}

// sim_dev or, when it applies, its register-resident specialisation
__device__ __forceinline__ int sim_any(const gp_timing& T, int policy, int iterations,
                                       const gp_trace* trace, double* makespan) {
    const int S = (int)T.n_stages;
#if !defined(K5_NO_REGS)
    if (iterations == 1 && !trace && S >= 1 && S <= 4 && T.microbatch > 0 && T.batch > 0)
        return sim_regs<4>(T, policy, makespan);
#endif
    return sim_dev(T, policy, iterations, trace, makespan);
}

// The PlanTiming of build_plan_timing (src/timing.py:176-231) for one
// explicit candidate, assembled from the stage / boundary tables; returns the
// _evaluate status (GP_ERR_NO_FEASIBLE for a memory-infeasible plan unless
// `any_memory`: build_plan_timing itself does not check memory).
__device__ int cand_timing(const DevInst& I, int k, const uint8_t* __restrict__ order,
                           const uint8_t* __restrict__ counts, int b, double opt_seconds,
                           bool any_memory, gp_timing& T) {
    uint8_t o[GP_MAX_STAGES];
    int p[GP_MAX_STAGES + 1];
    p[0] = 0;
    int st = GP_OK;
    unsigned seen = 0;
    for (int s = 0; s < k; ++s) {
        o[s] = order[s];
        int c = counts[s];
        if (o[s] >= I.F || (seen >> o[s]) & 1u || c == 0) st = GP_ERR_INPUT;
        seen |= 1u << (o[s] & 31);
        p[s + 1] = p[s] + c;
    }
    if (b >= I.nb * I.nm || p[k] > I.n) st = GP_ERR_INPUT;
    const int mi = b % I.nm;
    if (st == GP_OK) {
        long long M = I.batch[b / I.nm] / I.micro[mi];
        EvalOut r = eval_tables(I, k, o, p, mi, M);  // feasibility + errors, as _evaluate
        st = r.status;
        if (st == GP_OK && isinf(r.cost) && !any_memory) st = GP_ERR_NO_FEASIBLE;  // memory-infeasible
    }
    if (st != GP_OK) return st;
    const size_t N2 = (size_t)(I.n + 1) * (I.n + 1);
    T.n_stages = (uint32_t)k;
    T.pad = 0;
    T.batch = I.batch[b / I.nm];
    T.microbatch = I.micro[mi];
    for (int s = 0; s < GP_MAX_STAGES; ++s) {
        T.fwd[s] = T.bwd[s] = T.wgt[s] = T.sync[s] = T.opt[s] = 0.0;
        T.lat[s] = T.bw[s] = T.act[s] = T.grad[s] = 0.0;
    }
    for (int s = 0; s < k; ++s) {
        double4 v = I.fbws[(size_t)o[s] * N2 + tri_idx(I.n, p[s], p[s + 1])];
        T.fwd[s] = v.x; T.bwd[s] = v.y; T.wgt[s] = v.z; T.sync[s] = v.w; T.opt[s] = opt_seconds;
        if (s + 1 < k) {
            int g = I.gw[o[s] * I.F + o[s + 1]];
            T.lat[s] = I.lat[g];
            T.bw[s] = I.bw[g];
            T.act[s] = T.grad[s] = I.act[p[s + 1] - 1];
        }
    }
    return GP_OK;
}

// Candidates grouped by their (b, m) index before simulating: the event
// count of a 1F1B run grows with the micro-batch count M = b / m, so a warp
// of equal-M candidates walks its event loops in lock step (counting sort:
// histogram, exclusive scan, scatter of candidate indices).
__global__ void k5_bm_hist(long long n, const uint8_t* __restrict__ bm, int nbm, uint32_t* hist) {
    __shared__ uint32_t h[257];
    for (int j = threadIdx.x; j <= nbm; j += blockDim.x) h[j] = 0;
    __syncthreads();
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int b = bm[i] < nbm ? bm[i] : nbm;
        atomicAdd(&h[b], 1u);
    }
    __syncthreads();
    for (int j = threadIdx.x; j <= nbm; j += blockDim.x)
        if (h[j]) atomicAdd(&hist[j], h[j]);
}
__global__ void k5_bm_scan(int nbm, uint32_t* hist) {  // one thread: <= 257 buckets
    uint32_t acc = 0;
    for (int j = 0; j <= nbm; ++j) { const uint32_t v = hist[j]; hist[j] = acc; acc += v; }
}
__global__ void k5_bm_scatter(long long n, const uint8_t* __restrict__ bm, int nbm, uint32_t* offs,
                              uint32_t* __restrict__ perm) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int b = bm[i] < nbm ? bm[i] : nbm;
    perm[atomicAdd(&offs[b], 1u)] = (uint32_t)i;
}

// Timings grouped by (stage count, micro-batch count) before simulating
// (the event count grows with both): key = (S - 1) * 256 + min(M, 255).
#define K5_NKEYS (GP_MAX_STAGES * 256)
__device__ __forceinline__ int k5_tkey(const gp_timing& T) {
    const long long mb = T.microbatch > 0 ? T.microbatch : 1;
    long long M = T.batch > 0 ? (T.batch + mb - 1) / mb : 0;
    if (M > 255) M = 255;
    const int S = T.n_stages >= 1 && T.n_stages <= GP_MAX_STAGES ? (int)T.n_stages : 1;
    return (S - 1) * 256 + (int)M;
}
__global__ void k5_key_hist(long long n, const gp_timing* __restrict__ T, uint32_t* hist) {
    __shared__ uint32_t h[K5_NKEYS];
    for (int j = threadIdx.x; j < K5_NKEYS; j += blockDim.x) h[j] = 0;
    __syncthreads();
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        atomicAdd(&h[k5_tkey(T[i])], 1u);
    __syncthreads();
    for (int j = threadIdx.x; j < K5_NKEYS; j += blockDim.x)
        if (h[j]) atomicAdd(&hist[j], h[j]);
}
__global__ void k5_key_scan(uint32_t* hist) {  // one block of 256 threads, 8 keys each
    __shared__ uint32_t part[256];
    const int t = threadIdx.x;
    uint32_t v[K5_NKEYS / 256], acc = 0;
#pragma unroll
    for (int j = 0; j < K5_NKEYS / 256; ++j) { v[j] = hist[t * (K5_NKEYS / 256) + j]; acc += v[j]; }
    part[t] = acc;
    __syncthreads();
    if (t == 0) { uint32_t run = 0; for (int j = 0; j < 256; ++j) { const uint32_t x = part[j]; part[j] = run; run += x; } }
    __syncthreads();
    uint32_t run = part[t];
#pragma unroll
    for (int j = 0; j < K5_NKEYS / 256; ++j) { hist[t * (K5_NKEYS / 256) + j] = run; run += v[j]; }
}
__global__ void k5_key_scatter(long long n, const gp_timing* __restrict__ T, uint32_t* offs,
                               uint32_t* __restrict__ perm) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    perm[atomicAdd(&offs[k5_tkey(T[i])], 1u)] = (uint32_t)i;
}

// 1F1B makespan of explicit candidates (thread t simulates candidate
// perm[t], or t without a permutation).
__global__ void k5_sim_candidates(DevInst I, int k, long long ncand, const uint8_t* __restrict__ order,
                                  const uint8_t* __restrict__ counts, const uint8_t* __restrict__ bm,
                                  int iterations, double opt_seconds, double* __restrict__ makespan,
                                  uint8_t* __restrict__ status, const uint32_t* __restrict__ perm) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ncand) return;
    if (perm) i = perm[i];
    gp_timing T;
    int st = cand_timing(I, k, order + i * k, counts + i * k, bm[i], opt_seconds, false, T);
    if (st != GP_OK) { makespan[i] = NAN; status[i] = (uint8_t)st; return; }
    double ms = NAN;
    st = sim_any(T, GP_POLICY_1F1B, iterations, nullptr, &ms);
    makespan[i] = ms;
    status[i] = (uint8_t)st;
}

// PlanTiming records of explicit candidates (for the full simulator).
__global__ void k5_plan_timing(DevInst I, int k, long long ncand, const uint8_t* __restrict__ order,
                               const uint8_t* __restrict__ counts, const uint8_t* __restrict__ bm,
                               double opt_seconds, gp_timing* __restrict__ out,
                               uint8_t* __restrict__ status) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ncand) return;
    gp_timing T;
    int st = cand_timing(I, k, order + i * k, counts + i * k, bm[i], opt_seconds, true, T);
    if (st == GP_OK) out[i] = T;
    status[i] = (uint8_t)st;
}

__global__ void k5_sim_1f1b(const gp_timing* __restrict__ T, long long n, int policy, int iterations,
                            const gp_trace* __restrict__ traces, const uint32_t* __restrict__ tidx,
                            double* __restrict__ makespan, uint8_t* __restrict__ status,
                            const uint32_t* __restrict__ perm = nullptr) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (perm) i = perm[i];
    double ms = NAN;
    const gp_trace* tr = traces ? traces + (tidx ? tidx[i] : 0u) : nullptr;
    int st = sim_any(T[i], policy, iterations, tr, &ms);
    makespan[i] = ms;
    status[i] = (uint8_t)st;
}


// ----------------------------------------------------------------------------
// K5 full: PipelineEngine.run with every SimConfig option
// (src/engine.py:230-431): any policy and trace, the DynamicBatchAdapter
// hooks (src/adapter.py:133-224) and asynchronous iterations (:297-314),
// producing the SimReport ingredients (src/simulator.py:84-113).
//
// Under the adapter chunk sizes are data-dependent, so the W queues and the
// link FIFOs hold explicit sizes in per-timing scratch (global memory,
// interleaved by timing so neighbouring threads' same-index entries share
// sectors).  Pools: four tagged iteration slots per stage (asynchronous
// iterations keep at most three iterations of a stage live: a stage's
// iteration it+2 forwards need its optimizer step of it, which needs every
// stage's backward of it).  A slot or queue overflow is reported, never
// silently overwritten.
// ----------------------------------------------------------------------------
#define SIMF_SLOTS 4
#define AD_WINDOW 20

struct SimFPool {
    long long fwd_avail, fwd_taken, fwd_done, bwd_avail, bwd_taken, bwd_done, w_done;
    int it_tag, wq_head, wq_tail;
    int flags;          // bit0 sync_done, bit1 opt_done, bit2 activated, bit3 first_bwd_done
    int f_ids, b_ids;   // fwd_next_id / bwd_next_id (ops of a stage never overlap)
};

struct SimFEv {
    double t, t0;       // t0: start (op duration / transfer latency samples)
    unsigned long long seq;
    int code;           // kind<<31 | s<<20 | op<<16
    int it, mb;         // iteration, micro-batch id (-1: None)
    long long size;
};

// MonitorWindow (src/adapter.py:37-58): ring of the last 20 per-sample
// latencies (oldest at head), EMA baseline frozen while reduced.
struct AdWindow {
    double samples[AD_WINDOW];
    double baseline;
    long long count, since;
    int head, len, degraded, exists;
};

struct SimScratch {
    uint32_t* wq;               // [S*SLOTS*wcap][n]   W queue sizes
    unsigned long long* lq;     // [2*(S-1)*lcap][n]   link FIFOs: it<<32 | size
    SimFPool* pools;            // [n][smax*SLOTS]     iteration pools
    AdWindow* win;              // [n][2*(smax-1)]     adapter monitor windows
    long long n;                // timings in this launch (interleave stride)
    int wcap, lcap, smax;
};

__device__ __forceinline__ long long ad_halve(long long v) { return v / 2 > 1 ? v / 2 : 1; }

// Link FIFO entries pack iteration (16 bits), micro-batch id and size (24
// bits each); the host bounds batch < 2^24 and iterations < 2^16.
__device__ int sim_full(const gp_timing& T, int policy, int iterations, const gp_trace* trace,
                        const gp_sim_options& opt, SimScratch sc, long long tid,
                        gp_sim_report* rep, double* iter_ends, gp_op* ops_out, long long op_cap,
                        gp_transfer* xf_out, long long xf_cap, gp_action* act_out,
                        long long act_cap) {
    const int S = (int)T.n_stages;
    if (S < 1 || S > GP_MAX_STAGES || iterations < 1 || T.microbatch <= 0) return GP_ERR_TIMING;
    const long long B = T.batch, m = T.microbatch;
    if (B + 1 > sc.wcap || 2 * B + 2 > sc.lcap) return GP_ERR_INPUT;
    const bool adapter = opt.adapter != 0, async_it = opt.async_iterations != 0;
    if (S > sc.smax) return GP_ERR_INPUT;
    SimFPool* P = sc.pools + tid * (long long)(sc.smax * SIMF_SLOTS);
    for (int i = 0; i < SIMF_SLOTS * S; ++i) P[i].it_tag = -1;
    bool overflow = false;
    auto pool = [&](int s, int it) -> SimFPool& {
        SimFPool& p = P[s * SIMF_SLOTS + (it & (SIMF_SLOTS - 1))];
        if (p.it_tag != it) {
            if (p.it_tag >= 0 && !(p.flags & 2)) overflow = true;  // live iteration evicted
            p.fwd_avail = p.fwd_taken = p.fwd_done = p.bwd_avail = p.bwd_taken = p.bwd_done = 0;
            p.w_done = 0;
            p.wq_head = p.wq_tail = 0;
            p.flags = 0;
            p.f_ids = p.b_ids = 0;
            p.it_tag = it;
        }
        return p;
    };
    auto wq_at = [&](int s, int it, int j) -> uint32_t& {
        const long long q = (long long)(s * SIMF_SLOTS + (it & (SIMF_SLOTS - 1))) * sc.wcap + j;
        return sc.wq[q * sc.n + tid];
    };
    auto lq_at = [&](int l, long long j) -> unsigned long long& {
        const long long q = (long long)l * sc.lcap + (j % sc.lcap);
        return sc.lq[q * sc.n + tid];
    };
    // per-iteration counters (iteration_fwd_done, stages_closed), tagged ring
    long long it_fwd[SIMF_SLOTS];
    int it_closed[SIMF_SLOTS], it_tag[SIMF_SLOTS];
    for (int i = 0; i < SIMF_SLOTS; ++i) { it_fwd[i] = 0; it_closed[i] = 0; it_tag[i] = -1; }
    auto it_slot = [&](int it) -> int {
        const int k = it & (SIMF_SLOTS - 1);
        if (it_tag[k] != it) {
            if (it_tag[k] >= 0 && it_closed[k] != S) overflow = true;
            it_tag[k] = it; it_fwd[k] = 0; it_closed[k] = 0;
        }
        return k;
    };
    // adapter state (src/adapter.py:91-150)
    long long cur_sz[GP_MAX_STAGES];
    int phase[GP_MAX_STAGES];  // 0 FILL, 1 RUN, 2 DRAIN
    AdWindow* W = sc.win + tid * (long long)(2 * (sc.smax > 1 ? sc.smax - 1 : 1));
    unsigned actions = 0;
    for (int s = 0; s < S; ++s) { cur_sz[s] = m; phase[s] = 0; }
    for (int l = 0; l < 2 * (S - 1); ++l) {
        W[l].head = W[l].len = 0; W[l].baseline = 0.0; W[l].count = W[l].since = 0;
        W[l].degraded = W[l].exists = 0;
    }
    double now = 0.0;
    // _apply (src/adapter.py:158-165); signal 0 fill, 1 drain, 2 degraded, 3 recovered
    auto ad_apply = [&](int s, long long size, int signal) {
        if (size != cur_sz[s]) {
            if (act_out && actions < act_cap) {
                gp_action a;
                a.t = now; a.stage = s; a.old_size = (int32_t)cur_sz[s];
                a.new_size = (int32_t)size; a.signal = (uint32_t)signal;
                act_out[actions] = a;
            }
            ++actions;
            cur_sz[s] = size;
        }
    };
    auto activate = [&](int s, int it) {  // src/engine.py:259-267
        SimFPool& q = pool(s, it);
        if (q.flags & 4) return;
        q.flags |= 4;
        if (s == 0) q.fwd_avail = B;
        if (adapter) {  // on_iteration_start (src/adapter.py:200-211)
            phase[s] = 0;
            bool poor = false;
            for (int b = s - 1; b <= s; ++b)
                for (int d = 0; d < 2; ++d)
                    if (b >= 0 && b < S - 1 && W[2 * b + d].exists && W[2 * b + d].degraded) poor = true;
            ad_apply(s, poor ? ad_halve(m) : m, 0);
        }
    };
    auto on_transfer = [&](int bnd, int dir, double raw, long long size) {
        // on_transfer_complete (src/adapter.py:167-198)
        const int producer = dir == 0 ? bnd : bnd + 1;
        AdWindow& w = W[2 * bnd + dir];
        w.exists = 1;
        const bool reduced = cur_sz[producer] < m;
        const double lat = raw / (double)size;  // record_transfer (:61-74)
        if (w.len < AD_WINDOW) { w.samples[(w.head + w.len) % AD_WINDOW] = lat; ++w.len; }
        else { w.samples[w.head] = lat; w.head = (w.head + 1) % AD_WINDOW; }
        ++w.count; ++w.since;
        if (!reduced) {
            if (w.count == 1) w.baseline = lat;
            else w.baseline += 0.05 * (lat - w.baseline);
        }
        if (w.since < AD_WINDOW) return;
        // detect_fluctuation (:77-88)
        if (w.len != AD_WINDOW || w.baseline <= 0) return;
        NeumaierSum acc;
        acc.start(w.samples[w.head]);
        for (int i = 1; i < AD_WINDOW; ++i) acc.add(w.samples[(w.head + i) % AD_WINDOW]);
        const double mean = acc.value() / (double)AD_WINDOW;
        int sig = 0;
        if (mean > opt.degrade_factor * w.baseline) sig = 1;
        else if (reduced && mean < opt.recover_factor * w.baseline) sig = 2;
        if (sig == 0) return;
        w.degraded = sig == 1;
        // adjust (:105-113)
        const long long c = cur_sz[producer];
        long long ns = c;
        if (phase[producer] == 2 || sig == 1) ns = ad_halve(c);
        else ns = c * 2 < m ? c * 2 : m;
        if (ns != c) { w.since = 0; ad_apply(producer, ns, sig == 1 ? 2 : 3); }
    };

    int cur[GP_MAX_STAGES];
    bool busy[GP_MAX_STAGES];
    long long l_head[2 * GP_MAX_STAGES], l_tail[2 * GP_MAX_STAGES];
    bool l_busy[2 * GP_MAX_STAGES];
    NeumaierSum bsum[GP_MAX_STAGES];
    int bn[GP_MAX_STAGES];
    unsigned n_ops = 0, n_xfer = 0;
    SimFEv ev[3 * GP_MAX_STAGES];
    int nev = 0;
    unsigned long long seq = 0;
    for (int l = 0; l < 2 * (S - 1); ++l) { l_head[l] = l_tail[l] = 0; l_busy[l] = false; }
    if (iter_ends)
        for (int i = 0; i < iterations; ++i) iter_ends[i] = 0.0;
    for (int s = 0; s < S; ++s) {
        cur[s] = 0;
        busy[s] = false;
        bn[s] = 0;
        activate(s, 0);
    }
    auto push_op = [&](double tnow, double dur, int s, int k, int it, long long size, int mb) {
        SimFEv& e = ev[nev++];
        e.t = tnow + dur; e.t0 = tnow; e.seq = seq++;
        e.code = (s << 20) | (k << 16);
        e.it = it; e.size = size; e.mb = mb;
        if (ops_out && n_ops < op_cap) {  // ops[s].append(op) at start (src/engine.py:322-330)
            gp_op o;
            o.start = e.t0; o.end = e.t; o.size = (int32_t)size; o.microbatch_id = mb;
            o.iteration = (uint32_t)it; o.kind = (uint8_t)k; o.stage = (uint8_t)s; o.pad = 0;
            ops_out[n_ops] = o;
        }
        ++n_ops;
    };
    auto try_start = [&](double tnow, int bnd, int dir) {  // src/engine.py:276-289
        const int l = 2 * bnd + dir;
        if (l_busy[l] || l_head[l] >= l_tail[l]) return;
        const unsigned long long v = lq_at(l, l_head[l]++);
        l_busy[l] = true;
        const long long sz = (long long)(v & 0xffffffull);
        const double per = dir == 0 ? T.act[bnd] : T.grad[bnd];
        SimFEv& e = ev[nev++];
        e.t = transfer_end(tnow, per * (double)sz, T.bw[bnd], T.lat[bnd], trace, bnd);
        e.t0 = tnow; e.seq = seq++;
        e.code = (int)(1u << 31) | (bnd << 20) | (dir << 16);
        e.it = (int)(v >> 48); e.mb = (int)((v >> 24) & 0xffffffull); e.size = sz;
    };
    auto enqueue = [&](double tnow, int bnd, int dir, long long size, int it, int mb) {
        const int l = 2 * bnd + dir;
        if (l_tail[l] - l_head[l] >= sc.lcap) { overflow = true; return; }
        lq_at(l, l_tail[l]++) = ((unsigned long long)(unsigned)it << 48) |
                                ((unsigned long long)(unsigned)mb << 24) | (unsigned long long)size;
        try_start(tnow, bnd, dir);
    };
    while (!overflow) {
        bool progress = true;
        while (progress) {  // dispatch (src/engine.py:335-341)
            progress = false;
            for (int s = 0; s < S; ++s) {
                if (busy[s]) continue;
                const int it = cur[s];
                if (it >= iterations) continue;
                SimFPool& p = pool(s, it);
                const bool wq_any = p.wq_head < p.wq_tail;
                long long size = adapter ? cur_sz[s] : m, best_sz;
                const int k = ready_op(policy, S, s, B, m, size, p.fwd_avail, p.fwd_taken, p.fwd_done,
                                       p.bwd_avail, p.bwd_taken, p.bwd_done, p.w_done, wq_any,
                                       wq_any ? (long long)wq_at(s, it, p.wq_head) : 0,
                                       (p.flags & 1) != 0, (p.flags & 2) != 0, &best_sz);
                if (k < 0) {
                    if (async_it && p.fwd_taken == B && it + 1 < iterations) {
                        activate(s, it + 1);  // may resize the stage
                        size = adapter ? cur_sz[s] : m;
                        SimFPool& nx = pool(s, it + 1);
                        const long long rem = B - nx.fwd_taken;
                        const long long chunk = size < rem ? size : rem;
                        if (rem > 0 && nx.fwd_avail - nx.fwd_taken >= chunk) {
                            nx.fwd_taken += chunk;
                            busy[s] = true;
                            push_op(now, T.fwd[s] * (double)chunk, s, 0, it + 1, chunk, nx.f_ids++);
                            progress = true;
                        }
                    }
                    continue;
                }
                double dur;
                int mb = -1;
                switch (k) {
                    case 0: dur = T.fwd[s] * (double)best_sz; p.fwd_taken += best_sz; mb = p.f_ids++; break;
                    case 1: dur = T.bwd[s] * (double)best_sz; p.bwd_taken += best_sz; mb = p.b_ids++; break;
                    // W takes the queue head: the B of id wq_head (B ids are dense, FIFO)
                    case 2: dur = T.wgt[s] * (double)best_sz; mb = p.wq_head++; break;
                    case 3: dur = T.sync[s]; break;
                    default: dur = T.opt[s]; break;
                }
                busy[s] = true;
                push_op(now, dur, s, k, it, best_sz, mb);
                progress = true;
            }
        }
        if (nev == 0 || overflow) break;
        int bi = 0;
        for (int i = 1; i < nev; ++i)
            if (ev[i].t < ev[bi].t || (ev[i].t == ev[bi].t && ev[i].seq < ev[bi].seq)) bi = i;
        const SimFEv e = ev[bi];
        ev[bi] = ev[--nev];
        now = e.t;
        const int it = e.it, sb = (e.code >> 20) & 0x7ff, op = (e.code >> 16) & 0xf;
        if (e.code >= 0) {  // finish_op (src/engine.py:343-378)
            const int s = sb;
            SimFPool& p = pool(s, it);
            busy[s] = false;
            const double x = now - e.t0;
            if (bn[s]++ == 0) bsum[s].start(x); else bsum[s].add(x);
            if (op == 0) {
                p.fwd_done += e.size;
                if (s < S - 1) enqueue(now, s, 0, e.size, it, e.mb);
                const int ks = it_slot(it);
                it_fwd[ks] += e.size;
                if (adapter && it_fwd[ks] == (long long)S * B)
                    for (int q = 0; q < S; ++q) { phase[q] = 2; ad_apply(q, ad_halve(cur_sz[q]), 1); }
            } else if (op == 1) {
                p.bwd_done += e.size;
                if (p.wq_tail >= sc.wcap) { overflow = true; break; }
                wq_at(s, it, p.wq_tail++) = (uint32_t)e.size;
                if (!(p.flags & 8)) { p.flags |= 8; if (adapter) phase[s] = 1; }
                if (s > 0) enqueue(now, s - 1, 1, e.size, it, e.mb);
            } else if (op == 2) {
                p.w_done += e.size;
            } else if (op == 3) {
                p.flags |= 1;
            } else {
                p.flags |= 2;
                const int ks = it_slot(it);
                if (++it_closed[ks] == S && iter_ends) iter_ends[it] = now;
                cur[s] = it + 1;
                if (it + 1 < iterations) activate(s, it + 1);
            }
        } else {  // finish_transfer (src/engine.py:380-396)
            l_busy[2 * sb + op] = false;
            if (op == 0) pool(sb + 1, it).fwd_avail += e.size;
            else pool(sb, it).bwd_avail += e.size;
            if (xf_out && n_xfer < xf_cap) {  // transfers.append (src/engine.py:388-393)
                gp_transfer x;
                x.start = e.t0; x.end = now; x.size = (int32_t)e.size; x.microbatch_id = e.mb;
                x.iteration = (uint32_t)it; x.boundary = (uint8_t)sb; x.direction = (uint8_t)op;
                x.pad = 0;
                xf_out[n_xfer] = x;
            }
            ++n_xfer;
            if (adapter) on_transfer(sb, op, now - e.t0, e.size);
            try_start(now, sb, op);
        }
    }
    if (overflow) return GP_ERR_CUDA;  // capacity bound broken: never a silent result
    if ((ops_out && n_ops != op_cap) || (xf_out && n_xfer != xf_cap) ||
        (act_out && (long long)actions != act_cap))
        return GP_ERR_INPUT;
    rep->makespan = now;
    for (int s = 0; s < GP_MAX_STAGES; ++s) rep->busy[s] = s < S && bn[s] ? bsum[s].value() : 0.0;
    rep->adapter_actions = actions;
    rep->n_ops = n_ops;
    rep->n_transfers = n_xfer;
    rep->pad = 0;
    for (int s = 0; s < S; ++s)
        if (cur[s] < iterations) return GP_ERR_SCHEDULING;
    return GP_OK;
}

__global__ void k5_sim_full(const gp_timing* __restrict__ T, long long n, int policy, int iterations,
                            const gp_trace* __restrict__ traces, const uint32_t* __restrict__ tidx,
                            gp_sim_options opt, SimScratch sc, gp_sim_report* __restrict__ rep,
                            double* __restrict__ iter_ends, uint8_t* __restrict__ status,
                            const uint32_t* __restrict__ perm = nullptr) {
    const long long slot = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // scratch slot
    if (slot >= n) return;
    const long long i = perm ? (long long)perm[slot] : slot;  // timing (perm: global index)
    const gp_trace* tr = traces ? traces + (tidx ? tidx[i] : 0u) : nullptr;
    gp_sim_report r;
    int st = sim_full(T[i], policy, iterations, tr, opt, sc, slot, &r,
                      iter_ends ? iter_ends + i * (long long)iterations : nullptr, nullptr, 0,
                      nullptr, 0, nullptr, 0);
    if (st != GP_OK && st != GP_ERR_SCHEDULING) {
        r.makespan = NAN;
        for (int s = 0; s < GP_MAX_STAGES; ++s) r.busy[s] = 0.0;
        r.adapter_actions = r.n_ops = r.n_transfers = r.pad = 0;
    }
    if (st == GP_ERR_SCHEDULING) r.makespan = NAN;
    rep[i] = r;
    status[i] = (uint8_t)st;
}

// Schedules: as k5_sim_full, writing the op / transfer records of timing i
// at its offsets (sized by a previous report pass).
__global__ void k5_sim_schedule(const gp_timing* __restrict__ T, long long n, int policy,
                                int iterations, const gp_trace* __restrict__ traces,
                                const uint32_t* __restrict__ tidx, gp_sim_options opt, SimScratch sc,
                                const unsigned long long* __restrict__ op_off, gp_op* __restrict__ ops,
                                const unsigned long long* __restrict__ xf_off,
                                gp_transfer* __restrict__ xfers,
                                const unsigned long long* __restrict__ ac_off,
                                gp_action* __restrict__ acts, uint8_t* __restrict__ status) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const gp_trace* tr = traces ? traces + (tidx ? tidx[i] : 0u) : nullptr;
    gp_sim_report r;
    const long long o0 = (long long)op_off[i], o1 = (long long)op_off[i + 1];
    long long x0 = 0, x1 = 0;
    if (xfers) { x0 = (long long)xf_off[i]; x1 = (long long)xf_off[i + 1]; }
    long long a0 = 0, a1 = 0;
    if (acts) { a0 = (long long)ac_off[i]; a1 = (long long)ac_off[i + 1]; }
    int st = sim_full(T[i], policy, iterations, tr, opt, sc, i, &r, nullptr, ops + o0, o1 - o0,
                      xfers ? xfers + x0 : nullptr, x1 - x0, acts ? acts + a0 : nullptr, a1 - a0);
    status[i] = (uint8_t)st;
}
