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
                // _ready_op (src/engine.py:157-215): candidates F, B, W, SYNC,
                // OPT in this order; lowest priority wins, earliest on ties
                const bool zbc = policy == GP_POLICY_ZB_COMPACT, zbo = policy == GP_POLICY_ZB_ORIGINAL;
                const bool gpipe = policy == GP_POLICY_GPIPE;
                int best_pr = 100, best_k = -1;
                long long best_sz = 0;
                const long long fwd_rem = B - p.fwd_taken;
                if (fwd_rem > 0) {
                    const long long chunk = m < fwd_rem ? m : fwd_rem;
                    if (p.fwd_avail - p.fwd_taken >= chunk) {
                        int pr = -1;
                        if (zbc || gpipe) {
                            pr = zbc ? 0 : 1;
                        } else {
                            const long long quota = (long long)(S - s) * m;
                            if (p.fwd_taken < quota) pr = zbo ? 0 : 1;
                            else if (p.fwd_taken + chunk <= quota + p.bwd_done) pr = zbo ? 3 : 2;
                        }
                        if (pr >= 0) { best_pr = pr; best_k = 0; best_sz = chunk; }
                    }
                }
                const long long bwd_rem = B - p.bwd_taken;
                if (bwd_rem > 0 && (!gpipe || p.fwd_done == B)) {
                    const long long chunk = m < bwd_rem ? m : bwd_rem;
                    long long av = (p.bwd_avail < p.fwd_done ? p.bwd_avail : p.fwd_done) - p.bwd_taken;
                    if (s == S - 1) av = p.fwd_done - p.bwd_taken;
                    const int pr = (zbc || zbo) ? 1 : 2;
                    if (av >= chunk && pr < best_pr) { best_pr = pr; best_k = 1; best_sz = chunk; }
                }
                if (p.wq_head < p.wq_tail) {
                    const int pr = (gpipe || policy == GP_POLICY_1F1B) ? 0 : 2;
                    if (pr < best_pr) { best_pr = pr; best_k = 2; best_sz = chunk_size(p.wq_head); }
                }
                if (p.w_done == B && p.wq_head == p.wq_tail && !(p.flags & 1) && 8 < best_pr) {
                    best_pr = 8; best_k = 3; best_sz = 0;
                }
                if ((p.flags & 1) && !(p.flags & 2) && 9 < best_pr) { best_pr = 9; best_k = 4; best_sz = 0; }
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

// 1F1B makespan of explicit candidates: the PlanTiming of build_plan_timing
// (src/timing.py:176-231) assembled from the stage / boundary tables.
__global__ void k5_sim_candidates(DevInst I, int k, long long ncand, const uint8_t* __restrict__ order,
                                  const uint8_t* __restrict__ counts, const uint8_t* __restrict__ bm,
                                  int iterations, double opt_seconds, double* __restrict__ makespan,
                                  uint8_t* __restrict__ status) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ncand) return;
    uint8_t o[GP_MAX_STAGES];
    int p[GP_MAX_STAGES + 1];
    p[0] = 0;
    int st = GP_OK;
    unsigned seen = 0;
    for (int s = 0; s < k; ++s) {
        o[s] = order[i * k + s];
        int c = counts[i * k + s];
        if (o[s] >= I.F || (seen >> o[s]) & 1u || c == 0) st = GP_ERR_INPUT;
        seen |= 1u << (o[s] & 31);
        p[s + 1] = p[s] + c;
    }
    int b = bm[i];
    if (b >= I.nb * I.nm || p[k] > I.n) st = GP_ERR_INPUT;
    int mi = b % I.nm;
    if (st == GP_OK) {
        long long M = I.batch[b / I.nm] / I.micro[mi];
        EvalOut r = eval_tables(I, k, o, p, mi, M);  // feasibility + errors, as _evaluate
        st = r.status;
        if (st == GP_OK && isinf(r.cost)) st = GP_ERR_NO_FEASIBLE;  // memory-infeasible plan
    }
    if (st != GP_OK) { makespan[i] = NAN; status[i] = (uint8_t)st; return; }
    const size_t N2 = (size_t)(I.n + 1) * (I.n + 1);
    gp_timing T;
    T.n_stages = (uint32_t)k;
    T.batch = I.batch[b / I.nm];
    T.microbatch = I.micro[mi];
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
    double ms = NAN;
    st = sim_dev(T, GP_POLICY_1F1B, iterations, nullptr, &ms);
    makespan[i] = ms;
    status[i] = (uint8_t)st;
}

__global__ void k5_sim_1f1b(const gp_timing* __restrict__ T, long long n, int policy, int iterations,
                            const gp_trace* __restrict__ traces, const uint32_t* __restrict__ tidx,
                            double* __restrict__ makespan, uint8_t* __restrict__ status) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double ms = NAN;
    const gp_trace* tr = traces ? traces + (tidx ? tidx[i] : 0u) : nullptr;
    int st = sim_dev(T[i], policy, iterations, tr, &ms);
    makespan[i] = ms;
    status[i] = (uint8_t)st;
}

