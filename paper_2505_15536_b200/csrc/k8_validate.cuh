// k8_validate.cuh - K8: validate_schedule + bubble_fraction busy sums for a
// batch of schedules, one thread per schedule (src/schedule.py:95-182).
#pragma once
#include "common.cuh"

// ----------------------------------------------------------------------------
// The reference indexes ops by (stage, iteration, kind, micro-batch id) in a
// dict.  Engine schedules number F / B / W ops densely per (stage,
// iteration, kind) in list order, so the dict becomes a table: op k of
// (s, it, kind) sits at idx[base(s, it, kind) + k].  A schedule that breaks
// density (or carries an id on a sync / optimizer op) is rejected with
// GP_ERR_INPUT rather than validated differently.
//
// Violations are emitted in the reference's order: ends-before-starts in
// stage-major list order; overlaps per stage over the ops stably sorted by
// (start, end); dependency checks in dict insertion order (= stage-major
// list order, each op its own key under density); per stage, iteration
// close checks in order of first appearance.
// ----------------------------------------------------------------------------
struct K8Iter {
    double last_w;
    int n_sync, n_opt, sync_idx, opt_idx, have_w, done;
};

struct K8Scratch {
    uint32_t* tab;      // [n][S_MAX*iters*3][2]  count, base
    uint32_t* idx;      // [total ops]            table payload
    uint32_t* sorted;   // [total ops]            per-stage sort buffer
    uint32_t* lists;    // [total ops]            op indices, stage-major, list order
    K8Iter* its;        // [n][S_MAX*iters]
};

__device__ __forceinline__ void k8_emit(gp_violation* out, uint32_t max_v, uint32_t& nv, int code,
                                        int stage, int kind, uint32_t it, int32_t mb, double t) {
    if (nv < max_v) {
        gp_violation v;
        v.t = t; v.iteration = it; v.microbatch_id = mb;
        v.code = (uint8_t)code; v.stage = (uint8_t)stage; v.kind = (uint8_t)kind; v.pad = 0;
        v.pad2 = 0;
        out[nv] = v;
    }
    ++nv;
}

__global__ void k8_validate(const gp_timing* __restrict__ T_all, long long n,
                            const unsigned long long* __restrict__ op_off,
                            const gp_op* __restrict__ ops_all, const double* __restrict__ makespan,
                            int iterations, double tol_rel, uint32_t max_v,
                            gp_violation* __restrict__ viol, uint32_t* __restrict__ n_viol,
                            double* __restrict__ busy_out, uint8_t* __restrict__ status,
                            K8Scratch sc) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const gp_timing& T = T_all[i];
    const int S = (int)T.n_stages;
    const long long o0 = (long long)op_off[i], m = (long long)op_off[i + 1] - o0;
    const gp_op* ops = ops_all + o0;
    gp_violation* out = viol + i * (long long)max_v;
    const int nq = GP_MAX_STAGES * iterations * 3;
    uint32_t* tab = sc.tab + i * (long long)nq * 2;
    uint32_t* idx = sc.idx + o0;
    uint32_t* srt = sc.sorted + o0;
    uint32_t* lst = sc.lists + o0;
    K8Iter* its = sc.its + i * (long long)GP_MAX_STAGES * iterations;
    uint32_t nv = 0;
    n_viol[i] = 0;
    if (S < 1 || S > GP_MAX_STAGES) { status[i] = GP_ERR_TIMING; return; }
    // structure checks + table counts
    for (int q = 0; q < nq * 2; ++q) tab[q] = 0;
    for (long long j = 0; j < m; ++j) {
        const gp_op& o = ops[j];
        if (o.stage >= S || o.kind > 4 || (int)o.iteration >= iterations ||
            (o.kind <= 2 && o.microbatch_id < 0) || (o.kind > 2 && o.microbatch_id >= 0)) {
            status[i] = GP_ERR_INPUT;
            return;
        }
        if (o.kind <= 2) {
            const int q = (o.stage * iterations + (int)o.iteration) * 3 + o.kind;
            if ((uint32_t)o.microbatch_id != tab[2 * q]) { status[i] = GP_ERR_INPUT; return; }
            tab[2 * q]++;
        }
    }
    {
        uint32_t base = 0;
        for (int q = 0; q < nq; ++q) { tab[2 * q + 1] = base; base += tab[2 * q]; }
    }
    for (long long j = 0; j < m; ++j) {
        const gp_op& o = ops[j];
        if (o.kind <= 2) {
            const int q = (o.stage * iterations + (int)o.iteration) * 3 + o.kind;
            idx[tab[2 * q + 1] + o.microbatch_id] = (uint32_t)j;
        }
    }
    auto lookup = [&](int s, uint32_t it, int kind, int32_t k) -> long long {
        const int q = (s * iterations + (int)it) * 3 + kind;
        if (k < 0 || (uint32_t)k >= tab[2 * q]) return -1;
        return idx[tab[2 * q + 1] + k];
    };
    // per-stage op lists (stage-major, list order): every later phase walks
    // one stage's ops without rescanning the whole schedule
    int soff[GP_MAX_STAGES + 1];
    for (int s = 0; s <= S; ++s) soff[s] = 0;
    for (long long j = 0; j < m; ++j) soff[ops[j].stage + 1]++;
    for (int s = 0; s < S; ++s) soff[s + 1] += soff[s];
    {
        int fillp[GP_MAX_STAGES];
        for (int s = 0; s < S; ++s) fillp[s] = soff[s];
        for (long long j = 0; j < m; ++j) lst[fillp[ops[j].stage]++] = (uint32_t)j;
    }
    const double tol = tol_rel * (makespan[i] > 1.0 ? makespan[i] : 1.0);
    // 1. ops that end before they start; bubble_fraction busy sums
    for (int s = 0; s < S; ++s) {
        NeumaierSum b;
        bool first = true;
        for (int q = soff[s]; q < soff[s + 1]; ++q) {
            const gp_op& o = ops[lst[q]];
            if (o.end < o.start - tol) k8_emit(out, max_v, nv, 0, s, o.kind, 0, 0, 0.0);
            const double x = o.end - o.start;
            if (first) { b.start(x); first = false; } else b.add(x);
        }
        if (busy_out) busy_out[i * GP_MAX_STAGES + s] = first ? 0.0 : b.value();
    }
    if (busy_out)
        for (int s = S; s < GP_MAX_STAGES; ++s) busy_out[i * GP_MAX_STAGES + s] = 0.0;
    // 2. overlaps: stable sort by (start, end) per stage
    for (int s = 0; s < S; ++s) {
        long long c = 0;
        for (int q = soff[s]; q < soff[s + 1]; ++q) srt[c++] = lst[q];
        for (long long a = 1; a < c; ++a) {
            const uint32_t v = srt[a];
            const double vs = ops[v].start, ve = ops[v].end;
            long long b = a - 1;
            while (b >= 0 && (ops[srt[b]].start > vs || (ops[srt[b]].start == vs && ops[srt[b]].end > ve))) {
                srt[b + 1] = srt[b];
                --b;
            }
            srt[b + 1] = v;
        }
        double prev_end = 0.0;
        for (long long a = 0; a < c; ++a) {
            const gp_op& o = ops[srt[a]];
            if (a > 0 && o.start < prev_end - tol) k8_emit(out, max_v, nv, 1, s, 0, 0, 0, o.start);
            const double base = (a > 0 && prev_end != 0.0) ? prev_end : o.end;  // `prev_end or op.end`
            prev_end = o.end > base ? o.end : base;
        }
    }
    // 3. dependencies (dict order = stage-major list order)
    for (int s = 0; s < S; ++s)
        for (int qq = soff[s]; qq < soff[s + 1]; ++qq) {
            const gp_op& o = ops[lst[qq]];
            if (o.kind > 2) continue;
            const int32_t k = o.microbatch_id;
            const uint32_t it = o.iteration;
            if (o.kind == 0 && s > 0) {
                const long long u = lookup(s - 1, it, 0, k);
                if (u >= 0) {
                    const double arrival =
                        ops[u].end + (T.lat[s - 1] + (T.act[s - 1] * (double)o.size) / T.bw[s - 1]);
                    if (o.start < arrival - tol) k8_emit(out, max_v, nv, 2, s, 0, it, k, 0.0);
                }
            }
            if (o.kind == 1) {
                const long long f = lookup(s, it, 0, k);
                if (f >= 0 && o.start < ops[f].end - tol) k8_emit(out, max_v, nv, 3, s, 1, it, k, 0.0);
                if (s < S - 1) {
                    const long long d = lookup(s + 1, it, 1, k);
                    if (d >= 0) {
                        const double arrival =
                            ops[d].end + (T.lat[s] + (T.grad[s] * (double)o.size) / T.bw[s]);
                        if (o.start < arrival - tol) k8_emit(out, max_v, nv, 4, s, 1, it, k, 0.0);
                    }
                }
            }
            if (o.kind == 2) {
                const long long b = lookup(s, it, 1, k);
                if (b >= 0 && o.start < ops[b].end - tol) k8_emit(out, max_v, nv, 5, s, 2, it, k, 0.0);
            }
        }
    // 4. iteration close, iterations in first-appearance order per stage
    for (int s = 0; s < S; ++s) {
        K8Iter* st = its + (long long)s * iterations;
        for (int q = 0; q < iterations; ++q) {
            st[q].n_sync = st[q].n_opt = 0; st[q].sync_idx = st[q].opt_idx = -1;
            st[q].have_w = 0; st[q].done = 0; st[q].last_w = 0.0;
        }
        for (int qq = soff[s]; qq < soff[s + 1]; ++qq) {
            const int j = (int)lst[qq];
            const gp_op& o = ops[j];
            K8Iter& q = st[o.iteration];
            if (o.kind == 3) { q.n_sync++; q.sync_idx = j; }
            if (o.kind == 4) { q.n_opt++; q.opt_idx = j; }
            if (o.kind == 2) {
                if (!q.have_w || o.end > q.last_w) q.last_w = o.end;
                q.have_w = 1;
            }
        }
        for (int qq = soff[s]; qq < soff[s + 1]; ++qq) {
            const gp_op& o = ops[lst[qq]];
            K8Iter& q = st[o.iteration];
            if (q.done) continue;
            q.done = 1;
            if (q.n_sync != 1 || q.n_opt != 1) {
                k8_emit(out, max_v, nv, 6, s, 0, o.iteration, 0, 0.0);
                continue;
            }
            if (ops[q.sync_idx].start < q.last_w - tol) k8_emit(out, max_v, nv, 7, s, 0, o.iteration, 0, 0.0);
            if (ops[q.opt_idx].start < ops[q.sync_idx].end - tol)
                k8_emit(out, max_v, nv, 8, s, 0, o.iteration, 0, 0.0);
        }
    }
    n_viol[i] = nv;
    status[i] = GP_OK;
}
