// detail.cuh - winner plan detail (splits + CostBreakdown) and on-device key decode.
#pragma once
#include "k2_eval.cuh"

// ---- plan detail of one candidate (single thread) -----------------------------------
__device__ void plan_detail_warp(const DevInst& I, int k, const uint8_t* o, const int* p, int bm,
                                 gp_plan_info* out, int* status);

__global__ void k_plan_detail(DevInst I, int k, const uint8_t* order_in, const uint8_t* counts_in,
                              int bm, gp_plan_info* out, int* status) {
    uint8_t o[GP_MAX_STAGES];
    int p[GP_MAX_STAGES + 1];
    p[0] = 0;
    for (int s = 0; s < k; ++s) { o[s] = order_in[s]; p[s + 1] = p[s] + counts_in[s]; }
    plan_detail_warp(I, k, o, p, bm, out, status);
}

// Winner of the last arg-min -> decoded candidate + plan detail, on the
// device (no host round trip between the arg-min and the breakdown).
struct SolveOut {
    Key key;  // (sizeof is a multiple of 8: copied in 8-byte words)
    unsigned long long err;
    int status;        // of the detail evaluation
    uint32_t k, bm, flags;  // flags: the table-build flags word (FLAG_*)
    uint8_t order[GP_MAX_STAGES];
    uint8_t counts[GP_MAX_STAGES];
    gp_plan_info info;
    unsigned long long seq;  // gp_replan graph: written last, after a system fence
};

static_assert(sizeof(SolveOut) % 8 == 0, "SolveOut is copied in 8-byte words");

// Warp version of plan_detail_dev: lane s prepares stage s (split choice and
// table loads in parallel), lane 0 runs the short Eq. 1 chain.
__device__ void plan_detail_warp(const DevInst& I, int k, const uint8_t* o, const int* p, int bm,
                                 gp_plan_info* out, int* status) {
    const int lane = threadIdx.x & 31;
    const int n = I.n;
    const size_t N2 = (size_t)(n + 1) * (n + 1);
    const int mi = bm % I.nm;
    const double Md = I.mtab[bm];  // (double)(batch / micro), K1
    const double2* T = I.stg + (size_t)mi * I.F * N2;
    const double* X = I.xt + (size_t)mi * I.F * I.F * I.nxp;
    double2 e = make_double2(0.0, 0.0);
    double x = 0.0;
    uint8_t code = SC_OK;
    bool gw_bad = false;
    if (lane < k) {
        // the split of (group, a, b) comes from K1's tables (kind, first PP
        // share, group sizes); only groups with > 2 second-level groups
        // re-run choose_intra_split for their PP shares
        const int s = lane;
        gp_stage_info& st = out->stage[s];
        const int f = o[s], a = p[s], b = p[s + 1];
        const size_t ei = (size_t)f * N2 + tri_idx(n, a, b);
        const int kind = I.skind[ei];
        const int sh0 = I.sshare0[ei];
        const K1Grp g = I.grp[f];
        e = T[ei];
        code = I.scode[ei];
        if (s + 1 < k) {
            x = X[((size_t)f * I.F + o[s + 1]) * I.nxp + (b - 1)];
            gw_bad = I.gwbad[f * I.F + o[s + 1]] != 0;
        }
        const int np = kind == GP_UNIFORM ? 0 : (kind == GP_ASYM_TP_DP ? g.nmem : g.nsg);
        st.kind = (uint32_t)kind;
        st.n_parts = (uint32_t)np;
        if (kind == GP_ASYM_PP) {
            if (g.nsg == 2) {
                st.pp_sg[0] = 0u; st.pp_start[0] = (uint32_t)a; st.pp_end[0] = (uint32_t)(a + sh0);
                st.pp_sg[1] = 1u; st.pp_start[1] = (uint32_t)(a + sh0); st.pp_end[1] = (uint32_t)b;
            } else {
                int shares[GP_MAX_SGS], np2;
                choose_split(I, f, a, b, shares, &np2);
                int pos = a;
                for (int j = 0; j < np2; ++j) {
                    st.pp_sg[j] = (uint32_t)j;
                    st.pp_start[j] = (uint32_t)pos;
                    st.pp_end[j] = (uint32_t)(pos + shares[j]);
                    pos += shares[j];
                }
            }
        }
    }
    const unsigned infeas = __ballot_sync(0xffffffffu, lane < k && code == SC_INFEASIBLE);
    const unsigned errs = __ballot_sync(0xffffffffu, lane < k && code != SC_OK && code != SC_INFEASIBLE);
    const unsigned gbad = __ballot_sync(0xffffffffu, gw_bad);
    const int first_err = errs ? __shfl_sync(0xffffffffu, (int)code, __ffs(errs) - 1) : 0;
    // lane 0: the sequential chain; stage values arrive by shuffles
    double fill = 0.0, res = 0.0, xprev = 0.0, best = 0.0;
    int st = GP_OK;
    const bool feas = infeas == 0u;
    if (!feas) best = INFINITY;
    else if (p[k] != n) st = GP_ERR_TOPOLOGY;
    else if (errs) st = first_err;
    else if (gbad) st = GP_ERR_TOPOLOGY;
    for (int s = 0; s < k; ++s) {
        const double cx = __shfl_sync(0xffffffffu, e.x, s);
        const double cy = __shfl_sync(0xffffffffu, e.y, s);
        const double xs = __shfl_sync(0xffffffffu, x, s);
        if (!feas || st != GP_OK) continue;
        if (s > 0) res = res + gpd::max0(xprev - cx);
        const double run = Md * cx;
        const double total = ((fill + run) + res) + cy;
        best = (s == 0 || total > best) ? total : best;
        if (lane == 0) {
            out->stage[s].fill_seconds = fill;
            out->stage[s].run_seconds = run;
            out->stage[s].residual_seconds = res;
            out->stage[s].collective_seconds = cy;
        }
        if (s + 1 < k) {
            fill = fill + (cx + xs);
            xprev = xs;
        }
    }
    if (lane == 0) {
        out->k = (uint32_t)k;
        out->feasible = feas ? 1 : 0;
        out->plan_cost = best;
        *status = st;
    }
}

// Decode of one arg-min key + plan detail into `out` (shared memory); one
// warp.  Out of line so that the icache warm-up pass and the real pass run
// the same instructions.
__device__ __noinline__ void solve_body(const DevInst& I, int k, unsigned long long NC, int nbm,
                                        Key key, unsigned long long e, uint32_t flags,
                                        const unsigned long long* bsm, SolveOut* out) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
        out->key = key;
        out->err = e;
        out->k = (uint32_t)k;
        out->status = GP_OK;
        out->flags = flags;  // table flags travel back with the result
    }
    if (e != ~0ull || key.tie == ~0ull) return;
    const int n = I.n;
    const unsigned long long t = key.tie;
    int bm;
    unsigned long long pc;
    if (t < (1ull << 32)) {  // 32-bit division when the key fits (every realistic space)
        bm = (int)((unsigned)t % (unsigned)nbm);
        pc = (unsigned)t / (unsigned)nbm;
    } else {
        bm = (int)(t % (unsigned long long)nbm);
        pc = t / (unsigned long long)nbm;
    }
    uint8_t o[GP_MAX_STAGES];
    int p[GP_MAX_STAGES + 1];
    unsigned long long rem;
    if (pc < (1ull << 32) && NC < (1ull << 32)) {
        d_unrank_perm(k, (unsigned)pc / (unsigned)NC, o);
        rem = (unsigned)pc % (unsigned)NC;
    } else {
        d_unrank_perm(k, pc / NC, o);
        rem = pc % NC;
    }
    p[0] = 0;
    int prev = 0;
    auto C = [&](int nn, int r) -> unsigned long long {
        return (r < 0 || nn < 0) ? 0ull : bsm[nn * (k + 1) + r];
    };
    for (int j = 1; j < k; ++j) {
        const int r = k - 1 - j, lo = prev + 1;
        const unsigned long long tot = C(n - lo, r + 1), thr = tot - rem;
        int qsel = -1;
        for (int base = lo; qsel < 0 && base <= n - 1 - r; base += 32) {
            const int qq = base + lane;
            const bool ok = qq <= n - 1 - r && C(n - qq - 1, r + 1) < thr;
            const unsigned m = __ballot_sync(0xffffffffu, ok);
            if (m) qsel = base + __ffs(m) - 1;
        }
        if (qsel < 0) qsel = n - 1 - r;  // (unreachable for a valid key)
        rem -= tot - C(n - qsel, r + 1);
        p[j] = qsel;
        prev = qsel;
    }
    p[k] = n;
    if (lane == 0) {
        out->bm = (uint32_t)bm;
        for (int s = 0; s < k; ++s) {
            out->order[s] = o[s];
            out->counts[s] = (uint8_t)(p[s + 1] - p[s]);
        }
    }
    plan_detail_warp(I, k, o, p, bm, &out->info, &out->status);
}

__global__ void k_solve_detail(DevInst I, int k, unsigned long long NC, unsigned long long NP,
                               int nbm, const Key* result, const unsigned long long* err,
                               const unsigned long long* __restrict__ binom, SolveOut* out,
                               int warm, unsigned long long* seqctr) {
    // one warp: decode the arg-min key (cut positions by a 32-wide ballot
    // over the hockey-stick counts), then the warp plan detail
    (void)NP;
    const int lane = threadIdx.x & 31;
    TL_START();
    pdl_trigger();
    // the record is assembled in shared memory and leaves in one coalesced
    // pass (the destination may be mapped host memory)
    __shared__ __align__(16) SolveOut so;
    // the binomial columns the decode reads, staged once (independent loads
    // overlap) instead of one dependent global round trip per probe
    __shared__ unsigned long long bsm[(GP_MAX_LAYERS + 1) * (GP_MAX_STAGES + 1)];
    for (int nn = lane; nn <= I.n; nn += 32)
        for (int r = 0; r <= k; ++r) bsm[nn * (k + 1) + r] = binom[(size_t)nn * (GP_MAX_STAGES + 1) + r];
    __syncwarp();
    // inside the gp_replan graph this kernel is scheduled while the arg-min
    // still runs: one pass over candidate rank 0 (valid for every instance;
    // the tables it reads are this instance's) pulls the code of the decode
    // and detail into the instruction cache before the real key exists
    if (warm) solve_body(I, k, NC, nbm, Key{0.0, 0ull}, ~0ull, 0u, bsm, &so);
    {
        __syncwarp();
        unsigned long long* z = (unsigned long long*)&so;
        for (int q = lane; q < (int)(sizeof(SolveOut) / 8); q += 32) z[q] = 0ull;
        __syncwarp();
    }
    pdl_wait();  // the arg-min (binom is static: staged before the wait)
    TL_WAITED();
#if defined(GP_TIMELINE)
    const unsigned long long td0 = tl_now();
#endif
    solve_body(I, k, NC, nbm, *result, *err, *I.flags, bsm, &so);
#if defined(GP_TIMELINE)
    const unsigned long long td1 = tl_now();
#endif
    __syncwarp();
    const unsigned long long* src = (const unsigned long long*)&so;
    unsigned long long* d = (unsigned long long*)out;
    const int nw = (int)(offsetof(SolveOut, seq) / 8);
    for (int q = lane; q < nw; q += 32) d[q] = src[q];
    if (seqctr) {
        // the host polls `seq` instead of synchronising the stream: the
        // record's words are fenced to the system before the new number lands
        __threadfence_system();
        __syncwarp();
        if (lane == 0) {
            const unsigned long long v = *seqctr + 1ull;
            *seqctr = v;
            *(volatile unsigned long long*)&out->seq = v;
        }
    }
    TL_STOP(50);
#if defined(GP_TIMELINE)
    if (lane == 0) {  // sub-phases: real pass start / detail done / exit
        unsigned int i2 = atomicAdd(&g_tl_n, 1u);
        if (i2 < GP_TL_CAP) g_tl[i2] = TlRec{td0, td1, tl_now(), 51u, 0u, 0u, 0u};
    }
#endif
}


// ---- cost of an explicit plan -------------------------------------------------------
// plan_cost(plan, topology, model, groups, opt_seconds) (src/costmodel.py:92-100)
// = Eq. 1 over build_plan_timing(plan) (src/timing.py:176-231) for a plan
// whose splits are given (not chosen): only the split kind and the
// ASYMMETRIC_PP parts enter the cost (effective_capacity, collective
// volume); memory is not checked (plan_cost does not).  One warp: lane s
// builds stage s, lane 0 runs the Eq. 1 chain.  Optionally emits the
// PlanTiming record.
__global__ void k_plan_cost(DevInst I, int k, const gp_plan_stage* __restrict__ stages,
                            long long batch, long long micro, double opt_seconds,
                            gp_plan_info* out, gp_timing* timing, int* status) {
    const int lane = threadIdx.x & 31;
    const int n = I.n;
    const double md = (double)micro;
    double cx = 0.0, cy = 0.0, xs = 0.0;
    uint8_t code = SC_OK;
    bool gw_bad = false;
    if (lane < k) {
        const gp_plan_stage& g = stages[lane];
        const int f = (int)g.fg, a = (int)g.layer_start, b = (int)g.layer_end;
        const int m0 = I.fg_off[f], m1 = I.fg_off[f + 1], nmem = m1 - m0;
        const int s0 = I.fg_sg_off[f];
        const double P = Ssum(I, COL_PARAM, a, b);
        // effective_capacity (src/timing.py:116-143)
        double cap;
        if (g.kind == GP_ASYM_PP) {
            const double tot = Ssum(I, COL_TF, a, b);
            bool have = false;
            double best = 0.0;
            for (int j = 0; j < (int)g.n_parts; ++j) {
                const int st = (int)g.pp_start[j], en = (int)g.pp_end[j];
                const double sub = st < en ? Ssum(I, COL_TF, st, en) : 0.0;
                const double frac = sub / tot;
                if (frac > 0) {
                    const double val = I.sg_cap[s0 + g.pp_sg[j]] / frac;
                    if (!have || val < best) best = val;
                    have = true;
                }
            }
            cap = best;
            if (!have) code = SC_DEGENERATE;
        } else {
            cap = I.fg_cap[f];
            if (!(cap > 0)) code = SC_DEGENERATE;
        }
        const double Fp = Ssum(I, COL_FWD, a, b) / cap;
        const double Bp = Ssum(I, COL_BWD, a, b) / cap;
        const double Wp = Ssum(I, COL_WGT, a, b) / cap;
        const bool has = I.fg_has_minbw[f] != 0;
        const double mbw = I.fg_minbw[f];
        const double sync = (P == 0.0 || !has) ? 0.0 : (mbw > 0 ? P / mbw : NAN);
        if (code == SC_OK && has && !(mbw > 0) && (nmem >= 2 || P != 0.0)) code = SC_TOPOLOGY;
        double al = 0.0;
        if (nmem >= 2) {  // collective_volume / intra_group_seconds (:146-173)
            double V = 2.0 * P;
            if (g.kind == GP_ASYM_TP_DP) V = V + I.act[b - 1] * md;
            if (V != 0.0 && has && mbw > 0) al = V / mbw;
        }
        cx = ((Fp + Bp) + Wp) * md;
        cy = al;
        if (lane + 1 < k) {  // gateway boundary (src/timing.py:208-224)
            const int gl = I.gw[f * I.F + (int)stages[lane + 1].fg];
            const double bwv = I.bw[gl];
            gw_bad = !(bwv > 0);
            xs = I.lat[gl] + (I.act[b - 1] * md) / bwv;
            if (timing) {
                timing->lat[lane] = I.lat[gl];
                timing->bw[lane] = bwv;
                timing->act[lane] = timing->grad[lane] = I.act[b - 1];
            }
        }
        if (timing) {
            timing->fwd[lane] = Fp; timing->bwd[lane] = Bp; timing->wgt[lane] = Wp;
            timing->sync[lane] = sync; timing->opt[lane] = opt_seconds;
        }
    }
    // stage errors in stage order, then zero-bandwidth gateways (the
    // reference builds every StageTiming before the boundaries)
    const unsigned errs = __ballot_sync(0xffffffffu, lane < k && code != SC_OK);
    const unsigned gbad = __ballot_sync(0xffffffffu, gw_bad);
    const int first_err = errs ? __shfl_sync(0xffffffffu, (int)code, __ffs(errs) - 1) : 0;
    int st = errs ? first_err : (gbad ? GP_ERR_TOPOLOGY : GP_OK);
    double fill = 0.0, res = 0.0, xprev = 0.0, best = 0.0;
    const double Md = (double)(batch / micro);
    for (int s = 0; s < k; ++s) {
        const double ex = __shfl_sync(0xffffffffu, cx, s);
        const double ey = __shfl_sync(0xffffffffu, cy, s);
        const double xv = __shfl_sync(0xffffffffu, xs, s);
        if (st != GP_OK) continue;
        if (s > 0) res = res + gpd::max0(xprev - ex);
        const double run = Md * ex;
        const double total = ((fill + run) + res) + ey;
        best = (s == 0 || total > best) ? total : best;
        if (lane == 0) {
            out->stage[s].kind = stages[s].kind;
            out->stage[s].n_parts = stages[s].n_parts;
            out->stage[s].fill_seconds = fill;
            out->stage[s].run_seconds = run;
            out->stage[s].residual_seconds = res;
            out->stage[s].collective_seconds = ey;
        }
        if (s + 1 < k) {
            fill = fill + (ex + xv);
            xprev = xv;
        }
    }
    if (lane == 0) {
        out->k = (uint32_t)k;
        out->feasible = 1;
        out->plan_cost = best;
        if (timing) {
            timing->n_stages = (uint32_t)k;
            timing->pad = 0;
            timing->batch = batch;
            timing->microbatch = micro;
        }
        *status = st;
    }
}
