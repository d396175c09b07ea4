// k1_tables.cuh - K1: per-load table build (interval sums, group constants, stage and boundary tables).
#pragma once
#include "common.cuh"

// ---- K1a: interval sums -----------------------------------------------------
// sum(model.layers[i].<field> for i in range(a, b)) for every 0 <= a < b <= n,
// each interval summed from its own start (never prefix differences).
static __device__ void k1_intervals_block(const DevInst& I, int col) {
    // one CTA per column; the column is staged in shared memory so the
    // sequential Neumaier sweeps read on-chip values.  S is stored
    // transposed (b-major, see Ssum), so the lanes of a warp (consecutive a)
    // write consecutive addresses at every step of their sweeps.
    __shared__ double col_s[GP_MAX_LAYERS + 1];
    const int n = I.n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double x;
        switch (col) {
            case COL_FWD: x = I.fwd[i]; break;
            case COL_BWD: x = I.bwd_in[i]; break;
            case COL_WGT: x = I.bwd_w[i]; break;
            case COL_PARAM: x = I.param[i]; break;
            default: x = (I.fwd[i] + I.bwd_in[i]) + I.bwd_w[i]; break;  // total_flops
        }
        col_s[i] = x;
    }
    __syncthreads();
    const size_t N2 = (size_t)(n + 1) * (n + 1);
    double* out = I.S + col * N2;
    for (int a = threadIdx.x; a < n; a += blockDim.x) {
        NeumaierSum sm;
        sm.start(col_s[a]);
        out[s_idx(n, a, a + 1)] = sm.value();
        int b = a + 2;
        for (; b + 3 <= n; b += 4) {  // shared-memory loads of 4 steps issued together
            const double x0 = col_s[b - 1], x1 = col_s[b], x2 = col_s[b + 1], x3 = col_s[b + 2];
            sm.add(x0); out[s_idx(n, a, b)] = sm.value();
            sm.add(x1); out[s_idx(n, a, b + 1)] = sm.value();
            sm.add(x2); out[s_idx(n, a, b + 2)] = sm.value();
            sm.add(x3); out[s_idx(n, a, b + 3)] = sm.value();
        }
        for (; b <= n; ++b) {
            sm.add(col_s[b - 1]);
            out[s_idx(n, a, b)] = sm.value();
        }
    }
}

// ---- K1b: per-group constants ---------------------------------------------------
__device__ __forceinline__ double block_min128(double v, double* red) {
    // exact min over a 128-thread block (min is order-independent)
    for (int off = 16; off > 0; off >>= 1) {
        double o = __shfl_down_sync(0xffffffffu, v, off);
        v = o < v ? o : v;
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = red[w] < r ? red[w] : r;
    return r;
}

// TP memory threshold of one member: the largest non-NaN double P with
// !(((P * rf) * cf) > mem), i.e. the member accepts a stage of parameter sum
// P iff !(P > threshold).  Rounding is monotone, so for 0 < rf, cf < inf the
// accepted set is a down-set of the doubles and its top is found exactly:
// start from mem / (rf * cf) (a few ulps off) and step ulp by ulp to the
// boundary; a bisection over the ordered bit patterns covers what the walk
// cannot (non-finite estimate, > 64 steps).  *ok = false where the monotone
// argument does not apply (the caller keeps the member loop).
static __device__ __noinline__ double tp_threshold_bisect(double rf, double cf, double mem) {
    auto key = [](double d) -> unsigned long long {
        const unsigned long long u = (unsigned long long)__double_as_longlong(d);
        return (u >> 63) ? ~u : (u | (1ull << 63));
    };
    auto unkey = [](unsigned long long k) -> double {
        const unsigned long long u = (k >> 63) ? (k & ~(1ull << 63)) : ~k;
        return __longlong_as_double((long long)u);
    };
    auto accept = [&](double P) { return !(((P * rf) * cf) > mem); };
    unsigned long long lo = key(-INFINITY), hi = key(INFINITY);  // accept(lo), !accept(hi)
    while (hi - lo > 1ull) {
        const unsigned long long mid = lo + (hi - lo) / 2ull;
        if (accept(unkey(mid))) lo = mid; else hi = mid;
    }
    return unkey(lo);
}

static __device__ double tp_threshold(double rf, double cf, double mem, bool* ok) {
    *ok = rf > 0.0 && rf < INFINITY && cf > 0.0 && cf < INFINITY;
    if (!*ok) return 0.0;
    auto accept = [&](double P) { return !(((P * rf) * cf) > mem); };
    if (accept(INFINITY)) return INFINITY;
    if (!accept(-INFINITY)) { *ok = false; return 0.0; }
    double P = mem / (rf * cf);
    if (isfinite(P)) {
        for (int it = 0; it < 64; ++it) {
            if (!accept(P)) {
                P = nextafter(P, -INFINITY);
            } else {
                const double up = nextafter(P, INFINITY);
                if (!accept(up)) return P;
                P = up;
            }
        }
    }
    return tp_threshold_bisect(rf, cf, mem);
}

// one 128-thread block per group: members loaded in parallel into shared
// memory; the TP grid factorisation (split_asymmetric_tp_dp,
// src/planner.py:116-154) checks each candidate shape with every thread
// (one isclose per thread, block AND) and divides the fractions in parallel;
// only the short Neumaier sums run on one thread.  Ends with the packed
// K1Grp record phase 2 reads.
static __device__ void k1_group_block(const DevInst& I, int f) {
    __shared__ double caps[GP_MAX_MEMBERS];
    __shared__ double memv[GP_MAX_MEMBERS];
    __shared__ double red[4];
    __shared__ int shp[64];
    __shared__ int ns_sh;
    __shared__ double sums[2];
    const int m0 = I.fg_off[f], m1 = I.fg_off[f + 1];
    const int nmem = m1 - m0;
    const int s0 = I.fg_sg_off[f], s1 = I.fg_sg_off[f + 1];
    double mn = INFINITY;
    for (int j = threadIdx.x; j < nmem; j += blockDim.x) {
        const int d = I.fg_mem[m0 + j];
        caps[j] = I.p_c[d];
        const double mm = I.mem[d];
        memv[j] = mm;
        mn = mm < mn ? mm : mn;
    }
    mn = block_min128(mn, red);  // (synchronises: caps visible)
    if (threadIdx.x == 0) {
        I.g_minmem[f] = mn;
        // candidate shapes (r, n/r), r in [2, n), stably sorted by |r - c|
        int ns = 0;
        for (int r = 2; r < nmem && ns < 64; ++r)
            if (nmem % r == 0 && nmem / r >= 2) shp[ns++] = r;
        for (int i = 1; i < ns; ++i) {
            int r = shp[i], j = i - 1;
            int key = r - nmem / r; key = key < 0 ? -key : key;
            while (j >= 0) {
                int kj = shp[j] - nmem / shp[j]; kj = kj < 0 ? -kj : kj;
                if (kj <= key) break;
                shp[j + 1] = shp[j];
                --j;
            }
            shp[j + 1] = r;
        }
        ns_sh = ns;
    }
    if (threadIdx.x == 32 && s1 > s0) gpd::dp_fractions(I.sg_cap + s0, s1 - s0, I.g_dp + s0);
    __syncthreads();
    bool tp_ok = false;
    double thr = INFINITY;
    bool thr_ok = true;
    for (int q = 0; q < ns_sh; ++q) {
        const int r = shp[q], c = nmem / r;
        bool ok = true;
        for (int t = threadIdx.x; t < r * c; t += blockDim.x) {
            const int i = t / c, j = t % c;
            ok = ok && gpd::py_isclose(caps[j * r + i] * caps[0], caps[i] * caps[j * r], 1e-9);
        }
        if (!__syncthreads_and(ok)) continue;
        if (threadIdx.x == 0) {  // rows = grid[i][0] = caps[i]; cols = grid[0][j] = caps[j*r]
            NeumaierSum rs, cs;
            rs.start(caps[0]);
            for (int i = 1; i < r; ++i) rs.add(caps[i]);
            cs.start(caps[0]);
            for (int j = 1; j < c; ++j) cs.add(caps[j * r]);
            sums[0] = rs.value();
            sums[1] = cs.value();
        }
        __syncthreads();
        for (int kk = threadIdx.x; kk < nmem; kk += blockDim.x) {
            const double rf = caps[kk % r] / sums[0], cf = caps[(kk / r) * r] / sums[1];
            I.g_rf[m0 + kk] = rf;
            I.g_cf[m0 + kk] = cf;
            bool okx;
            const double tx = tp_threshold(rf, cf, memv[kk], &okx);
            thr_ok = thr_ok && okx;
            thr = tx < thr ? tx : thr;
        }
        tp_ok = true;
        break;
    }
    if (tp_ok) {  // (block-uniform)
        thr = block_min128(thr, red);
        thr_ok = __syncthreads_and(thr_ok) != 0;
    }
    if (threadIdx.x == 0) I.g_tp_ok[f] = tp_ok ? 1 : 0;
    // second-level minimum memories: one warp per second-level group
    __shared__ double sgmin_s[4];
    {
        const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int g = s0 + w; g < s1; g += (int)(blockDim.x >> 5)) {
            const int x0 = I.sg_off[g], x1 = I.sg_off[g + 1];
            double sm = INFINITY;
            for (int x = x0 + lane; x < x1; x += 32) {
                const double mm = I.mem[I.sg_mem[x]];
                sm = mm < sm ? mm : sm;
            }
            for (int off = 16; off > 0; off >>= 1) {
                const double o = __shfl_down_sync(0xffffffffu, sm, off);
                sm = o < sm ? o : sm;
            }
            if (lane == 0) {
                const double v = x1 > x0 ? sm : 0.0;
                I.sg_minmem[g] = v;
                if (g - s0 < 4) sgmin_s[g - s0] = v;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double sgmin[4] = {0.0, 0.0, 0.0, 0.0};
        uint8_t sgne = 0;
        for (int j = 0; j < 4 && j < s1 - s0; ++j) {
            sgmin[j] = sgmin_s[j];
            if (I.sg_off[s0 + j + 1] > I.sg_off[s0 + j]) sgne |= (uint8_t)(1u << j);
        }
        K1Grp R;
        R.cap = I.fg_cap[f];
        R.mbw = 0.0;  // (bandwidth-dependent: phase 2 reads I.fg_minbw)
        R.minmem = mn;
        R.tp_thr = thr;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            R.sgcap[j] = j < s1 - s0 ? I.sg_cap[s0 + j] : 0.0;
            R.sgmin[j] = sgmin[j];
        }
        R.nmem = nmem;
        R.s0 = s0;
        R.nsg = s1 - s0;
        R.has = 0;
        R.tp_ok = tp_ok ? 1 : 0;
        R.thr_ok = tp_ok && thr_ok ? 1 : 0;
        R.sgne = sgne;
        R.fast = s1 - s0 <= 2 ? 1 : 0;
        R.pad[0] = R.pad[1] = R.pad[2] = 0;
        I.grp[f] = R;
    }
}

// recompute min_intra_bandwidth over member pairs (bandwidth snapshots;
// src/grouping.py:69-75 on the rebuilt topology)
static __global__ void k1_minbw(DevInst I, double* out) {
    int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= I.F) return;
    int m0 = I.fg_off[f], m1 = I.fg_off[f + 1];
    double mn = 0.0;
    bool have = false;
    for (int x = m0; x < m1; ++x)
        for (int y = x + 1; y < m1; ++y) {
            double w = I.bw[(size_t)I.fg_mem[x] * I.D + I.fg_mem[y]];
            if (!have || w < mn) mn = w;
            have = true;
        }
    out[f] = have ? mn : 0.0;
}

// split choice for one (group, layer range): choose_intra_split
// (src/planner.py:157-200).  Writes PP shares when kind == ASYM_PP.
static __device__ __noinline__ int choose_split(const DevInst& I, int f, int a, int b, int* shares,
                                         int* nparts) {
    int nmem = I.fg_off[f + 1] - I.fg_off[f];
    int s0 = I.fg_sg_off[f], nsg = I.fg_sg_off[f + 1] - s0;
    *nparts = 0;
    if (nmem == 1 || nsg == 1) return GP_UNIFORM;
    const double* caps = I.sg_cap + s0;
    int nl = b - a;
    if (nsg <= nl && gpd::proportional_split(nl, caps, nsg, 1, shares)) {
        double times[GP_MAX_SGS];
        int pos = a;
        for (int j = 0; j < nsg; ++j) {
            times[j] = Ssum(I, COL_TF, pos, pos + shares[j]) / caps[j];
            pos += shares[j];
        }
        double mean = gpd::psum(times, nsg) / (double)nsg;
        double mx = times[0];
        for (int j = 1; j < nsg; ++j) mx = times[j] > mx ? times[j] : mx;
        if (mx <= I.bf * mean) { *nparts = nsg; return GP_ASYM_PP; }
    }
    if (I.g_tp_ok[f]) { *nparts = nmem; return GP_ASYM_TP_DP; }
    *nparts = nsg;
    return GP_ASYM_DP;
}

// ---- K1c: stage table, generic path ---------------------------------------------
// Generic stage entry (any number of second-level groups): the reference
// order step by step, reading group data from global memory.
static __device__ __noinline__ void k1_stage_generic(const DevInst& I, int f, int a, int b, size_t e) {
#if defined(GP_TIMELINE)
    const unsigned long long tt0 = tl_now();
#endif
    const int n = I.n;
    const size_t N2 = (size_t)(n + 1) * (n + 1);
    int shares[GP_MAX_SGS], np;
    int kind = choose_split(I, f, a, b, shares, &np);
#if defined(GP_TIMELINE)
    const unsigned long long ttw = tl_now();
#endif
    I.skind[e] = (uint8_t)kind;
    I.sshare0[e] = kind == GP_ASYM_PP ? (uint8_t)shares[0] : (uint8_t)0;
    double P = Ssum(I, COL_PARAM, a, b);
    int m0 = I.fg_off[f], m1 = I.fg_off[f + 1];
    int s0 = I.fg_sg_off[f];
    // memory feasibility: bytes_needed > memory_bytes -> infeasible
    // (no early exit: the loads of every member / part are independent, so
    // they overlap instead of forming a chain of dependent round trips)
    bool feas = true;
    if (kind == GP_ASYM_PP) {
        int pos = a;
        for (int j = 0; j < np; ++j) {
            double sub = Ssum(I, COL_PARAM, pos, pos + shares[j]);
            if (I.sg_off[s0 + j + 1] > I.sg_off[s0 + j]) feas = feas & !(sub > I.sg_minmem[s0 + j]);
            pos += shares[j];
        }
    } else if (kind == GP_ASYM_TP_DP) {
        for (int x = m0; x < m1; ++x)
            feas = feas & !(((P * I.g_rf[x]) * I.g_cf[x]) > I.mem[I.fg_mem[x]]);
    } else {
        feas = !(P > I.g_minmem[f]);
    }
    // effective_capacity (src/timing.py:116-143)
    uint8_t code = SC_OK;
    double cap;
    if (kind == GP_ASYM_PP) {
        double tot = Ssum(I, COL_TF, a, b);
        bool have = false;
        double best = 0.0;
        int pos = a;
        for (int j = 0; j < np; ++j) {
            double sub = Ssum(I, COL_TF, pos, pos + shares[j]);
            pos += shares[j];
            double frac = sub / tot;
            if (frac > 0) {
                double val = I.sg_cap[s0 + j] / frac;
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
    // per-sample times (src/timing.py:198-200) and C1 (src/costmodel.py:59)
    double Fp = Ssum(I, COL_FWD, a, b) / cap;
    double Bp = Ssum(I, COL_BWD, a, b) / cap;
    double Wp = Ssum(I, COL_WGT, a, b) / cap;
    double c1 = (Fp + Bp) + Wp;
    I.C1[e] = c1;
    // collective + sync rule (src/timing.py:146-173)
    int nmem = m1 - m0;
    bool has = I.fg_has_minbw[f] != 0;
    double mbw = I.fg_minbw[f];
    // StageTiming.sync_seconds = intra_group_seconds(params, fg) (src/timing.py:195)
    double sync = (P == 0.0 || !has) ? 0.0 : (mbw > 0 ? P / mbw : NAN);
    I.fbws[e] = make_double4(Fp, Bp, Wp, sync);
    if (code == SC_OK && has && !(mbw > 0) && (nmem >= 2 || P != 0.0)) code = SC_TOPOLOGY;
    bool overflow = false;
    for (int mi = 0; mi < I.nm; ++mi) {
        double md = (double)I.micro[mi];
        double al = 0.0;
        if (nmem >= 2) {
            double V = 2.0 * P;
            if (kind == GP_ASYM_TP_DP) V = V + I.act[b - 1] * md;
            if (V != 0.0 && has && mbw > 0) al = V / mbw;
        }
        double cm = c1 * md;
        if (feas && isinf(cm)) overflow = true;
        I.vtab[((size_t)mi * I.F + f) * ((size_t)n * (n + 1) / 2) + (a * n - a * (a - 1) / 2) + (b - a - 1)] =
            nmem >= 2 ? (kind == GP_ASYM_TP_DP ? 2.0 * P + I.act[b - 1] * md : 2.0 * P) : 0.0;
        double2 v = make_double2(feas ? cm : INFINITY, al);
        I.stg[(size_t)mi * I.F * N2 + e] = v;
        size_t ntri = (size_t)n * (n + 1) / 2;
        I.tpk[((size_t)mi * I.F + f) * ntri + (a * n - a * (a - 1) / 2) + (b - a - 1)] = v;
        if (b == n) I.tcol[((size_t)mi * I.F + f) * (n + 1) + a] = v;
    }
    I.scode[e] = feas ? code : SC_INFEASIBLE;
    if (feas && code != SC_OK) atomicOr(I.flags, FLAG_STAGE_ERROR);
    if (overflow) atomicOr(I.flags, FLAG_OVERFLOW);
#if defined(GP_TIMELINE)
    {   // per-thread record: kid 22, blk = f<<16 | a<<8 | b, pad = split kind
        const unsigned long long tt1 = tl_now();
        unsigned int _i = atomicAdd(&g_tl_n, 1u);
        if (_i < GP_TL_CAP)
            g_tl[_i] = TlRec{tt0, ttw, tt1, 22u, (unsigned)((f << 16) | (a << 8) | b), 0u,
                             (unsigned)kind};
    }
#endif
}

// proportional_split (src/planner.py:65-87) for exactly two parts with
// minimum = 1, in registers: the stable sort by (-rem, index) is one compare.
// Returns 1 ok, 0 where the reference raises InfeasibleSplitError, -1 when
// an operand is not finite (the caller takes the generic path).
__device__ __forceinline__ int prop_split2(int total, double w0, double w1, int& s0, int& s1) {
    NeumaierSum ws;
    ws.start(w0);
    ws.add(w1);
    const double wsum = ws.value();
    const double raw0 = ((double)total * w0) / wsum, raw1 = ((double)total * w1) / wsum;
    const double fl0 = floor(raw0), fl1 = floor(raw1);
    if (!(isfinite(raw0) && isfinite(raw1) && fl0 >= 0.0 && fl1 >= 0.0 && fl0 < 1e9 && fl1 < 1e9))
        return -1;
    s0 = (int)fl0;
    s1 = (int)fl1;
    const double k0 = -(raw0 - fl0), k1 = -(raw1 - fl1);  // sort keys -rem
    const long long leftover = (long long)total - ((long long)s0 + s1);
    const long long take = leftover >= 0 ? (leftover < 2 ? leftover : 2)
                                         : (2 + leftover > 0 ? 2 + leftover : 0);
    const int rank0 = k1 < k0 ? 1 : 0, rank1 = k0 <= k1 ? 1 : 0;  // (ties: index order)
    s0 += rank0 < take ? 1 : 0;
    s1 += rank1 < take ? 1 : 0;
    // donation loop (shares are >= 0, so at most one move per part)
    if (s0 < 1) {
        if (s1 > s0) { if (s1 <= 1) return 0; s1 -= 1; s0 += 1; }
        else return 0;  // donor = part 0 itself with share 0 <= minimum
    }
    if (s1 < 1) {
        if (s0 >= s1) { if (s0 <= 1) return 0; s0 -= 1; s1 += 1; }
        else { return 0; }
    }
    return 1;
}

// ---- K1c: stage table -------------------------------------------------------------
// One thread per (group, a, b).  memory_feasible is local to a stage because
// every group appears in exactly one stage (src/planner.py:226-253).  The
// register path issues every independent load up front (group record, the
// five interval sums, the micro-batch sizes), keeps the split in registers
// and stores last, so a thread waits on two round trips instead of a chain of
// dependent ones; the arithmetic is the generic path's, operation by operation.
static __device__ void k1_stage_t(const DevInst& I, long long t, const double* md_s) {
    const int n = I.n;
    const int N1 = n + 1, NN = N1 * N1;
    if (t >= (long long)I.F * NN) return;
    const int f = (int)(t / NN);
    const int rem = (int)(t - (long long)f * NN);
    const int a = rem / N1, b = rem - a * N1;
    const size_t N2 = (size_t)NN;
    const size_t e = (size_t)f * N2 + rem;
    if (a >= b) {
        I.scode[e] = SC_INFEASIBLE;
        I.skind[e] = 0;
        I.sshare0[e] = 0;
        I.C1[e] = INFINITY;
        I.fbws[e] = make_double4(NAN, NAN, NAN, NAN);
        for (int mi = 0; mi < I.nm; ++mi) {
            I.stg[(size_t)mi * I.F * N2 + e] = make_double2(INFINITY, 0.0);
            if (a == n && b == n) I.tcol[((size_t)mi * I.F + f) * (n + 1) + n] = make_double2(INFINITY, 0.0);
        }
        return;
    }
    const K1Grp g = I.grp[f];
    if (!g.fast || md_s == nullptr) { k1_stage_generic(I, f, a, b, e); return; }
#if defined(GP_TIMELINE)
    const unsigned long long tt0 = tl_now();
#endif
    const double* __restrict__ S = I.S;
    const int si = s_idx(n, a, b);
    const double sF = S[COL_FWD * N2 + si], sB = S[COL_BWD * N2 + si], sW = S[COL_WGT * N2 + si];
    const double sP = S[COL_PARAM * N2 + si], sT = S[COL_TF * N2 + si];
    const double act_b = I.act[b - 1];
    const double mbw = I.fg_minbw[f];
    const bool has = I.fg_has_minbw[f] != 0;
    // choose_intra_split (src/planner.py:157-200)
    const int nmem = g.nmem;
    int kind, sh0 = 0, sh1 = 0;
    double subT0 = 0.0, subT1 = 0.0, subP0 = 0.0, subP1 = 0.0;
    bool pp = false;
    if (nmem == 1 || g.nsg == 1) {
        kind = GP_UNIFORM;
    } else {
        if (b - a >= 2) {
            const int ps = prop_split2(b - a, g.sgcap[0], g.sgcap[1], sh0, sh1);
            if (ps < 0) { k1_stage_generic(I, f, a, b, e); return; }
            if (ps == 1) {
                const int q0 = s_idx(n, a, a + sh0), q1 = s_idx(n, a + sh0, a + sh0 + sh1);
                subT0 = S[COL_TF * N2 + q0];
                subT1 = S[COL_TF * N2 + q1];
                subP0 = S[COL_PARAM * N2 + q0];
                subP1 = S[COL_PARAM * N2 + q1];
                const double t0 = subT0 / g.sgcap[0], t1 = subT1 / g.sgcap[1];
                NeumaierSum ts;
                ts.start(t0);
                ts.add(t1);
                const double mean = ts.value() / 2.0;
                const double mx = t1 > t0 ? t1 : t0;
                pp = mx <= I.bf * mean;
            }
        }
        kind = pp ? GP_ASYM_PP : (g.tp_ok ? GP_ASYM_TP_DP : GP_ASYM_DP);
    }
    // memory_feasible (src/planner.py:226-253)
    bool feas;
    if (kind == GP_ASYM_PP) {
        feas = !((g.sgne & 1) && subP0 > g.sgmin[0]) && !((g.sgne & 2) && subP1 > g.sgmin[1]);
    } else if (kind == GP_ASYM_TP_DP) {
        if (g.thr_ok) {
            feas = !(sP > g.tp_thr);
        } else {
            feas = true;
            const int m0 = I.fg_off[f];
            for (int x = m0; x < m0 + nmem; ++x)
                feas = feas & !(((sP * I.g_rf[x]) * I.g_cf[x]) > I.mem[I.fg_mem[x]]);
        }
    } else {
        feas = !(sP > g.minmem);
    }
    // effective_capacity (src/timing.py:116-143)
    uint8_t code = SC_OK;
    double cap;
    if (kind == GP_ASYM_PP) {
        const double fr0 = subT0 / sT, fr1 = subT1 / sT;
        bool hv = false;
        double best = 0.0;
        if (fr0 > 0) { best = g.sgcap[0] / fr0; hv = true; }
        if (fr1 > 0) { const double v1 = g.sgcap[1] / fr1; if (!hv || v1 < best) best = v1; hv = true; }
        cap = best;
        if (!hv) code = SC_DEGENERATE;
    } else {
        cap = g.cap;
        if (!(cap > 0)) code = SC_DEGENERATE;
    }
    const double Fp = sF / cap, Bp = sB / cap, Wp = sW / cap;
    const double c1 = (Fp + Bp) + Wp;
    const double sync = (sP == 0.0 || !has) ? 0.0 : (mbw > 0 ? sP / mbw : NAN);
    if (code == SC_OK && has && !(mbw > 0) && (nmem >= 2 || sP != 0.0)) code = SC_TOPOLOGY;
#if defined(GP_TIMELINE)
    const unsigned long long ttw = tl_now();
#endif
    I.skind[e] = (uint8_t)kind;
    I.sshare0[e] = pp ? (uint8_t)sh0 : (uint8_t)0;
    I.C1[e] = c1;
    I.fbws[e] = make_double4(Fp, Bp, Wp, sync);
    const size_t ntri = (size_t)n * (n + 1) / 2;
    const size_t pk = (size_t)(a * n - a * (a - 1) / 2) + (b - a - 1);
    bool overflow = false;
#pragma unroll 1
    for (int mi = 0; mi < I.nm; ++mi) {
        const double md = md_s[mi];
        double al = 0.0;
        double V = 0.0;
        if (nmem >= 2) {
            V = 2.0 * sP;
            if (kind == GP_ASYM_TP_DP) V = V + act_b * md;
            if (V != 0.0 && has && mbw > 0) al = V / mbw;
        }
        const double cm = c1 * md;
        if (feas && isinf(cm)) overflow = true;
        I.vtab[((size_t)mi * I.F + f) * ntri + pk] = V;
        const double2 v = make_double2(feas ? cm : INFINITY, al);
        I.stg[(size_t)mi * I.F * N2 + e] = v;
        I.tpk[((size_t)mi * I.F + f) * ntri + pk] = v;
        if (b == n) I.tcol[((size_t)mi * I.F + f) * (n + 1) + a] = v;
    }
    I.scode[e] = feas ? code : SC_INFEASIBLE;
    if (feas && code != SC_OK) atomicOr(I.flags, FLAG_STAGE_ERROR);
    if (overflow) atomicOr(I.flags, FLAG_OVERFLOW);
#if defined(GP_TIMELINE)
    {
        const unsigned long long tt1 = tl_now();
        unsigned int _i = atomicAdd(&g_tl_n, 1u);
        if (_i < GP_TL_CAP)
            g_tl[_i] = TlRec{tt0, ttw, tt1, 23u, (unsigned)((f << 16) | (a << 8) | b), 0u,
                             (unsigned)kind};
    }
#endif
}

// ---- K1d: gateways and boundary transfer table -------------------------------------
// gateway_link (src/timing.py:104-113): argmin over (p_t, u, v) with string
// order of ids, u in the upstream group, v in the downstream group.
static __device__ void k1_gateway_warp(const DevInst& I, int warp, int lane) {
    // one warp per ordered pair (fa, fb); lanes scan member pairs, then a
    // warp argmin on the key (p_t, rank(u), rank(v))
    const int fa = warp / I.F, fb = warp % I.F;
    const int a0 = I.fg_off[fa], na = I.fg_off[fa + 1] - a0;
    const int b0 = I.fg_off[fb], nbm = I.fg_off[fb + 1] - b0;
    bool have = false;
    double bp = 0.0;
    unsigned int bu = 0, bv = 0, ru = 0xffffffffu, rv = 0xffffffffu;
#pragma unroll 8
    for (int t = lane; t < na * nbm; t += 32) {  // unrolled: the member / p_t loads overlap
        const unsigned int u = I.fg_mem[a0 + t / nbm], v = I.fg_mem[b0 + t % nbm];
        const double p = I.p_t[(size_t)u * I.D + v];
        const unsigned int qu = I.id_rank[u], qv = I.id_rank[v];
        bool less = !have || p < bp || (p == bp && (qu < ru || (qu == ru && qv < rv)));
        if (less) { have = true; bp = p; bu = u; bv = v; ru = qu; rv = qv; }
    }
    for (int off = 16; off > 0; off >>= 1) {
        const bool oh = __shfl_down_sync(0xffffffffu, have, off);
        const double op = __shfl_down_sync(0xffffffffu, bp, off);
        const unsigned int ou = __shfl_down_sync(0xffffffffu, bu, off);
        const unsigned int ov = __shfl_down_sync(0xffffffffu, bv, off);
        const unsigned int oru = __shfl_down_sync(0xffffffffu, ru, off);
        const unsigned int orv = __shfl_down_sync(0xffffffffu, rv, off);
        bool take = oh && (!have || op < bp || (op == bp && (oru < ru || (oru == ru && orv < rv))));
        if (take) { have = true; bp = op; bu = ou; bv = ov; ru = oru; rv = orv; }
    }
    // (a zero-bandwidth gateway raises FLAG_GATEWAY_ERROR in k1_boundary_t,
    // so phase 1 never touches the flags word it resets)
    if (lane == 0) I.gw[warp] = (int)(bu * I.D + bv);
}

static __global__ void k1_gateways(DevInst I) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (warp < I.F * I.F) k1_gateway_warp(I, warp, threadIdx.x & 31);
}

// K1 phase 1 in one launch: blocks [0,5) interval sums, [5, 5+F) group
// constants, the rest gateways (one warp per ordered group pair)
__device__ void k1_intervals_block(const DevInst& I, int col);
__device__ void k1_gateway_warp(const DevInst& I, int warp, int lane);

// gp_replan graph head: instance arena host -> device by loads from the
// mapped pinned staging buffer (16 B per thread, grid-stride)
static __global__ void k_arena_pull(const uint4* __restrict__ src, uint4* __restrict__ dst,
                             unsigned long long n16) {
    TL_START();
    pdl_trigger();
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
         i += (unsigned long long)gridDim.x * blockDim.x)
        dst[i] = src[i];
    TL_STOP(5);
}

// Per-run scratch that the gp_replan graph resets inside phase 1 instead of
// with memset nodes (null pointers: nothing to reset).
struct K1Reset {
    unsigned long long* err_idx;  // first erroring candidate -> ~0
    unsigned int* item_ctr;       // K3 sweep per-item task counters -> 0
    unsigned int n_items;
};

static __global__ void __launch_bounds__(128) k1_phase1(DevInst I, K1Reset R) {
    const int b = blockIdx.x;
    TL_START();
    pdl_trigger();  // phase 2 may be scheduled now (it waits for this grid)
    pdl_wait();     // the instance arena (k_arena_pull in the gp_replan graph)
    TL_WAITED();
    if (b == (int)gridDim.x - 1) {  // (a gateway block: the shortest role)
        if (threadIdx.x == 0) {
            *I.flags = 0u;
            if (R.err_idx) *R.err_idx = ~0ull;
        }
        for (unsigned int t = threadIdx.x; R.item_ctr && t < R.n_items; t += blockDim.x)
            R.item_ctr[t] = 0u;
        // M = batch / micro per (b, m) index, for the per-candidate kernels
        for (int t = threadIdx.x; t < I.nb * I.nm; t += blockDim.x)
            I.mtab[t] = (double)(I.batch[t / I.nm] / I.micro[t % I.nm]);
    }
    if (b < 5) k1_intervals_block(I, b);
    else if (b < 5 + I.F) k1_group_block(I, b - 5);
    else {
        const int warp = (b - 5 - I.F) * 4 + (threadIdx.x >> 5);
        if (warp < I.F * I.F) k1_gateway_warp(I, warp, threadIdx.x & 31);
    }
#if defined(GP_TIMELINE)
    __syncthreads();
    TL_STOP(b < 5 ? 10 : (b < 5 + I.F ? 11 : 12));  // intervals / groups / gateways
#endif
}

static __device__ void k1_boundary_t(const DevInst& I, long long t) {
    long long total = (long long)I.nm * I.F * I.F * I.n;
    if (t >= total) return;
    int j = (int)(t % I.n);
    long long r = t / I.n;
    int pair = (int)(r % (I.F * I.F));
    int mi = (int)(r / (I.F * I.F));
    int g = I.gw[pair];
    if (mi == 0 && j == 0) {
        const bool bad = !(I.bw[g] > 0);
        I.gwbad[pair] = bad ? 1 : 0;
        if (bad && pair / I.F != pair % I.F) atomicOr(I.flags, FLAG_GATEWAY_ERROR);  // zero-bandwidth gateway
    }
    double md = (double)I.micro[mi];
    // transfer_seconds: latency + (act*m)/bandwidth (src/timing.py:91-97)
    I.xt[(size_t)r * I.nxp + j] = I.lat[g] + (I.act[j] * md) / I.bw[g];
}

// K1 phase 2 in one launch: stage table entries, then boundary x entries
static __global__ void k1_phase2(DevInst I, long long n_stage) {
    TL_START();
    pdl_trigger();
    pdl_wait();  // phase 1's interval sums, group constants and gateways
    TL_WAITED();
    __shared__ double md_s[16];  // (double)micro[mi] for the register path
    if (threadIdx.x < 16 && threadIdx.x < I.nm) md_s[threadIdx.x] = (double)I.micro[threadIdx.x];
    __syncthreads();
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_stage) k1_stage_t(I, t, I.nm <= 16 ? md_s : nullptr);
    else k1_boundary_t(I, t - n_stage);
#if defined(GP_TIMELINE)
    __syncthreads();
    TL_STOP(blockIdx.x * blockDim.x < n_stage ? 20 : 21);  // stage / boundary blocks
#endif
}

