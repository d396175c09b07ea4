// k1_tables.cuh - K1: per-load table build (interval sums, group constants, stage and boundary tables).
#pragma once
#include "common.cuh"

// ---- K1a: interval sums -----------------------------------------------------
// sum(model.layers[i].<field> for i in range(a, b)) for every 0 <= a < b <= n,
// each interval summed from its own start (never prefix differences).
__device__ void k1_intervals_block(const DevInst& I, int col) {
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
        for (int b = a + 2; b <= n; ++b) {
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

// one 128-thread block per group: members loaded in parallel into shared
// memory; the TP grid factorisation (split_asymmetric_tp_dp,
// src/planner.py:116-154) checks each candidate shape with every thread
// (one isclose per thread, block AND) and divides the fractions in parallel;
// only the short Neumaier sums run on one thread.
__device__ void k1_group_block(const DevInst& I, int f) {
    __shared__ double caps[GP_MAX_MEMBERS];
    __shared__ double red[4];
    __shared__ int shp[64];
    __shared__ int ns_sh;
    __shared__ double sums[2];
    const int m0 = I.fg_off[f], m1 = I.fg_off[f + 1];
    const int nmem = m1 - m0;
    double mn = INFINITY;
    for (int j = threadIdx.x; j < nmem; j += blockDim.x) {
        const int d = I.fg_mem[m0 + j];
        caps[j] = I.p_c[d];
        const double mm = I.mem[d];
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
        const int s0 = I.fg_sg_off[f], s1 = I.fg_sg_off[f + 1];
        if (s1 > s0) gpd::dp_fractions(I.sg_cap + s0, s1 - s0, I.g_dp + s0);
    }
    __syncthreads();
    bool tp_ok = false;
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
            I.g_rf[m0 + kk] = caps[kk % r] / sums[0];
            I.g_cf[m0 + kk] = caps[(kk / r) * r] / sums[1];
        }
        tp_ok = true;
        break;
    }
    if (threadIdx.x == 0) I.g_tp_ok[f] = tp_ok ? 1 : 0;
    const int s0 = I.fg_sg_off[f], s1 = I.fg_sg_off[f + 1];
    for (int g = s0; g < s1; ++g) {
        double sm = INFINITY;
        for (int x = I.sg_off[g] + threadIdx.x; x < (int)I.sg_off[g + 1]; x += blockDim.x) {
            const double mm = I.mem[I.sg_mem[x]];
            sm = mm < sm ? mm : sm;
        }
        sm = block_min128(sm, red);
        if (threadIdx.x == 0) I.sg_minmem[g] = I.sg_off[g + 1] > I.sg_off[g] ? sm : 0.0;
    }
}

// recompute min_intra_bandwidth over member pairs (bandwidth snapshots;
// src/grouping.py:69-75 on the rebuilt topology)
__global__ void k1_minbw(DevInst I, double* out) {
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
__device__ int choose_split(const DevInst& I, int f, int a, int b, int* shares, int* nparts) {
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

// ---- K1c: stage table -------------------------------------------------------------
// One thread per (group, a, b).  memory_feasible is local to a stage because
// every group appears in exactly one stage (src/planner.py:226-253).
__device__ void k1_stage_t(const DevInst& I, long long t) {
#if defined(GP_TIMELINE)
    const unsigned long long tt0 = tl_now();
#endif
    int n = I.n;
    int N1 = n + 1;
    long long total = (long long)I.F * N1 * N1;
    if (t >= total) return;
    int f = (int)(t / (N1 * N1));
    int rem = (int)(t % (N1 * N1));
    int a = rem / N1, b = rem % N1;
    size_t N2 = (size_t)N1 * N1;
    size_t e = (size_t)f * N2 + rem;
    if (a >= b) {
        I.scode[e] = SC_INFEASIBLE;
        I.skind[e] = 0;
        I.C1[e] = INFINITY;
        I.fbws[e] = make_double4(NAN, NAN, NAN, NAN);
        for (int mi = 0; mi < I.nm; ++mi) {
            I.stg[(size_t)mi * I.F * N2 + e] = make_double2(INFINITY, 0.0);
            if (a == n && b == n) I.tcol[((size_t)mi * I.F + f) * (n + 1) + n] = make_double2(INFINITY, 0.0);
        }
        return;
    }
    int shares[GP_MAX_SGS], np;
    int kind = choose_split(I, f, a, b, shares, &np);
#if defined(GP_TIMELINE)
    const unsigned long long ttw = tl_now();
#endif
    I.skind[e] = (uint8_t)kind;
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

// ---- K1d: gateways and boundary transfer table -------------------------------------
// gateway_link (src/timing.py:104-113): argmin over (p_t, u, v) with string
// order of ids, u in the upstream group, v in the downstream group.
__device__ void k1_gateway_warp(const DevInst& I, int warp, int lane) {
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

__global__ void k1_gateways(DevInst I) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (warp < I.F * I.F) k1_gateway_warp(I, warp, threadIdx.x & 31);
}

// K1 phase 1 in one launch: blocks [0,5) interval sums, [5, 5+F) group
// constants, the rest gateways (one warp per ordered group pair)
__device__ void k1_intervals_block(const DevInst& I, int col);
__device__ void k1_gateway_warp(const DevInst& I, int warp, int lane);

// gp_replan graph head: instance arena host -> device by loads from the
// mapped pinned staging buffer (16 B per thread, grid-stride)
__global__ void k_arena_pull(const uint4* __restrict__ src, uint4* __restrict__ dst,
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

__global__ void __launch_bounds__(128) k1_phase1(DevInst I, K1Reset R) {
    const int b = blockIdx.x;
    TL_START();
    pdl_trigger();  // phase 2 may be scheduled now (it waits for this grid)
    pdl_wait();     // the instance arena (k_arena_pull in the gp_replan graph)
    TL_WAITED();
    if (b == 0) {
        if (threadIdx.x == 0) {
            *I.flags = 0u;
            if (R.err_idx) *R.err_idx = ~0ull;
        }
        for (unsigned int t = threadIdx.x; R.item_ctr && t < R.n_items; t += blockDim.x)
            R.item_ctr[t] = 0u;
    }
    if (b == 0)  // M = batch / micro per (b, m) index, for the per-candidate kernels
        for (int t = threadIdx.x; t < I.nb * I.nm; t += blockDim.x)
            I.mtab[t] = (double)(I.batch[t / I.nm] / I.micro[t % I.nm]);
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

__device__ void k1_boundary_t(const DevInst& I, long long t) {
    long long total = (long long)I.nm * I.F * I.F * I.n;
    if (t >= total) return;
    int j = (int)(t % I.n);
    long long r = t / I.n;
    int pair = (int)(r % (I.F * I.F));
    int mi = (int)(r / (I.F * I.F));
    int g = I.gw[pair];
    if (mi == 0 && j == 0 && pair / I.F != pair % I.F && !(I.bw[g] > 0))
        atomicOr(I.flags, FLAG_GATEWAY_ERROR);  // zero-bandwidth gateway
    double md = (double)I.micro[mi];
    // transfer_seconds: latency + (act*m)/bandwidth (src/timing.py:91-97)
    I.xt[(size_t)r * I.nxp + j] = I.lat[g] + (I.act[j] * md) / I.bw[g];
}

// K1 phase 2 in one launch: stage table entries, then boundary x entries
__global__ void k1_phase2(DevInst I, long long n_stage) {
    TL_START();
    pdl_trigger();
    pdl_wait();  // phase 1's interval sums, group constants and gateways
    TL_WAITED();
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_stage) k1_stage_t(I, t);
    else k1_boundary_t(I, t - n_stage);
#if defined(GP_TIMELINE)
    __syncthreads();
    TL_STOP(blockIdx.x * blockDim.x < n_stage ? 20 : 21);  // stage / boundary blocks
#endif
}

