// engine.cu - B200 (sm_100a) plan-evaluation engine behind the C-ABI of
// include/geopipe_b200.h.
//
// Data path:
//   gp_ctx_load    H2D of the packed instance, then K1:
//                    k1_intervals  Neumaier interval sums S[col][a][b]
//                    k1_groups     per-group TP tiles, DP fractions, memory minima
//                    k1_stages     per (group, a, b): split choice, memory
//                                  feasibility, capacity, C1 = (F+Bi)+W, and per m
//                                  the table {C1*m | +inf, AL}
//                    k1_boundary   gateway pair per ordered group pair and
//                                  x = lat + (act*m)/bw per boundary layer
//   gp_eval_batch  K2: one thread per explicit candidate
//   gp_argmin_range K3: one CTA per (b,m, order, comp-chunk); the varying last
//                  cut sweeps a shared-memory triangle of the stage table;
//                  warp-shuffle + CTA + last-block argmin on the reference key
//
// Every floating-point operation mirrors the reference operation order
// (src/costmodel.py:56-89, src/timing.py:116-231, src/planner.py:157-253);
// the file is compiled with -fmad=false.  There is no CPU fallback.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/geopipe_b200.h"
#include "device_math.cuh"

using gpd::NeumaierSum;

// ----------------------------------------------------------------------------
// error plumbing
// ----------------------------------------------------------------------------
static thread_local char g_err[512] = "";

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

#define CUDA_TRY(expr)                                                        \
    do {                                                                      \
        cudaError_t e_ = (expr);                                              \
        if (e_ != cudaSuccess)                                                \
            return fail(GP_ERR_CUDA, "%s: %s (%s:%d)", #expr,                 \
                        cudaGetErrorString(e_), __FILE__, __LINE__);          \
    } while (0)

// stage-table codes (per group, layer range)
enum : uint8_t { SC_OK = 0, SC_INFEASIBLE = 1, SC_DEGENERATE = 4, SC_TOPOLOGY = 5 };
// context flags that force the generic (status-tracking) range kernel
enum : uint32_t { FLAG_STAGE_ERROR = 1, FLAG_OVERFLOW = 2, FLAG_GATEWAY_ERROR = 4 };
#define K3_THREADS 256
#define K3_TILE 256
#define K3_SEG 32
#ifndef K3S_THREADS
#define K3S_THREADS 256
#endif
#ifndef K3S_MINB
#define K3S_MINB 2
#endif
#ifndef K3_MINB
#define K3_MINB 3
#endif
#define BINOM_ROWS 257

// ----------------------------------------------------------------------------
// device-side view of one loaded instance
// ----------------------------------------------------------------------------
struct DevInst {
    int n;          // layers
    int F;          // first-level groups
    int D;          // devices
    int nb, nm;     // |B|, |M|
    const double *fwd, *bwd_in, *bwd_w, *act, *param;
    const long long *batch, *micro;
    const double *p_c, *mem, *p_t, *lat, *bw;
    const uint32_t* id_rank;
    const uint32_t *fg_off, *fg_mem, *fg_sg_off, *sg_off, *sg_mem;
    const double *fg_cap, *sg_cap;
    const double* fg_minbw;      // current min_intra_bandwidth
    const uint8_t* fg_has_minbw;
    double bf;                   // bottleneck_factor
    // K1 outputs
    double* S;                   // [5][(n+1)^2]: fwd, bwd_in, bwd_w, param, total_flops
    uint8_t* g_tp_ok;            // [F]
    double *g_rf, *g_cf;         // [fg member slots]
    double* g_dp;                // [sg slots]
    double* g_minmem;            // [F]
    double* sg_minmem;           // [n_sgs]
    double2* stg;                // [nm][F][(n+1)^2] {C1*m or +inf, AL}
    uint8_t* scode;              // [F][(n+1)^2]
    uint8_t* skind;              // [F][(n+1)^2]
    double* C1;                  // [F][(n+1)^2] per-sample (F+Bi)+W (detail)
    double4* fbws;               // [F][(n+1)^2] {F, Bi, W per sample, sync seconds} (K5)
    double* vtab;                // [nm][F][ntri] collective volume V (0 if no collective) (K6)
    int* gw;                     // [F*F] gateway u*D+v
    double* xt;                  // [nm][F][F][nxp] (rows padded to 16 B)
    int nxp;                     // x row stride: n rounded up to even
    double2* tpk;                // [nm][F][n(n+1)/2] packed rows a: b = a+1..n
    double2* tcol;               // [nm][F][n+1] entry (q, n) at q
    uint32_t* flags;             // [1]
};

__device__ __forceinline__ int tri_idx(int n, int a, int b) { return a * (n + 1) + b; }

enum { COL_FWD = 0, COL_BWD = 1, COL_WGT = 2, COL_PARAM = 3, COL_TF = 4 };

__device__ __forceinline__ double Ssum(const DevInst& I, int col, int a, int b) {
    size_t N2 = (size_t)(I.n + 1) * (I.n + 1);
    return I.S[col * N2 + tri_idx(I.n, a, b)];
}

// ---- K1a: interval sums -----------------------------------------------------
// sum(model.layers[i].<field> for i in range(a, b)) for every 0 <= a < b <= n,
// each interval summed from its own start (never prefix differences).
__device__ void k1_intervals_block(const DevInst& I, int col) {
    // one CTA per column; the column is staged in shared memory so the
    // sequential Neumaier sweeps read on-chip values
    __shared__ double col_s[GP_MAX_LAYERS + 1];
    for (int i = threadIdx.x; i < I.n; i += blockDim.x) {
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
    size_t N2 = (size_t)(I.n + 1) * (I.n + 1);
    double* out = I.S + col * N2;
    for (int a = threadIdx.x; a < I.n; a += blockDim.x) {
        NeumaierSum sm;
        for (int b = a + 1; b <= I.n; ++b) {
            if (b == a + 1) sm.start(col_s[b - 1]); else sm.add(col_s[b - 1]);
            out[tri_idx(I.n, a, b)] = sm.value();
        }
    }
}

__global__ void k1_intervals(DevInst I) { k1_intervals_block(I, blockIdx.x); }

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
// memory, then the (sequential) factorisation runs on-chip
__device__ void k1_group_block(const DevInst& I, int f) {
    __shared__ double caps[GP_MAX_MEMBERS];
    __shared__ double red[4];
    const int m0 = I.fg_off[f], m1 = I.fg_off[f + 1];
    const int nmem = m1 - m0;
    double mn = INFINITY;
    for (int j = threadIdx.x; j < nmem; j += blockDim.x) {
        const int d = I.fg_mem[m0 + j];
        caps[j] = I.p_c[d];
        const double mm = I.mem[d];
        mn = mm < mn ? mm : mn;
    }
    mn = block_min128(mn, red);
    if (threadIdx.x == 0) {
        I.g_minmem[f] = mn;
        I.g_tp_ok[f] = gpd::tp_grid(caps, nmem, I.g_rf + m0, I.g_cf + m0) ? 1 : 0;
        const int s0 = I.fg_sg_off[f], s1 = I.fg_sg_off[f + 1];
        if (s1 > s0) gpd::dp_fractions(I.sg_cap + s0, s1 - s0, I.g_dp + s0);
    }
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

__global__ void k1_groups(DevInst I) { k1_group_block(I, blockIdx.x); }

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
    I.skind[e] = (uint8_t)kind;
    double P = Ssum(I, COL_PARAM, a, b);
    int m0 = I.fg_off[f], m1 = I.fg_off[f + 1];
    int s0 = I.fg_sg_off[f];
    // memory feasibility: bytes_needed > memory_bytes -> infeasible
    bool feas = true;
    if (kind == GP_ASYM_PP) {
        int pos = a;
        for (int j = 0; j < np && feas; ++j) {
            double sub = Ssum(I, COL_PARAM, pos, pos + shares[j]);
            if (I.sg_off[s0 + j + 1] > I.sg_off[s0 + j]) feas = !(sub > I.sg_minmem[s0 + j]);
            pos += shares[j];
        }
    } else if (kind == GP_ASYM_TP_DP) {
        for (int x = m0; x < m1 && feas; ++x)
            feas = !(((P * I.g_rf[x]) * I.g_cf[x]) > I.mem[I.fg_mem[x]]);
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
}

__global__ void k1_stages(DevInst I) { k1_stage_t(I, (long long)blockIdx.x * blockDim.x + threadIdx.x); }

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
    for (int t = lane; t < na * nbm; t += 32) {
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
    if (lane == 0) {
        I.gw[warp] = (int)(bu * I.D + bv);
        if (fa != fb && !(I.bw[(size_t)bu * I.D + bv] > 0)) atomicOr(I.flags, FLAG_GATEWAY_ERROR);
    }
}

__global__ void k1_gateways(DevInst I) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (warp < I.F * I.F) k1_gateway_warp(I, warp, threadIdx.x & 31);
}

// K1 phase 1 in one launch: blocks [0,5) interval sums, [5, 5+F) group
// constants, the rest gateways (one warp per ordered group pair)
__device__ void k1_intervals_block(const DevInst& I, int col);
__device__ void k1_gateway_warp(const DevInst& I, int warp, int lane);

__global__ void __launch_bounds__(128) k1_phase1(DevInst I) {
    const int b = blockIdx.x;
    if (b < 5) { k1_intervals_block(I, b); return; }
    if (b < 5 + I.F) { k1_group_block(I, b - 5); return; }
    const int warp = (b - 5 - I.F) * 4 + (threadIdx.x >> 5);
    if (warp < I.F * I.F) k1_gateway_warp(I, warp, threadIdx.x & 31);
}

__device__ void k1_boundary_t(const DevInst& I, long long t);
__global__ void k1_boundary(DevInst I) {
    k1_boundary_t(I, (long long)blockIdx.x * blockDim.x + threadIdx.x);
}
__device__ void k1_boundary_t(const DevInst& I, long long t) {
    long long total = (long long)I.nm * I.F * I.F * I.n;
    if (t >= total) return;
    int j = (int)(t % I.n);
    long long r = t / I.n;
    int pair = (int)(r % (I.F * I.F));
    int mi = (int)(r / (I.F * I.F));
    int g = I.gw[pair];
    double md = (double)I.micro[mi];
    // transfer_seconds: latency + (act*m)/bandwidth (src/timing.py:91-97)
    I.xt[(size_t)r * I.nxp + j] = I.lat[g] + (I.act[j] * md) / I.bw[g];
}

// K1 phase 2 in one launch: stage table entries, then boundary x entries
__global__ void k1_phase2(DevInst I, long long n_stage) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_stage) k1_stage_t(I, t);
    else k1_boundary_t(I, t - n_stage);
}

// ----------------------------------------------------------------------------
// generic evaluation of one candidate from the tables (status-tracking path)
// ----------------------------------------------------------------------------
struct EvalOut {
    double cost;
    int status;
};

// p[0..k] are cut positions (p[0] = 0); order[s] group of stage s.
__device__ EvalOut eval_tables(const DevInst& I, int k, const uint8_t* order, const int* p,
                               int mi, long long M) {
    int n = I.n;
    size_t N2 = (size_t)(n + 1) * (n + 1);
    EvalOut out{0.0, GP_OK};
    bool feas = true;
    for (int s = 0; s < k; ++s)
        if (I.scode[(size_t)order[s] * N2 + tri_idx(n, p[s], p[s + 1])] == SC_INFEASIBLE)
            feas = false;
    if (!feas) { out.cost = INFINITY; return out; }
    if (p[k] != n) { out.status = GP_ERR_TOPOLOGY; return out; }  // src/timing.py:183-186
    for (int s = 0; s < k; ++s) {
        uint8_t c = I.scode[(size_t)order[s] * N2 + tri_idx(n, p[s], p[s + 1])];
        if (c != SC_OK) { out.status = c; return out; }
    }
    for (int s = 0; s + 1 < k; ++s) {
        int g = I.gw[order[s] * I.F + order[s + 1]];
        if (!(I.bw[g] > 0)) { out.status = GP_ERR_TOPOLOGY; return out; }
    }
    const double2* T = I.stg + (size_t)mi * I.F * N2;
    const double* X = I.xt + (size_t)mi * I.F * I.F * I.nxp;
    double Md = (double)M;
    double fill = 0.0, res = 0.0, best = 0.0, xprev = 0.0;
    for (int s = 0; s < k; ++s) {
        double2 e = T[(size_t)order[s] * N2 + tri_idx(n, p[s], p[s + 1])];
        double c = e.x;
        if (s > 0) res = res + gpd::max0(xprev - c);
        double total = ((fill + Md * c) + res) + e.y;
        best = (s == 0 || total > best) ? total : best;
        if (s + 1 < k) {
            double x = X[((size_t)order[s] * I.F + order[s + 1]) * I.nxp + (p[s + 1] - 1)];
            fill = fill + (c + x);
            xprev = x;
        }
    }
    out.cost = best;
    return out;
}

// ---- K2: explicit batch, one thread per candidate -------------------------------
// max(0.0, x) = x > 0 ? x : +0.0 without the FP64 pipe: clear every bit
// when the sign bit is set (-0.0 -> +0.0, negatives -> +0.0).  Exact for
// every non-NaN x (NaN cannot occur: operands are finite or +inf).
__device__ __forceinline__ double max0f(double x) {
    long long b = __double_as_longlong(x);
    return __longlong_as_double(b & ~(b >> 63));
}
// a > b ? a : b (first-max; no NaNs occur)
__device__ __forceinline__ double gtsel(double a, double b) {
    double r;
    asm("{\n\t.reg .pred p;\n\tsetp.gt.f64 p, %1, %2;\n\tselp.f64 %0, %1, %2, p;\n\t}"
        : "=d"(r) : "d"(a), "d"(b));
    return r;
}

// Fast per-candidate evaluation when the tables carry no error entries:
// infeasible stages are +inf in the table, so the cost needs only the K stage
// entries and K-1 boundary values - all loads issued before any arithmetic.
template <int K>
__device__ __forceinline__ double eval_fast(const DevInst& I, const uint8_t* o, const int* p,
                                            int mi, double Md) {
    const size_t N2 = (size_t)(I.n + 1) * (I.n + 1);
    const double2* T = I.stg + (size_t)mi * I.F * N2;
    const double* X = I.xt + (size_t)mi * I.F * I.F * I.nxp;
    double2 e[K];
    double x[K];
#pragma unroll
    for (int s = 0; s < K; ++s) {
        e[s] = __ldg(&T[(size_t)o[s] * N2 + tri_idx(I.n, p[s], p[s + 1])]);
        if (s + 1 < K) x[s] = __ldg(&X[((size_t)o[s] * I.F + o[s + 1]) * I.nxp + (p[s + 1] - 1)]);
    }
    double fill = 0.0, res = 0.0, best = 0.0;
#pragma unroll
    for (int s = 0; s < K; ++s) {
        if (s > 0) res = res + max0f(x[s - 1] - e[s].x);
        const double total = ((fill + Md * e[s].x) + res) + e[s].y;
        best = (s == 0 || total > best) ? total : best;
        if (s + 1 < K) fill = fill + (e[s].x + x[s]);
    }
    return best;
}

__global__ void k2_eval_batch(DevInst I, int k, long long ncand, const uint8_t* __restrict__ order,
                              const uint8_t* __restrict__ counts, const uint8_t* __restrict__ bm,
                              double* __restrict__ cost, uint8_t* __restrict__ status) {
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
    if (st != GP_OK) { cost[i] = NAN; status[i] = (uint8_t)st; return; }
    int mi = b % I.nm;
    long long M = I.batch[b / I.nm] / I.micro[mi];
    if (*I.flags == 0u && p[k] == I.n && k >= 2 && k <= 6) {
        const double Md = (double)M;
        double c;
        switch (k) {
            case 2: c = eval_fast<2>(I, o, p, mi, Md); break;
            case 3: c = eval_fast<3>(I, o, p, mi, Md); break;
            case 4: c = eval_fast<4>(I, o, p, mi, Md); break;
            case 5: c = eval_fast<5>(I, o, p, mi, Md); break;
            default: c = eval_fast<6>(I, o, p, mi, Md); break;
        }
        cost[i] = c;
        status[i] = GP_OK;
        return;
    }
    EvalOut r = eval_tables(I, k, o, p, mi, M);
    cost[i] = r.status == GP_OK ? r.cost : NAN;
    status[i] = (uint8_t)r.status;
}

// ----------------------------------------------------------------------------
// K3: exhaustive argmin over an enumeration-index range
// ----------------------------------------------------------------------------
struct RangeGeom {
    int k;
    int nbm;                 // |B| * |M|
    unsigned long long NC;   // C(n-1, k-1)
    unsigned long long NP;   // k!
    unsigned long long lo, hi;
    unsigned long long item0;          // first item touched
    unsigned long long chunks_per_item;  // CTAs sharing one item
    unsigned long long chunk;          // (generic kernel: unused)
    unsigned int* item_ctr;            // per-item tile counters (zeroed per launch)
    const uint8_t* tiles;              // cut positions at every K3_TILE-th rank, or null
    int items_mode;                    // generic kernel: [lo, hi) indexes (b, item, comp)
    unsigned long long it_lo, it_span; // item range of items_mode
    int nm;                            // |M| (items_mode decode)
};

__device__ unsigned long long d_binom(int n, int r) {
    if (r < 0 || r > n) return 0ull;
    unsigned long long res = 1;
    for (int i = 1; i <= r; ++i) res = res * (unsigned long long)(n - r + i) / (unsigned long long)i;
    return res;
}

__device__ void d_unrank_perm(int k, unsigned long long r, uint8_t* perm) {
    uint8_t pool[GP_MAX_STAGES];
    unsigned long long f = 1;
    for (int i = 0; i < k; ++i) { pool[i] = (uint8_t)i; if (i > 0) f *= (unsigned long long)i; }
    int left = k;
    for (int i = 0; i < k; ++i) {
        // f = (k-1-i)!
        unsigned long long q = r / f;
        r %= f;
        perm[i] = pool[q];
        for (int j = (int)q; j + 1 < left; ++j) pool[j] = pool[j + 1];
        --left;
        if (k - 1 - i > 0) f /= (unsigned long long)(k - 1 - i);
    }
}

// composition rank -> cut positions p[1..k-1] (lexicographic in counts)
__device__ void d_unrank_cuts(int n, int k, unsigned long long r, int* p) {
    p[0] = 0;
    int prev = 0;
    for (int j = 1; j < k; ++j) {
        for (int q = prev + 1;; ++q) {
            unsigned long long cnt = d_binom(n - q - 1, k - 1 - j);
            if (r < cnt) { p[j] = q; prev = q; break; }
            r -= cnt;
        }
    }
    p[k] = n;
}

struct Key {
    double cost;
    unsigned long long tie;
};

__device__ __forceinline__ bool key_less(const Key& a, const Key& b) {
    return a.cost < b.cost || (a.cost == b.cost && a.tie < b.tie);
}

__device__ __forceinline__ Key warp_min(Key v) {
    for (int off = 16; off > 0; off >>= 1) {
        Key o;
        o.cost = __shfl_down_sync(0xffffffffu, v.cost, off);
        o.tie = __shfl_down_sync(0xffffffffu, v.tie, off);
        if (key_less(o, v)) v = o;
    }
    return v;
}

struct ArgminScratch {
    Key* blk;                 // [grid]
    unsigned int* counter;    // [1]
    Key* result;              // [1]
    int* err;                 // [1] first error (index<<4|code) low 32 bits unused
    unsigned long long* err_idx;
};

// CTA-wide reduction of per-thread keys, then last-block grid reduction.
// Reduction over a group of `nblk` CTAs (the whole grid, or one snapshot's
// CTAs): CTA `bidx` of the group writes its key; the last one to finish
// reduces the group's keys into *S.result and re-arms the counter.
__device__ void block_argmin_finish(Key mine, const ArgminScratch& S, unsigned int nblk,
                                    unsigned int bidx) {
    __shared__ Key wbest[32];
    __shared__ bool last;
    Key w = warp_min(mine);
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) wbest[wid] = w;
    __syncthreads();
    if (wid == 0) {
        int nw = (blockDim.x + 31) >> 5;
        Key v = lane < nw ? wbest[lane] : Key{INFINITY, ~0ull};
        v = warp_min(v);
        if (lane == 0) {
            S.blk[bidx] = v;
            __threadfence();
            unsigned int done = atomicAdd(S.counter, 1u);
            last = (done == nblk - 1);
        }
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    Key v{INFINITY, ~0ull};
    for (unsigned int b = threadIdx.x; b < nblk; b += blockDim.x) {
        Key o;
        o.cost = __ldcg(&S.blk[b].cost);
        o.tie = __ldcg(&S.blk[b].tie);
        if (key_less(o, v)) v = o;
    }
    v = warp_min(v);
    if (lane == 0) wbest[wid] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        int nw = (blockDim.x + 31) >> 5;
        Key r = wbest[0];
        for (int i = 1; i < nw; ++i) if (key_less(wbest[i], r)) r = wbest[i];
        *S.result = r;
        *S.counter = 0;  // re-arm for the next launch
    }
}

__device__ __forceinline__ void block_argmin_finish(Key mine, const ArgminScratch& S) {
    block_argmin_finish(mine, S, gridDim.x, blockIdx.x);
}

// Fast path (all stage entries error-free, k >= 3).
//
// CTA = (item, chunk) with item = (bm, order); its comp ranks are split into
// contiguous per-warp ranges and each warp sweeps its range in windows of 32
// consecutive ranks (lane j takes rank r0 + j), so all lanes run the same
// instruction stream.  A candidate = prefix cuts p[1..k-3] (stages 0..k-4,
// folded once into per-lane scalars and refreshed only when a lane crosses
// into the next prefix) plus the pair (a, q) = (p[k-2], p[k-1]) that bounds
// the last three stages:
//     stage k-3 = [p[k-3], a)   table T1 = {C1*m, AL} of group order[k-3]
//     stage k-2 = [a, q)        table T2 of group order[k-2]
//     stage k-1 = [q, n)        column of group order[k-1]
// MODE 2: T1 and T2 triangles, the column and both boundary rows in shared
// memory; MODE 1: T1 from L1/L2; MODE 0: everything from L1/L2.
__device__ __forceinline__ int rowoff(int n, int a) { return a * n - a * (a - 1) / 2; }

// lexicographic successor of the prefix cuts p[1..k-3] (p_j <= n - k + j)
__device__ __forceinline__ bool next_prefix(int* p, int n, int k) {
    int j = k - 3;
    while (j >= 1 && p[j] >= n - k + j) --j;
    if (j < 1) return false;
    ++p[j];
    for (int t = j + 1; t <= k - 3; ++t) p[t] = p[t - 1] + 1;
    return true;
}

// advance (prefix, a, q) by s ranks; returns false past the last pair
__device__ __forceinline__ bool advance_pair(int* p, int& a, int& q, int s, int n, int k,
                                             bool& dirty) {
    q += s;
    while (q > n - 1) {
        int o = q - (n - 1);
        ++a;
        if (a > n - 2) {
            if (k < 4 || !next_prefix(p, n, k)) return false;
            a = p[k - 3] + 1;
            dirty = true;
        }
        q = a + o;
    }
    return true;
}



// ---- TMA (bulk async copy) helpers ----------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(smem_u32(bar)), "r"(phase) : "memory");
}

// CTA group = item = (micro-batch index mi, order); chunks_per_item CTAs
// share an item and pull K3_TILE-rank tiles of its composition space from a
// per-item atomic counter (dynamic balance across warps and CTAs).  Every
// candidate (order, cuts, m) is evaluated for all NB batch sizes at once:
// the tables {C1*m, AL} and x depend on m only, and the fill / residual
// chains do not depend on the batch size, so only the M*c terms and the
// totals are per batch (tie order (cost, order, cuts, b) is kept by
// scanning batch sizes innermost).
//
// Staging: one elected thread moves the packed stage-table triangles, the
// last-stage column, stage 0's row and the boundary rows HBM/L2 -> shared
// memory with bulk async copies (TMA, cp.async.bulk) on one mbarrier.
template <int MODE, int NB>
__global__ void __launch_bounds__(K3_THREADS, K3_MINB) k3_argmin(DevInst I, RangeGeom G, ArgminScratch S,
                                                           const unsigned long long* __restrict__ binom,
                                                           const uint32_t* skip_if_flags) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = I.n, k = G.k;
    const int ntri = n * (n + 1) / 2;
    const int KB = k + 1;  // binomial sub-table columns r = 0..k
    const unsigned long long islot = blockIdx.x / G.chunks_per_item;
    const unsigned long long item = G.item0 + islot;  // mi * NP + perm
    const int mi = (int)(item / G.NP);
    const unsigned long long perm_rank = item % G.NP;
    // per-batch clip of [0, NC) against [lo, hi)
    unsigned long long blo[NB], bhi[NB];
    unsigned long long u_lo = ~0ull, u_hi = 0;
    bool all_in = true;
#pragma unroll
    for (int bi = 0; bi < NB; ++bi) {
        unsigned long long base = (((unsigned long long)bi * I.nm + mi) * G.NP + perm_rank) * G.NC;
        unsigned long long l = 0, h = G.NC;
        if (base + l < G.lo) l = G.lo - base < h ? G.lo - base : h;
        if (base + h > G.hi) h = G.hi > base + l ? G.hi - base : l;
        blo[bi] = l;
        bhi[bi] = h;
        if (l != 0 || h != G.NC) all_in = false;
        if (l < h) { u_lo = l < u_lo ? l : u_lo; u_hi = h > u_hi ? h : u_hi; }
    }
    if (skip_if_flags && *skip_if_flags) u_hi = 0;  // tables carry errors: generic kernel decides
    uint8_t order[GP_MAX_STAGES];
    d_unrank_perm(k, perm_rank, order);
    double Mv[NB];
#pragma unroll
    for (int bi = 0; bi < NB; ++bi) Mv[bi] = (double)(I.batch[bi] / I.micro[mi]);
    const size_t N2 = (size_t)(n + 1) * (n + 1);
    const double2* T = I.stg + (size_t)mi * I.F * N2;
    const double* X = I.xt + (size_t)mi * I.F * I.F * I.nxp;
    const int f1 = order[k - 3], f2 = order[k - 2], f3 = order[k - 1];
    const double2* P0 = I.tpk + ((size_t)mi * I.F + order[0]) * ntri;  // row 0 = first n
    const double2* P1 = I.tpk + ((size_t)mi * I.F + f1) * ntri;
    const double2* P2 = I.tpk + ((size_t)mi * I.F + f2) * ntri;
    const double2* C3 = I.tcol + ((size_t)mi * I.F + f3) * (n + 1);
    const double* X01 = X + ((size_t)order[0] * I.F + order[1]) * I.nxp;
    const double* X12 = X + ((size_t)f1 * I.F + f2) * I.nxp;
    const double* X23 = X + ((size_t)f2 * I.F + f3) * I.nxp;

    // shared: mbarrier | binom | T2 | col | x12 | x23 | row0 | x01 | T1
    uint64_t* bar = (uint64_t*)smem_raw;
    unsigned long long* bn = (unsigned long long*)(smem_raw + 16);
    unsigned char* tail = smem_raw + 16 + (((size_t)(n + 1) * KB * 8 + 15) & ~(size_t)15);
    double2* tri2 = (double2*)tail;
    double2* col3 = tri2 + (MODE >= 1 ? ntri : 0);
    double* x12s = (double*)(col3 + (MODE >= 1 ? n + 1 : 0));
    double* x23s = x12s + (MODE >= 1 ? I.nxp : 0);
    double2* row0 = (double2*)(x23s + (MODE >= 1 ? I.nxp : 0));
    double* x01s = (double*)(row0 + (MODE >= 1 ? n : 0));
    double2* tri1 = (double2*)(x01s + (MODE >= 1 ? I.nxp : 0));
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        if (MODE >= 1) {
            uint32_t bytes = (uint32_t)(ntri * 16 + (n + 1) * 16 + 3 * I.nxp * 8 + n * 16) +
                             (MODE == 2 ? (uint32_t)ntri * 16 : 0u);
            mbar_expect_tx(bar, bytes);
            tma_bulk_g2s(tri2, P2, (uint32_t)ntri * 16, bar);
            tma_bulk_g2s(col3, C3, (uint32_t)(n + 1) * 16, bar);
            tma_bulk_g2s(x12s, X12, (uint32_t)I.nxp * 8, bar);
            tma_bulk_g2s(x23s, X23, (uint32_t)I.nxp * 8, bar);
            tma_bulk_g2s(row0, P0, (uint32_t)n * 16, bar);
            tma_bulk_g2s(x01s, X01, (uint32_t)I.nxp * 8, bar);
            if (MODE == 2) tma_bulk_g2s(tri1, P1, (uint32_t)ntri * 16, bar);
        }
    }
    for (int t = threadIdx.x; t < (n + 1) * KB; t += blockDim.x)
        bn[t] = binom[(t / KB) * (GP_MAX_STAGES + 1) + (t % KB)];
    __syncthreads();
    if (MODE >= 1) mbar_wait(bar, 0);

    Key mine{INFINITY, ~0ull};
    const int lane = threadIdx.x & 31;
    double best_c = INFINITY;
    unsigned long long best_t = ~0ull;  // rank * NB + bi
    if (u_lo < u_hi) {
        const unsigned long long tile_lo = u_lo / K3_TILE;
        const unsigned long long ntiles = (u_hi + K3_TILE - 1) / K3_TILE - tile_lo;
        int p[GP_MAX_STAGES + 1];
        p[0] = 0;
        for (;;) {
            unsigned int t = 0;
            if (lane == 0) t = atomicAdd(&G.item_ctr[islot], 1u);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= ntiles) break;
            const unsigned long long rank0 = (tile_lo + t) * K3_TILE;
            // cut positions of rank0: precomputed tile table or ballot decode
            if (G.tiles) {
                const uint8_t* tp = G.tiles + (rank0 / K3_TILE) * 16;
                for (int j = 1; j < k; ++j) p[j] = tp[j - 1];
            } else {
                // for cut j pick the smallest q with C(n-q-1, r+1) <
                // C(n-lo, r+1) - rem (hockey stick), 32 candidates per ballot
                unsigned long long rem = rank0;
                int prev = 0;
                for (int j = 1; j < k; ++j) {
                    const int r = k - 1 - j, lo = prev + 1;
                    const unsigned long long tot = bn[(n - lo) * KB + r + 1];
                    const unsigned long long thr = tot - rem;
                    int qsel = -1;
                    for (int base = lo; qsel < 0; base += 32) {
                        int qq = base + lane;
                        bool ok = qq <= n - 1 - r && bn[(n - qq - 1) * KB + r + 1] < thr;
                        unsigned m = __ballot_sync(0xffffffffu, ok);
                        if (m) qsel = base + __ffs(m) - 1;
                    }
                    rem -= tot - bn[(n - qsel) * KB + r + 1];
                    p[j] = qsel;
                    prev = qsel;
                }
            }
            int a = p[k - 2], q = p[k - 1];
            bool dirty = true;
            const int tlen = (int)((rank0 + K3_TILE <= u_hi ? K3_TILE : u_hi - rank0));
            int rl = lane;  // rank within the tile
            bool live = rl < tlen && advance_pair(p, a, q, lane, n, k, dirty);
            double fill = 0.0, res = 0.0, xprev = 0.0;
            double mx[NB];
            int base1 = 0, base2 = 0, a_cached = -1;
            while (__any_sync(0xffffffffu, live)) {
                if (live) {
                    if (dirty) {
                        dirty = false;
                        fill = 0.0; res = 0.0; xprev = 0.0;
#pragma unroll
                        for (int bi = 0; bi < NB; ++bi) mx[bi] = -INFINITY;
                        for (int s = 0; s + 3 < k; ++s) {
                            double2 e;
                            double x;
                            if (MODE >= 1 && s == 0) {
                                e = row0[p[1] - 1];
                                x = x01s[p[1] - 1];
                            } else {
                                e = __ldg(&T[(size_t)order[s] * N2 + tri_idx(n, p[s], p[s + 1])]);
                                x = __ldg(&X[((size_t)order[s] * I.F + order[s + 1]) * I.nxp + (p[s + 1] - 1)]);
                            }
                            if (s > 0) res = res + max0f(xprev - e.x);
#pragma unroll
                            for (int bi = 0; bi < NB; ++bi) {
                                double tot = ((fill + Mv[bi] * e.x) + res) + e.y;
                                mx[bi] = (s == 0) ? tot : gtsel(tot, mx[bi]);
                            }
                            fill = fill + (e.x + x);
                            xprev = x;
                        }
                        const int pk3 = p[k - 3];
                        base1 = rowoff(n, pk3) - pk3 - 1;
                        a_cached = -1;
                    }
                    if (a != a_cached) {
                        a_cached = a;
                        base2 = rowoff(n, a) - a - 1;
                    }
                    double2 e1, e2, e3;
                    double x1, x2;
                    if (MODE == 2) e1 = tri1[base1 + a];
                    else e1 = __ldg(&P1[base1 + a]);
                    if (MODE >= 1) {
                        e2 = tri2[base2 + q];
                        e3 = col3[q];
                        x1 = x12s[a - 1];
                        x2 = x23s[q - 1];
                    } else {
                        e2 = __ldg(&P2[base2 + q]);
                        e3 = __ldg(&C3[q]);
                        x1 = __ldg(&X12[a - 1]);
                        x2 = __ldg(&X23[q - 1]);
                    }
                    // batch-independent chains (src/costmodel.py:68-81)
                    const double res1 = (k > 3) ? res + max0f(xprev - e1.x) : res;
                    const double fill2 = fill + (e1.x + x1);
                    const double res2 = res1 + max0f(x1 - e2.x);
                    const double fill3 = fill2 + (e2.x + x2);
                    const double res3 = res2 + max0f(x2 - e3.x);
                    const unsigned long long rabs = rank0 + rl;
#pragma unroll
                    for (int bi = 0; bi < NB; ++bi) {
                        if (!all_in && (rabs < blo[bi] || rabs >= bhi[bi])) continue;
                        double t1 = ((fill + Mv[bi] * e1.x) + res1) + e1.y;
                        double t2 = ((fill2 + Mv[bi] * e2.x) + res2) + e2.y;
                        double t3 = ((fill3 + Mv[bi] * e3.x) + res3) + e3.y;
                        double c = (k > 3) ? gtsel(t1, mx[bi]) : t1;
                        c = gtsel(t2, c);
                        c = gtsel(t3, c);
                        unsigned long long tk = rabs * NB + bi;
                        if (c < best_c || (c == best_c && tk < best_t)) { best_c = c; best_t = tk; }
                    }
                    rl += 32;
                    live = rl < tlen && advance_pair(p, a, q, 32, n, k, dirty);
                }
            }
        }
    }
    if (best_t != ~0ull) {
        unsigned long long rr = best_t / NB, bi = best_t % NB;
        mine.cost = best_c;
        mine.tie = ((perm_rank * G.NC) + rr) * (unsigned long long)G.nbm +
                   (unsigned long long)(bi * I.nm + mi);
    }
    block_argmin_finish(mine, S);
}

// ---------------------------------------------------------------------------
// K3 sweep (full items): the candidates of one (m, order) item are grouped
// into RUNS = (prefix cuts p[1..k-3], a = p[k-2], a segment of <= K3_SEG
// consecutive last cuts q).  A lane owns a run: the stages fixed by the run
// (0..k-3) are folded once into per-lane scalars, then the lane walks q.
// Runs are ordered by length (all full K3_SEG runs first, then the partial
// ones grouped by length) so the 32 lanes of a warp walk in lock step, and
// lanes of equal a read the same shared-memory row (broadcast).
// A run group = {first run id, a | len << 16, rows, segs_per_row}; the run
// id -> (group, prefix row, segment) map is a binary search in smem.
// ---------------------------------------------------------------------------
struct SweepGeom {
    int k, nbm;
    unsigned long long NC, NP;
    unsigned long long item0;       // first (mi * NP + perm) item
    unsigned long long cpi;         // CTAs per item
    unsigned int W;                 // runs per item
    int ngroups;
    const uint4* groups;            // [ngroups]
    unsigned int* item_ctr;         // per-item task counters
    const uint8_t* prefixes;        // colex-ordered (k-3)-subsets, 16-byte records
    int gsteps;                     // largest power of two <= ngroups
    // snapshot batches (K6): tables and results per snapshot
    unsigned int items;             // items per snapshot in this launch
    const double2* tpk;             // packed triangles of snapshot 0
    const double2* tcol;
    const double* xt;
    unsigned long long s_tpk, s_tcol, s_xt;  // per-snapshot strides (elements)
    const unsigned long long* bnk;  // C(nn, r), nn <= n, r <= k: contiguous [n+1][k+1]
};

template <int MODE, int NB>
__global__ void __launch_bounds__(K3S_THREADS, K3S_MINB) k3_sweep(DevInst I, SweepGeom G, ArgminScratch S,
                                                          const unsigned long long* __restrict__ binom,
                                                          const uint32_t* skip_if_flags) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = I.n, k = G.k;
    const int ntri = n * (n + 1) / 2;
    const int KB = k + 1;
    const unsigned int per_snap = G.items * (unsigned int)G.cpi;
    const unsigned int snap = blockIdx.x / per_snap, local = blockIdx.x % per_snap;
    const unsigned long long islot = local / G.cpi;
    const unsigned long long item = G.item0 + islot;
    const int mi = (int)(item / G.NP);
    const unsigned long long perm_rank = item % G.NP;
    uint8_t order[GP_MAX_STAGES];
    d_unrank_perm(k, perm_rank, order);
    double Mv[NB];
#pragma unroll
    for (int bi = 0; bi < NB; ++bi) Mv[bi] = (double)(I.batch[bi] / I.micro[mi]);
    const double2* TPm = G.tpk + snap * G.s_tpk + (size_t)mi * I.F * ntri;
    const double* X = G.xt + snap * G.s_xt + (size_t)mi * I.F * I.F * I.nxp;
    const int f1 = order[k - 3], f2 = order[k - 2], f3 = order[k - 1];
    const double2* P0 = TPm + (size_t)order[0] * ntri;
    const double2* P1 = TPm + (size_t)f1 * ntri;
    const double2* P2 = TPm + (size_t)f2 * ntri;
    const double2* C3 = G.tcol + snap * G.s_tcol + ((size_t)mi * I.F + f3) * (n + 1);
    const double* X01 = X + ((size_t)order[0] * I.F + order[1]) * I.nxp;
    const double* X12 = X + ((size_t)f1 * I.F + f2) * I.nxp;
    const double* X23 = X + ((size_t)f2 * I.F + f3) * I.nxp;

    // shared: mbarrier | binom | groups | T2 | col | x12 | x23 | row0 | x01 | T1
    uint64_t* bar = (uint64_t*)smem_raw;
    unsigned long long* bn = (unsigned long long*)(smem_raw + 16);
    uint4* grp = (uint4*)(smem_raw + 16 + (((size_t)(n + 1) * KB * 8 + 15) & ~(size_t)15));
    unsigned char* tail = (unsigned char*)(grp + G.ngroups);
    double2* tri2 = (double2*)tail;
    double2* col3 = tri2 + (MODE >= 1 ? ntri : 0);
    double* x12s = (double*)(col3 + (MODE >= 1 ? n + 1 : 0));
    double* x23s = x12s + (MODE >= 1 ? I.nxp : 0);
    double2* row0 = (double2*)(x23s + (MODE >= 1 ? I.nxp : 0));
    double* x01s = (double*)(row0 + (MODE >= 1 ? n : 0));
    double2* tri1 = (double2*)(x01s + (MODE >= 1 ? I.nxp : 0));
    if (threadIdx.x == 0) {
        // every table this CTA reads arrives by bulk async copy on one mbarrier
        const uint32_t bn_bytes = (uint32_t)(((size_t)(n + 1) * KB * 8 + 15) & ~(size_t)15);
        uint32_t bytes = bn_bytes + (uint32_t)G.ngroups * 16;
        if (MODE >= 1)
            bytes += (uint32_t)(ntri * 16 + (n + 1) * 16 + 3 * I.nxp * 8 + n * 16) +
                     (MODE == 2 ? (uint32_t)ntri * 16 : 0u);
        mbar_init(bar, 1);
        mbar_expect_tx(bar, bytes);
        tma_bulk_g2s(bn, G.bnk, bn_bytes, bar);
        tma_bulk_g2s(grp, G.groups, (uint32_t)G.ngroups * 16, bar);
        if (MODE >= 1) {
            tma_bulk_g2s(tri2, P2, (uint32_t)ntri * 16, bar);
            tma_bulk_g2s(col3, C3, (uint32_t)(n + 1) * 16, bar);
            tma_bulk_g2s(x12s, X12, (uint32_t)I.nxp * 8, bar);
            tma_bulk_g2s(x23s, X23, (uint32_t)I.nxp * 8, bar);
            tma_bulk_g2s(row0, P0, (uint32_t)n * 16, bar);
            tma_bulk_g2s(x01s, X01, (uint32_t)I.nxp * 8, bar);
            if (MODE == 2) tma_bulk_g2s(tri1, P1, (uint32_t)ntri * 16, bar);
        }
    }
    __syncthreads();
    mbar_wait(bar, 0);

    const int lane = threadIdx.x & 31;
    double best_c = INFINITY;
    unsigned long long best_t = ~0ull;  // R * NB + bi
    const bool skip = skip_if_flags && skip_if_flags[snap];  // generic kernel decides
    unsigned int* const ctr = &G.item_ctr[(size_t)snap * G.items + islot];
    unsigned int t_next = 0;
    if (lane == 0 && !skip) t_next = atomicAdd(ctr, 1u);
    for (; !skip;) {
        const unsigned int t = __shfl_sync(0xffffffffu, t_next, 0);
        if ((unsigned long long)t * 32 >= G.W) break;
        if (lane == 0) t_next = atomicAdd(ctr, 1u);  // next task, latency hidden by this one
        const unsigned int u = t * 32 + lane;
        int len = 0, a = 0, q0 = 0;
        double fill2 = 0.0, res1 = 0.0, x1 = 0.0;
        double mx1[NB];
        unsigned long long rpre = 0;  // comp rank of (prefix, a, q = a + 1)
        if (u < G.W) {
            // run id -> group (fixed-trip binary search), prefix row, segment
            int gi = 0;
            for (int step = G.gsteps; step > 0; step >>= 1) {
                int mid = gi + step;
                if (mid < G.ngroups && grp[mid].x <= u) gi = mid;
            }
            const uint4 g = grp[gi];
            const unsigned int local = u - g.x;
            a = (int)(g.y & 0xffffu);
            len = (int)(g.y >> 16);
            unsigned int row;
            if (g.w) { row = local / g.w; q0 = a + 1 + (int)(local % g.w) * K3_SEG; }
            else { row = local; q0 = n - len; }
            // prefix cuts p[1..k-3]: colex row `row` (subsets of [1, a-1] come first)
            int p[GP_MAX_STAGES + 1];
            p[0] = 0;
            if (k > 3) {
                const uint8_t* pr = G.prefixes + (size_t)row * 16;
                for (int j = 1; j <= k - 3; ++j) p[j] = pr[j - 1];
            }
            p[k - 2] = a;
            // rank prefix: sum_j C(n - p[j-1] - 1, k - j) - C(n - p[j], k - j), j <= k-2
            for (int j = 1; j <= k - 2; ++j)
                rpre += bn[(n - p[j - 1] - 1) * KB + (k - j)] - bn[(n - p[j]) * KB + (k - j)];
            // stages 0..k-4 (fixed by the prefix)
            double fill = 0.0, res = 0.0, xprev = 0.0;
            double mx[NB];
#pragma unroll
            for (int bi = 0; bi < NB; ++bi) mx[bi] = -INFINITY;
            for (int s = 0; s + 3 < k; ++s) {
                double2 e;
                double x;
                if (MODE >= 1 && s == 0) {
                    e = row0[p[1] - 1];
                    x = x01s[p[1] - 1];
                } else {
                    e = __ldg(&TPm[(size_t)order[s] * ntri + rowoff(n, p[s]) + (p[s + 1] - p[s] - 1)]);
                    x = __ldg(&X[((size_t)order[s] * I.F + order[s + 1]) * I.nxp + (p[s + 1] - 1)]);
                }
                if (s > 0) res = res + max0f(xprev - e.x);
#pragma unroll
                for (int bi = 0; bi < NB; ++bi) {
                    double tot = ((fill + Mv[bi] * e.x) + res) + e.y;
                    mx[bi] = (s == 0) ? tot : gtsel(tot, mx[bi]);
                }
                fill = fill + (e.x + x);
                xprev = x;
            }
            // stage k-3 = [p[k-3], a) (fixed by the run)
            const int pk3 = p[k - 3];
            double2 e1 = (MODE == 2) ? tri1[rowoff(n, pk3) - pk3 - 1 + a]
                                     : __ldg(&P1[rowoff(n, pk3) - pk3 - 1 + a]);
            x1 = (MODE >= 1) ? x12s[a - 1] : __ldg(&X12[a - 1]);
            res1 = (k > 3) ? res + max0f(xprev - e1.x) : res;
#pragma unroll
            for (int bi = 0; bi < NB; ++bi) {
                double t1 = ((fill + Mv[bi] * e1.x) + res1) + e1.y;
                mx1[bi] = (k > 3) ? gtsel(t1, mx[bi]) : t1;
            }
            fill2 = fill + (e1.x + x1);
        }
        int lmax = len;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            int o = __shfl_xor_sync(0xffffffffu, lmax, off);
            lmax = o > lmax ? o : lmax;
        }
        // walk q: per-run minimum with strict < (ranks increase with q, and
        // with the batch index inside one q), merged into the lane's best
        // under the full key (cost, rank, batch) when the run ends
        const double2* e2p = (MODE >= 1 ? tri2 : P2) + (rowoff(n, a) - a - 1) + q0;
        const double2* e3p = (MODE >= 1 ? col3 : C3) + q0;
        const double* x2p = (MODE >= 1 ? x23s : X23) + (q0 - 1);
        double run_c = INFINITY;
        int run_i = -1, run_b = 0;
        for (int i = 0; i < lmax; ++i) {
            if (i < len) {
                double2 e2, e3;
                double x2;
                if (MODE >= 1) { e2 = e2p[i]; e3 = e3p[i]; x2 = x2p[i]; }
                else { e2 = __ldg(&e2p[i]); e3 = __ldg(&e3p[i]); x2 = __ldg(&x2p[i]); }
                // stages k-2 = [a, q) and k-1 = [q, n) (src/costmodel.py:68-81)
                const double res2 = res1 + max0f(x1 - e2.x);
                const double fill3 = fill2 + (e2.x + x2);
                const double res3 = res2 + max0f(x2 - e3.x);
                double cmin = INFINITY;
                int bmin = 0;
#pragma unroll
                for (int bi = 0; bi < NB; ++bi) {
                    double t2 = ((fill2 + Mv[bi] * e2.x) + res2) + e2.y;
                    double t3 = ((fill3 + Mv[bi] * e3.x) + res3) + e3.y;
                    double c = gtsel(t2, mx1[bi]);
                    c = gtsel(t3, c);
                    if (bi == 0 || c < cmin) { cmin = c; bmin = bi; }
                }
                if (run_i < 0 || cmin < run_c) { run_c = cmin; run_i = i; run_b = bmin; }
            }
        }
        if (run_i >= 0 && run_c <= best_c) {
            unsigned long long tk = (rpre + (unsigned long long)(q0 + run_i - a - 1)) * NB + run_b;
            if (run_c < best_c || tk < best_t) { best_c = run_c; best_t = tk; }
        }
    }
    Key mine{INFINITY, ~0ull};
    if (best_t != ~0ull) {
        unsigned long long rr = best_t / NB, bi = best_t % NB;
        mine.cost = best_c;
        mine.tie = ((perm_rank * G.NC) + rr) * (unsigned long long)G.nbm +
                   (unsigned long long)(bi * I.nm + mi);
    }
    ArgminScratch Ss = S;
    Ss.blk = S.blk + (size_t)snap * per_snap;
    Ss.counter = S.counter + snap;
    Ss.result = S.result + snap;
    block_argmin_finish(mine, Ss, per_snap, local);
}

// Tile table: cut positions p[1..k-1] (u8) of every K3_TILE-th composition
// rank (16-byte records); depends on (n, k) only.
__global__ void k_tiles(int n, int k, unsigned long long ntiles, uint8_t* out) {
    unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    int p[GP_MAX_STAGES + 1];
    d_unrank_cuts(n, k, t * K3_TILE, p);
    for (int j = 1; j < 16; ++j) out[t * 16 + j - 1] = j < k ? (uint8_t)p[j] : 0;
    out[t * 16 + 15] = 0;
}

// Generic range kernel (status-tracking): one thread per index; records the
// first erroring candidate in enumeration order.
__global__ void __launch_bounds__(256) k3_argmin_generic(DevInst I, RangeGeom G, ArgminScratch S,
                                                         const uint32_t* only_if_flags) {
    // fix-up launch behind a fast-path kernel: do nothing unless the table
    // build raised a flag (then this kernel's result replaces the fast one)
    if (only_if_flags && *only_if_flags == 0u) return;
    Key mine{INFINITY, ~0ull};
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long t = G.lo + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
         t < G.hi; t += stride) {
        unsigned long long idx = t;
        if (G.items_mode) {  // t = (b * span + item offset) * NC + comp
            unsigned long long comp0 = t % G.NC, r0 = t / G.NC;
            unsigned long long item = G.it_lo + r0 % G.it_span, b = r0 / G.it_span;
            idx = ((b * G.nm + item / G.NP) * G.NP + item % G.NP) * G.NC + comp0;
        }
        unsigned long long comp = idx % G.NC;
        unsigned long long r = idx / G.NC;
        unsigned long long perm_rank = r % G.NP;
        int bmi = (int)(r / G.NP);
        uint8_t order[GP_MAX_STAGES];
        int p[GP_MAX_STAGES + 1];
        d_unrank_perm(G.k, perm_rank, order);
        d_unrank_cuts(I.n, G.k, comp, p);
        int mi = bmi % I.nm;
        long long M = I.batch[bmi / I.nm] / I.micro[mi];
        EvalOut e = eval_tables(I, G.k, order, p, mi, M);
        if (e.status != GP_OK) {
            atomicMin(S.err_idx, (idx << 4) | (unsigned long long)e.status);
        } else {
            Key o{e.cost, ((perm_rank * G.NC) + comp) * (unsigned long long)G.nbm + (unsigned long long)bmi};
            if (key_less(o, mine)) mine = o;
        }
    }
    block_argmin_finish(mine, S);
}

// ---- plan detail of one candidate (single thread) -----------------------------------
__device__ void plan_detail_dev(const DevInst& I, int k, const uint8_t* o, const int* p, int bm,
                                gp_plan_info* out, int* status) {
    int n = I.n;
    size_t N2 = (size_t)(n + 1) * (n + 1);
    int mi = bm % I.nm;
    long long M = I.batch[bm / I.nm] / I.micro[mi];
    EvalOut r = eval_tables(I, k, o, p, mi, M);
    *status = r.status;
    out->k = (uint32_t)k;
    out->plan_cost = r.cost;
    bool feas = true;
    for (int s = 0; s < k; ++s)
        if (I.scode[(size_t)o[s] * N2 + tri_idx(n, p[s], p[s + 1])] == SC_INFEASIBLE) feas = false;
    out->feasible = feas ? 1 : 0;
    const double2* T = I.stg + (size_t)mi * I.F * N2;
    const double* X = I.xt + (size_t)mi * I.F * I.F * I.nxp;
    double Md = (double)M;
    double fill = 0.0, res = 0.0, xprev = 0.0;
    for (int s = 0; s < k; ++s) {
        gp_stage_info& st = out->stage[s];
        int shares[GP_MAX_SGS], np;
        int kind = choose_split(I, o[s], p[s], p[s + 1], shares, &np);
        st.kind = (uint32_t)kind;
        st.n_parts = (uint32_t)np;
        if (kind == GP_ASYM_PP) {
            int pos = p[s];
            for (int j = 0; j < np; ++j) {
                st.pp_sg[j] = (uint32_t)j;
                st.pp_start[j] = (uint32_t)pos;
                st.pp_end[j] = (uint32_t)(pos + shares[j]);
                pos += shares[j];
            }
        }
        if (!feas || r.status != GP_OK) continue;
        double2 e = T[(size_t)o[s] * N2 + tri_idx(n, p[s], p[s + 1])];
        if (s > 0) res = res + gpd::max0(xprev - e.x);
        st.fill_seconds = fill;
        st.run_seconds = Md * e.x;
        st.residual_seconds = res;
        st.collective_seconds = e.y;
        if (s + 1 < k) {
            double x = X[((size_t)o[s] * I.F + o[s + 1]) * I.nxp + (p[s + 1] - 1)];
            fill = fill + (e.x + x);
            xprev = x;
        }
    }
}

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
    Key key;
    unsigned long long err;
    int status;        // of the detail evaluation
    uint32_t k, bm, pad;
    uint8_t order[GP_MAX_STAGES];
    uint8_t counts[GP_MAX_STAGES];
    gp_plan_info info;
};

// Warp version of plan_detail_dev: lane s prepares stage s (split choice and
// table loads in parallel), lane 0 runs the short Eq. 1 chain.
__device__ void plan_detail_warp(const DevInst& I, int k, const uint8_t* o, const int* p, int bm,
                                 gp_plan_info* out, int* status) {
    const int lane = threadIdx.x & 31;
    const int n = I.n;
    const size_t N2 = (size_t)(n + 1) * (n + 1);
    const int mi = bm % I.nm;
    const long long M = I.batch[bm / I.nm] / I.micro[mi];
    const double2* T = I.stg + (size_t)mi * I.F * N2;
    const double* X = I.xt + (size_t)mi * I.F * I.F * I.nxp;
    double2 e = make_double2(0.0, 0.0);
    double x = 0.0;
    uint8_t code = SC_OK;
    bool gw_bad = false;
    if (lane < k) {
        const int s = lane;
        gp_stage_info& st = out->stage[s];
        int shares[GP_MAX_SGS], np;
        const int kind = choose_split(I, o[s], p[s], p[s + 1], shares, &np);
        st.kind = (uint32_t)kind;
        st.n_parts = (uint32_t)np;
        if (kind == GP_ASYM_PP) {
            int pos = p[s];
            for (int j = 0; j < np; ++j) {
                st.pp_sg[j] = (uint32_t)j;
                st.pp_start[j] = (uint32_t)pos;
                st.pp_end[j] = (uint32_t)(pos + shares[j]);
                pos += shares[j];
            }
        }
        const size_t ei = (size_t)o[s] * N2 + tri_idx(n, p[s], p[s + 1]);
        e = T[ei];
        code = I.scode[ei];
        if (s + 1 < k) {
            x = X[((size_t)o[s] * I.F + o[s + 1]) * I.nxp + (p[s + 1] - 1)];
            gw_bad = !(I.bw[I.gw[o[s] * I.F + o[s + 1]]] > 0);
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
    const double Md = (double)M;
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

__global__ void k_solve_detail(DevInst I, int k, unsigned long long NC, unsigned long long NP,
                               int nbm, const Key* result, const unsigned long long* err,
                               const unsigned long long* __restrict__ binom, SolveOut* out) {
    // one warp: decode the arg-min key (cut positions by a 32-wide ballot
    // over the hockey-stick counts), then the warp plan detail
    const int lane = threadIdx.x & 31;
    const Key key = *result;
    const unsigned long long e = *err;
    if (lane == 0) {
        out->key = key;
        out->err = e;
        out->k = (uint32_t)k;
        out->status = GP_OK;
    }
    if (e != ~0ull || key.tie == ~0ull) return;
    const int n = I.n;
    const unsigned long long t = key.tie;
    const int bm = (int)(t % (unsigned long long)nbm);
    const unsigned long long pc = t / (unsigned long long)nbm;
    uint8_t o[GP_MAX_STAGES];
    int p[GP_MAX_STAGES + 1];
    d_unrank_perm(k, pc / NC, o);
    p[0] = 0;
    unsigned long long rem = pc % NC;
    int prev = 0;
    auto C = [&](int nn, int r) -> unsigned long long {
        return (r < 0 || nn < 0) ? 0ull : binom[(size_t)nn * (GP_MAX_STAGES + 1) + r];
    };
    for (int j = 1; j < k; ++j) {
        const int r = k - 1 - j, lo = prev + 1;
        const unsigned long long tot = C(n - lo, r + 1), thr = tot - rem;
        int qsel = -1;
        for (int base = lo; qsel < 0; base += 32) {
            const int qq = base + lane;
            const bool ok = qq <= n - 1 - r && C(n - qq - 1, r + 1) < thr;
            const unsigned m = __ballot_sync(0xffffffffu, ok);
            if (m) qsel = base + __ffs(m) - 1;
        }
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

// ----------------------------------------------------------------------------
// K4: exact arg-min by branch-and-bound over the layer cuts, with min-max DP
// bounds - for stage counts where the exhaustive sweep explodes.
//
// One warp per item (b, m, order).  R[s][a] = min over completions of
// max_{s' >= s} M*c_{s'} is a min-max DP over the stage table (exact: only
// min / max of table values).  A node fixes stages 0..d with exact reference
// arithmetic (fill, residual, running max pm); for every completion the true
// cost is >= max(pm, fl(fill_{d+1} + R[d+1][b])) because all terms are
// non-negative and rounding is monotone, so the bound is exact in floating
// point (no epsilon band).  Children (next cut b) are evaluated 32 at a time
// by the lanes; a node is pruned when its bound exceeds the best finite cost
// found by any warp (atomicMin on the IEEE bits) or reaches the warp's own
// best (a later candidate of the same item has a larger rank).  Nodes are
// visited in lexicographic order of the cuts, so the first strict
// improvement is the smallest rank among equal costs (reference tie-break).
// ----------------------------------------------------------------------------
struct BnbGeom {
    int k, nbm;
    unsigned long long NC, NP;
    unsigned long long* gbest;     // global best finite cost bits
};

__global__ void __launch_bounds__(32) k4_bnb(DevInst I, BnbGeom G, ArgminScratch S,
                                             const unsigned long long* __restrict__ binom) {
    extern __shared__ __align__(16) double R[];   // [k][n+1]
    const int lane = threadIdx.x;
    const int n = I.n, k = G.k;
    const size_t N2 = (size_t)(n + 1) * (n + 1);
    // item = (bi, mi, perm) in bm-major order
    const unsigned long long item = blockIdx.x;
    const int bm = (int)(item / G.NP);
    const unsigned long long perm_rank = item % G.NP;
    const int bi = bm / I.nm, mi = bm % I.nm;
    uint8_t o[GP_MAX_STAGES];
    d_unrank_perm(k, perm_rank, o);
    const double Md = (double)(I.batch[bi] / I.micro[mi]);
    const double2* T = I.stg + (size_t)mi * I.F * N2;
    const double* X = I.xt + (size_t)mi * I.F * I.F * I.nxp;
    auto cm = [&](int s, int a, int b) -> double2 {
        return __ldg(&T[(size_t)o[s] * N2 + tri_idx(n, a, b)]);
    };
    // ---- exact-in-reals DP: with P_s the cost prefix before
    // stage s (fill + earlier residual terms) and, for stage s = [a, b),
    //   L_s = M*c + AL + rho_s,  rho_s = max0(x_{s-1}(a) - c),  G_s = c + x_s(b),
    // the plan cost is max_s (P_s + L_s) and P_{s+1} = P_s + rho_s + G_s, so
    //   W(s, a) = min_b max(L_s(a,b), rho_s(a,b) + G_s(a,b) + W(s+1, b))
    // is the optimal completion from stage s starting at a.  Computed in
    // floating point; node bounds scale it by (1 - 2^-40) - far more than the
    // relative rounding gap to the reference-order cost - so pruning is exact.
    auto xrow = [&](int s2, int j) -> double {  // x of boundary s2 at layer j
        return __ldg(&X[((size_t)o[s2] * I.F + o[s2 + 1]) * I.nxp + j]);
    };
    for (int a = lane; a <= n; a += 32) {
        double w = INFINITY;
        if (a >= k - 1 && a < n) {
            const double2 e = cm(k - 1, a, n);
            const double rho = k > 1 ? max0f(xrow(k - 2, a - 1) - e.x) : 0.0;
            w = ((Md * e.x) + e.y) + rho;
        }
        R[(size_t)(k - 1) * (n + 1) + a] = w;
    }
    __syncwarp();
    for (int s = k - 2; s >= 0; --s) {
        const int bmax = n - (k - 1 - s);
        for (int a = lane; a <= n; a += 32) {
            double best = INFINITY;
            if (a >= s && (s > 0 || a == 0)) {
                const double xin = s > 0 ? xrow(s - 1, a - 1) : 0.0;
                for (int b = a + 1; b <= bmax; ++b) {
                    const double2 e = cm(s, a, b);
                    const double rho = s > 0 ? max0f(xin - e.x) : 0.0;
                    const double L = ((Md * e.x) + e.y) + rho;
                    const double rest = (rho + (e.x + xrow(s, b - 1))) + R[(size_t)(s + 1) * (n + 1) + b];
                    const double v = rest > L ? rest : L;
                    best = v < best ? v : best;
                }
            }
            R[(size_t)s * (n + 1) + a] = best;
        }
        __syncwarp();
    }
    const double QMARGIN = 1.0 - 0x1p-40;
    // ---- seed the shared incumbent with the DP's greedy path, evaluated
    // exactly (only its cost is used: as a pruning bound, never as the answer)
    {
        int a = 0;
        double fill = 0.0, res = 0.0, xprev = 0.0, pm = 0.0;
        for (int s2 = 0; s2 < k; ++s2) {
            int b = n;
            if (s2 < k - 1) {
                const int bmax = n - (k - 1 - s2);
                double bv = INFINITY;
                b = 0x7fffffff;
                for (int bb = a + 1 + lane; bb <= bmax; bb += 32) {
                    const double2 e = cm(s2, a, bb);
                    const double rho = s2 > 0 ? max0f(xprev - e.x) : 0.0;
                    const double L = ((Md * e.x) + e.y) + rho;
                    const double rest = (rho + (e.x + xrow(s2, bb - 1))) + R[(size_t)(s2 + 1) * (n + 1) + bb];
                    const double v = rest > L ? rest : L;
                    if (v < bv || b == 0x7fffffff) { bv = v; b = bb; }
                }
                for (int off = 16; off > 0; off >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
                    const int ob = __shfl_xor_sync(0xffffffffu, b, off);
                    if (ov < bv || (ov == bv && ob < b)) { bv = ov; b = ob; }
                }
            }
            const double2 e = cm(s2, a, b);
            if (s2 > 0) res = res + max0f(xprev - e.x);
            const double tot = ((fill + Md * e.x) + res) + e.y;
            pm = (s2 == 0) ? tot : gtsel(tot, pm);
            if (s2 + 1 < k) {
                const double x = xrow(s2, b - 1);
                fill = fill + (e.x + x);
                xprev = x;
            }
            a = b;
        }
        if (lane == 0 && !isinf(pm) && !isnan(pm))
            atomicMin(G.gbest, (unsigned long long)__double_as_longlong(pm));
    }
    // ---- depth-first branch-and-bound (warp-uniform control flow)
    struct Frame { int a, b0; unsigned mask; double fill, res, xprev, pm; };
    Frame F[GP_MAX_STAGES];
    int cut[GP_MAX_STAGES + 1];
    cut[0] = 0;
    double loc_c = INFINITY;
    unsigned long long loc_r = ~0ull;
    bool have = false;
    int d = 0;
    F[0].a = 0; F[0].b0 = 1; F[0].fill = 0.0; F[0].res = 0.0; F[0].xprev = 0.0; F[0].pm = -INFINITY;
    bool need_eval = true;
    for (;;) {
        Frame& f = F[d];
        const int bmax = (d == k - 1) ? n : n - (k - 1 - d);
        if (need_eval) {
            need_eval = false;
            const int b = f.b0 + lane;
            const bool valid = b <= bmax && b > f.a;
            const double bound = __longlong_as_double((long long)*(volatile unsigned long long*)G.gbest);
            bool keep = false;
            double leaf_cost = INFINITY;
            if (valid) {
                const double2 e = cm(d, f.a, b);
                const double res1 = (d > 0) ? f.res + max0f(f.xprev - e.x) : f.res;
                const double tot = ((f.fill + Md * e.x) + res1) + e.y;
                const double pm1 = (d == 0) ? tot : gtsel(tot, f.pm);
                if (d == k - 1) {
                    leaf_cost = pm1;  // b == n: the last stage
                } else {
                    const double x = __ldg(&X[((size_t)o[d] * I.F + o[d + 1]) * I.nxp + (b - 1)]);
                    const double fill1 = f.fill + (e.x + x);
                    if (d == k - 2) {
                        // leaf: stage k-1 = [b, n)
                        const double2 e3 = cm(k - 1, b, n);
                        const double res3 = res1 + max0f(x - e3.x);
                        const double t3 = ((fill1 + Md * e3.x) + res3) + e3.y;
                        leaf_cost = gtsel(t3, pm1);
                    } else {
                        // P_{d+1} = fill + all residual terms so far (res1)
                        const double lbr = ((fill1 + res1) + R[(size_t)(d + 1) * (n + 1) + b]) * QMARGIN;
                        const double lb = gtsel(lbr, pm1);
                        keep = !(lb > bound) && (!have || lb < loc_c);
                    }
                }
            }
            if (d >= k - 2) {
                // leaves of this chunk: warp arg-min on (cost, b), then strict update
                double c = valid ? leaf_cost : INFINITY;
                int bb = valid ? b : 0x7fffffff;
                for (int off = 16; off > 0; off >>= 1) {
                    const double oc = __shfl_xor_sync(0xffffffffu, c, off);
                    const int ob = __shfl_xor_sync(0xffffffffu, bb, off);
                    if (oc < c || (oc == c && ob < bb)) { c = oc; bb = ob; }
                }
                if (bb != 0x7fffffff && (!have || c < loc_c)) {
                    cut[d + 1] = bb;
                    // composition rank of (cut[1..k-1])
                    unsigned long long r = 0;
                    for (int j = 1; j < k; ++j) {
                        const int nn1 = n - cut[j - 1] - 1, nn2 = n - cut[j];
                        const unsigned long long c1 = nn1 >= 0 ? binom[(size_t)nn1 * (GP_MAX_STAGES + 1) + (k - j)] : 0ull;
                        const unsigned long long c2 = nn2 >= 0 ? binom[(size_t)nn2 * (GP_MAX_STAGES + 1) + (k - j)] : 0ull;
                        r += c1 - c2;
                    }
                    have = true;
                    loc_c = c;
                    loc_r = r;
                    if (lane == 0 && !isinf(c))
                        atomicMin(G.gbest, (unsigned long long)__double_as_longlong(c));
                }
                f.mask = 0u;
            } else {
                f.mask = __ballot_sync(0xffffffffu, keep);
            }
        }
        if (f.mask == 0u) {
            f.b0 += 32;
            if (f.b0 > bmax || d == k - 1) {
                if (d == 0) break;
                --d;
                continue;
            }
            need_eval = true;
            continue;
        }
        // descend into the first surviving child
        const int c = __ffs(f.mask) - 1;
        f.mask &= ~(1u << c);
        const int b = f.b0 + c;
        const double2 e = cm(d, f.a, b);
        const double res1 = (d > 0) ? f.res + max0f(f.xprev - e.x) : f.res;
        const double tot = ((f.fill + Md * e.x) + res1) + e.y;
        const double x = __ldg(&X[((size_t)o[d] * I.F + o[d + 1]) * I.nxp + (b - 1)]);
        Frame& g = F[d + 1];
        g.a = b;
        g.b0 = b + 1;
        g.fill = f.fill + (e.x + x);
        g.res = res1;
        g.xprev = x;
        g.pm = (d == 0) ? tot : gtsel(tot, f.pm);
        cut[d + 1] = b;
        ++d;
        need_eval = true;
    }
    Key mine{INFINITY, ~0ull};
    if (have && lane == 0) {
        mine.cost = loc_c;
        mine.tie = ((perm_rank * G.NC) + loc_r) * (unsigned long long)G.nbm + (unsigned long long)bm;
    }
    block_argmin_finish(mine, S);
}

// ----------------------------------------------------------------------------
// K6: bandwidth-snapshot re-plan.  A snapshot rescales link bandwidths only
// (p_t, grouping, gateway pairs, splits and memory feasibility are
// unchanged - SURVEY.md CS4), so per snapshot the engine re-derives
//   min_intra_bandwidth per group            (src/grouping.py:69-75)
//   AL = V / min_bw per stage-table entry     (src/timing.py:146-173)
//   x = lat + (act*m)/bw per gateway/boundary (src/timing.py:91-97, 209-225)
// into per-snapshot copies of the packed tables, then one K3 sweep launch
// covers every (snapshot, item) with a per-snapshot arg-min.
// ----------------------------------------------------------------------------
struct SnapGeom {
    int nsnap;
    const double* bw;            // [nsnap][D*D]
    double* mbw;                 // [nsnap][F]
    uint32_t* flags;             // [nsnap]
    double2* tpk;                // [nsnap][nm][F][ntri]
    double2* tcol;               // [nsnap][nm][F][n+1]
    double* xt;                  // [nsnap][nm][F][F][nxp]
    unsigned long long s_tpk, s_tcol, s_xt;
};

__global__ void k6_minbw(DevInst I, SnapGeom Z) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= Z.nsnap * I.F) return;
    const int sn = t / I.F, f = t % I.F;
    const double* bw = Z.bw + (size_t)sn * I.D * I.D;
    const int m0 = I.fg_off[f], m1 = I.fg_off[f + 1];
    double mn = 0.0;
    bool have = false;
    for (int x = m0; x < m1; ++x)
        for (int y = x + 1; y < m1; ++y) {
            double w = bw[(size_t)I.fg_mem[x] * I.D + I.fg_mem[y]];
            if (!have || w < mn) mn = w;
            have = true;
        }
    Z.mbw[(size_t)sn * I.F + f] = have ? mn : 0.0;
    if (I.fg_has_minbw[f] && !(mn > 0)) atomicOr(&Z.flags[sn], FLAG_STAGE_ERROR);
    if (f == 0)
        for (int pr = 0; pr < I.F * I.F; ++pr) {
            const int fa = pr / I.F, fb = pr % I.F;
            if (fa != fb && !(bw[I.gw[pr]] > 0)) atomicOr(&Z.flags[sn], FLAG_GATEWAY_ERROR);
        }
}

__global__ void k6_patch(DevInst I, SnapGeom Z) {
    const int n = I.n;
    const long long ntri = (long long)n * (n + 1) / 2;
    const long long per_snap_tri = (long long)I.nm * I.F * ntri;
    const long long per_snap_x = (long long)I.nm * I.F * I.F * n;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int sn = blockIdx.y;
    const double* mbw = Z.mbw + (size_t)sn * I.F;
    if (t < per_snap_tri) {
        const int f = (int)((t / ntri) % I.F);
        const int mi = (int)(t / (ntri * I.F));
        const int e = (int)(t % ntri);
        // packed entry e -> (a, b): row a holds n - a entries
        int a = 0, off = e;
        while (off >= n - a) { off -= n - a; ++a; }
        const int b = a + 1 + off;
        double2 v = I.tpk[t];
        const double V = I.vtab[t];
        const double mb = mbw[f];
        v.y = (V != 0.0 && I.fg_has_minbw[f] && mb > 0) ? V / mb : 0.0;
        Z.tpk[sn * Z.s_tpk + t] = v;
        if (b == n) Z.tcol[sn * Z.s_tcol + ((size_t)mi * I.F + f) * (n + 1) + a] = v;
        if (a == 0 && b == 1)
            Z.tcol[sn * Z.s_tcol + ((size_t)mi * I.F + f) * (n + 1) + n] = make_double2(INFINITY, 0.0);
    } else if (t < per_snap_tri + per_snap_x) {
        const long long u = t - per_snap_tri;
        const int j = (int)(u % n);
        const long long r = u / n;  // mi * F * F + pair
        const int pair = (int)(r % (I.F * I.F));
        const int mi = (int)(r / (I.F * I.F));
        const int g = I.gw[pair];
        const double md = (double)I.micro[mi];
        const double bw = Z.bw[(size_t)sn * I.D * I.D + g];
        Z.xt[sn * Z.s_xt + (size_t)r * I.nxp + j] = I.lat[g] + (I.act[j] * md) / bw;
    }
}

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

__device__ int sim_1f1b_dev(const gp_timing& T, int iterations, double* makespan) {
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
        const double bw = T.bw[bnd] * 1.0;  // base * multiplier(1.0)
        SimEv& e = ev[nev++];
        e.t = (tnow + (per * (double)sz) / bw) + T.lat[bnd];
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
                // _ready_op (src/engine.py:157-215), ONE_F_ONE_B priorities
                int best_pr = 100, best_k = -1;
                long long best_sz = 0;
                const long long fwd_rem = B - p.fwd_taken;
                if (fwd_rem > 0) {
                    const long long chunk = m < fwd_rem ? m : fwd_rem;
                    if (p.fwd_avail - p.fwd_taken >= chunk) {
                        const long long quota = (long long)(S - s) * m;
                        int pr = -1;
                        if (p.fwd_taken < quota) pr = 1;
                        else if (p.fwd_taken + chunk <= quota + p.bwd_done) pr = 2;
                        if (pr >= 0) { best_pr = pr; best_k = 0; best_sz = chunk; }
                    }
                }
                const long long bwd_rem = B - p.bwd_taken;
                if (bwd_rem > 0) {
                    const long long chunk = m < bwd_rem ? m : bwd_rem;
                    long long av = (p.bwd_avail < p.fwd_done ? p.bwd_avail : p.fwd_done) - p.bwd_taken;
                    if (s == S - 1) av = p.fwd_done - p.bwd_taken;
                    if (av >= chunk && 2 < best_pr) { best_pr = 2; best_k = 1; best_sz = chunk; }
                }
                if (p.wq_head < p.wq_tail && 0 < best_pr) {
                    best_pr = 0; best_k = 2; best_sz = chunk_size(p.wq_head);
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
    st = sim_1f1b_dev(T, iterations, &ms);
    makespan[i] = ms;
    status[i] = (uint8_t)st;
}

__global__ void k5_sim_1f1b(const gp_timing* __restrict__ T, long long n, int iterations,
                            double* __restrict__ makespan, uint8_t* __restrict__ status) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double ms = NAN;
    int st = sim_1f1b_dev(T[i], iterations, &ms);
    makespan[i] = ms;
    status[i] = (uint8_t)st;
}

// ----------------------------------------------------------------------------
// context
// ----------------------------------------------------------------------------
// bumped on every device (re)allocation: a captured CUDA graph is only
// replayed while the buffers it was captured with are still in place
static unsigned long long g_alloc_gen = 0;

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t count) {
        if (count <= cap && p) return cudaSuccess;
        __atomic_add_fetch(&g_alloc_gen, 1ull, __ATOMIC_RELAXED);
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t c = count ? count : 1;
        cudaError_t e = cudaMalloc(&p, c * sizeof(T));
        if (e == cudaSuccess) cap = c;
        return e;
    }
    void release() { if (p) cudaFree(p); p = nullptr; cap = 0; }
};

template <typename T>
struct ArenaPtr {
    T* p = nullptr;
    void release() { p = nullptr; }
};

struct gp_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool loaded = false;
    uint32_t flags = 0;
    int n = 0, F = 0, D = 0, nb = 0, nm = 0, nsg = 0;
    std::vector<long long> h_batch, h_micro;
    // raw instance arrays live in the arena (one allocation, one H2D copy)
    ArenaPtr<double> fwd, bwd_in, bwd_w, act, param, p_c, mem, p_t, lat, bw, fg_cap, sg_cap,
        fg_minbw, fg_minbw_in;
    ArenaPtr<long long> batch, micro;
    ArenaPtr<uint32_t> id_rank, fg_off, fg_mem, fg_sg_off, sg_off, sg_mem;
    ArenaPtr<uint8_t> fg_has;
    // derived tables
    DBuf<double> S, g_rf, g_cf, g_dp, g_minmem, sg_minmem, C1, xt;
    DBuf<double4> fbws;
    DBuf<double> vtab;
    DBuf<double2> tpk, tcol;
    DBuf<uint32_t> flagsbuf;
    DBuf<uint8_t> g_tp_ok, scode, skind;
    DBuf<double2> stg;
    DBuf<int> gw;
    // K3 scratch
    DBuf<Key> blk, result;
    DBuf<unsigned int> counter;
    DBuf<unsigned long long> err_idx;
    DBuf<int> err_dummy;
    // K2 staging
    DBuf<uint8_t> b_order, b_counts, b_bm, b_status;
    DBuf<double> b_cost;
    DBuf<gp_plan_info> info;
    DBuf<gp_group_info> ginfo;
    DBuf<int> dstatus;
    DBuf<SolveOut> dsolve;
    DBuf<unsigned long long> gbest;  // K4 shared incumbent
    DBuf<gp_timing> s_tim;       // K5 staging
    // K6 snapshot batch buffers
    DBuf<double> z_bw, z_mbw, z_xt;
    DBuf<uint32_t> z_flags;
    DBuf<double2> z_tpk, z_tcol;
    DBuf<Key> z_res;
    DBuf<unsigned int> z_cnt;
    DBuf<double> s_ms;
    DBuf<uint8_t> s_st;
    SolveOut* h_solve = nullptr;  // pinned
    RangeGeom last_geom{};
    bool last_generic = false;
    unsigned long long last_lo = 0, last_hi = 0;
    int smem_max = 0;
    int n_sms = 148;
    uint32_t* h_flags = nullptr;      // pinned
    cudaEvent_t flags_ev = nullptr;
    cudaEvent_t arena_ev = nullptr;
    bool flags_known = false;
    // raw instance arena: one pinned staging buffer -> one H2D copy
    unsigned char* h_arena = nullptr;
    size_t h_arena_cap = 0;
    DBuf<unsigned char> arena;
    int cache_n = -1, cache_k = -1;   // (n, k) of the enumeration helpers
    // gp_replan: CUDA graph of H2D + K1 + K3 + detail + D2H for one shape
    cudaGraphExec_t graph_exec = nullptr;
    unsigned long long graph_key[10] = {0};
    unsigned long long graph_gen = 0;
    RangeGeom graph_geom{};
    unsigned long long graph_lo = 0, graph_hi = 0;
    bool capturing = false;
    size_t arena_bytes = 0;
    int force_mode = -1;  // -1 auto; 0/1/2 fast-path variant; 3 generic kernel
    DBuf<unsigned long long> binom;
    DBuf<unsigned int> item_ctr;
    DBuf<uint8_t> tiles;
    bool tiles_ok = false;
    DBuf<uint4> groups;       // K3 sweep run groups
    DBuf<uint8_t> prefixes;   // colex (k-3)-subsets for the sweep
    DBuf<unsigned long long> bnk;  // binomial sub-table [n+1][k+1] (TMA-staged)
    int ngroups = 0;
    unsigned int sweep_W = 0;
    bool sweep_ok = false;

    DevInst view() {
        DevInst I;
        I.n = n; I.F = F; I.D = D; I.nb = nb; I.nm = nm;
        I.fwd = fwd.p; I.bwd_in = bwd_in.p; I.bwd_w = bwd_w.p; I.act = act.p; I.param = param.p;
        I.batch = batch.p; I.micro = micro.p;
        I.p_c = p_c.p; I.mem = mem.p; I.p_t = p_t.p; I.lat = lat.p; I.bw = bw.p;
        I.id_rank = id_rank.p;
        I.fg_off = fg_off.p; I.fg_mem = fg_mem.p; I.fg_sg_off = fg_sg_off.p;
        I.sg_off = sg_off.p; I.sg_mem = sg_mem.p;
        I.fg_cap = fg_cap.p; I.sg_cap = sg_cap.p;
        I.fg_minbw = fg_minbw.p; I.fg_has_minbw = fg_has.p;
        I.bf = bf;
        I.S = S.p; I.g_tp_ok = g_tp_ok.p; I.g_rf = g_rf.p; I.g_cf = g_cf.p; I.g_dp = g_dp.p;
        I.g_minmem = g_minmem.p; I.sg_minmem = sg_minmem.p;
        I.stg = stg.p; I.scode = scode.p; I.skind = skind.p; I.C1 = C1.p; I.fbws = fbws.p; I.vtab = vtab.p;
        I.gw = gw.p; I.xt = xt.p; I.flags = flagsbuf.p;
        I.nxp = (n + 1) & ~1;
        I.tpk = tpk.p; I.tcol = tcol.p;
        return I;
    }
    double bf = 1.25;
};

template <typename T>
static cudaError_t upload(cudaStream_t s, DBuf<T>& d, const T* h, size_t count) {
    cudaError_t e = d.ensure(count);
    if (e != cudaSuccess) return e;
    if (count == 0) return cudaSuccess;
    return cudaMemcpyAsync(d.p, h, count * sizeof(T), cudaMemcpyHostToDevice, s);
}

static unsigned long long h_binom(int n, int r) {
    if (r < 0 || r > n) return 0ull;
    unsigned long long res = 1;
    for (int i = 1; i <= r; ++i) res = res * (unsigned long long)(n - r + i) / (unsigned long long)i;
    return res;
}

extern "C" {

const char* gp_version(void) { return "geopipe_b200 0.1 (sm_100a)"; }
const char* gp_last_error(void) { return g_err; }

int gp_ctx_create(int device, gp_ctx** out) {
    if (!out) return fail(GP_ERR_INPUT, "null output pointer");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(GP_ERR_CUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
    if (device < 0 || device >= count) return fail(GP_ERR_INPUT, "device %d out of range", device);
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(GP_ERR_CUDA, "device %d is sm_%d%d; this engine is built for sm_100a",
                    device, prop.major, prop.minor);
    CUDA_TRY(cudaSetDevice(device));
    gp_ctx* c = new gp_ctx();
    c->device = device;
    c->smem_max = (int)prop.sharedMemPerBlockOptin;
    c->n_sms = prop.multiProcessorCount;
    if (const char* fm = getenv("GP_K3_MODE")) c->force_mode = atoi(fm);
    if (cudaHostAlloc((void**)&c->h_flags, sizeof(uint32_t), cudaHostAllocDefault) != cudaSuccess ||
        cudaHostAlloc((void**)&c->h_solve, sizeof(SolveOut), cudaHostAllocDefault) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->flags_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->arena_ev, cudaEventDisableTiming) != cudaSuccess) {
        gp_ctx_destroy(c);
        return fail(GP_ERR_CUDA, "pinned flag / event allocation failed");
    }
    cudaError_t se = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (se != cudaSuccess) { delete c; return fail(GP_ERR_CUDA, "stream: %s", cudaGetErrorString(se)); }
    *out = c;
    return GP_OK;
}

void* gp_ctx_stream(gp_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

void gp_ctx_destroy(gp_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    DBuf<double>* dd[] = {&c->S, &c->g_rf, &c->g_cf, &c->g_dp, &c->g_minmem, &c->sg_minmem,
                          &c->C1, &c->xt, &c->b_cost};
    for (auto* b : dd) b->release();
    c->fbws.release();
    c->vtab.release();
    c->flagsbuf.release();
    DBuf<uint8_t>* bb[] = {&c->g_tp_ok, &c->scode, &c->skind, &c->b_order, &c->b_counts,
                           &c->b_bm, &c->b_status};
    for (auto* b : bb) b->release();
    c->arena.release();
    if (c->h_arena) cudaFreeHost(c->h_arena);
    if (c->h_flags) cudaFreeHost(c->h_flags);
    if (c->h_solve) cudaFreeHost(c->h_solve);
    c->z_bw.release(); c->z_mbw.release(); c->z_xt.release(); c->z_flags.release();
    c->z_tpk.release(); c->z_tcol.release(); c->z_res.release(); c->z_cnt.release();
    c->dsolve.release(); c->gbest.release(); c->s_tim.release(); c->s_ms.release(); c->s_st.release();
    if (c->flags_ev) cudaEventDestroy(c->flags_ev);
    if (c->arena_ev) cudaEventDestroy(c->arena_ev);
    if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
    c->binom.release(); c->item_ctr.release(); c->tiles.release(); c->groups.release(); c->prefixes.release(); c->bnk.release();
    c->tpk.release(); c->tcol.release();
    c->stg.release(); c->gw.release(); c->blk.release(); c->result.release();
    c->counter.release(); c->err_idx.release(); c->err_dummy.release(); c->info.release();
    c->ginfo.release(); c->dstatus.release();
    cudaStreamDestroy(c->stream);
    delete c;
}

static int run_tables(gp_ctx* c, bool full) {
    DevInst I = c->view();
    cudaStream_t s = c->stream;
    CUDA_TRY(cudaMemsetAsync(c->flagsbuf.p, 0, sizeof(uint32_t), s));
    if (full) {
        // interval sums + group constants + gateways (independent) in one launch
        const int gw_blocks = (c->F * c->F + 3) / 4;
        k1_phase1<<<5 + c->F + gw_blocks, 128, 0, s>>>(I);
    } else {
        k1_gateways<<<(c->F * c->F * 32 + 127) / 128, 128, 0, s>>>(I);
    }
    // stage table + boundary table in one launch
    long long ns = (long long)c->F * (c->n + 1) * (c->n + 1);
    long long nx = (long long)c->nm * c->F * c->F * c->n;
    k1_phase2<<<(unsigned)((ns + nx + 127) / 128), 128, 0, s>>>(I, ns);
    CUDA_TRY(cudaGetLastError());
    // flags travel back asynchronously; kernels consult the device copy when
    // the host copy is not known yet (no synchronisation on the load path)
    CUDA_TRY(cudaMemcpyAsync(c->h_flags, c->flagsbuf.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaEventRecord(c->flags_ev, s));
    c->flags_known = false;
    return GP_OK;
}

// host-side flags when the async read-back has landed; -1 when still pending
static int known_flags(gp_ctx* c) {
    if (c->capturing) return -1;  // graph: device-side dispatch
    if (c->flags_known) return (int)c->flags;
    if (cudaEventQuery(c->flags_ev) == cudaSuccess) {
        c->flags = *c->h_flags;
        c->flags_known = true;
        return (int)c->flags;
    }
    return -1;
}

int gp_ctx_load(gp_ctx* c, const gp_instance* in) {
    if (!c || !in) return fail(GP_ERR_INPUT, "null argument");
    if (in->n_layers < 1 || in->n_layers > GP_MAX_LAYERS)
        return fail(GP_ERR_INPUT, "n_layers %u outside [1, %d]", in->n_layers, GP_MAX_LAYERS);
    if (in->n_fgs < 1 || in->n_fgs > GP_MAX_STAGES)
        return fail(GP_ERR_INPUT, "n_fgs %u outside [1, %d]", in->n_fgs, GP_MAX_STAGES);
    if (in->n_batch < 1 || in->n_micro < 1 || in->n_batch * in->n_micro > 255)
        return fail(GP_ERR_INPUT, "bad (batch, micro) candidate counts");
    for (uint32_t i = 0; i < in->n_batch; ++i)
        for (uint32_t j = 0; j < in->n_micro; ++j)
            if (in->batch[i] <= 0 || in->micro[j] <= 0 || in->batch[i] % in->micro[j])
                return fail(GP_ERR_INPUT, "micro-batch %lld does not divide batch %lld",
                            (long long)in->micro[j], (long long)in->batch[i]);
    uint32_t nsg = in->fg_sg_offset[in->n_fgs];
    for (uint32_t f = 0; f < in->n_fgs; ++f) {
        uint32_t nm = in->fg_member_offset[f + 1] - in->fg_member_offset[f];
        uint32_t ng = in->fg_sg_offset[f + 1] - in->fg_sg_offset[f];
        if (nm < 1 || nm > GP_MAX_MEMBERS) return fail(GP_ERR_INPUT, "group %u has %u members", f, nm);
        if (ng > GP_MAX_SGS) return fail(GP_ERR_INPUT, "group %u has %u subgroups", f, ng);
    }
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    uint32_t n = in->n_layers, D = in->n_devices, F = in->n_fgs;
    c->n = (int)n; c->F = (int)F; c->D = (int)D; c->nb = (int)in->n_batch; c->nm = (int)in->n_micro;
    c->nsg = (int)nsg;
    c->bf = in->bottleneck_factor;
    c->h_batch.assign(in->batch, in->batch + in->n_batch);
    c->h_micro.assign(in->micro, in->micro + in->n_micro);
    size_t DD = (size_t)D * D;
    uint32_t nfm = in->fg_member_offset[F];
    uint32_t nsm = in->sg_member_offset[nsg];
    // arena layout: every array 16-byte aligned
    struct Seg { const void* src; size_t bytes; size_t off; };
    Seg seg[24];
    int ns = 0;
    size_t off = 0;
    auto add = [&](const void* src, size_t bytes) {
        seg[ns].src = src; seg[ns].bytes = bytes; seg[ns].off = off;
        off += (bytes + 15) & ~(size_t)15;
        return ns++;
    };
    const int i_fwd = add(in->fwd_flops, n * 8), i_bwd = add(in->bwd_input_flops, n * 8),
              i_wgt = add(in->bwd_weight_flops, n * 8), i_act = add(in->activation_out_bytes, n * 8),
              i_par = add(in->param_bytes, n * 8), i_b = add(in->batch, in->n_batch * 8),
              i_m = add(in->micro, in->n_micro * 8), i_pc = add(in->p_c, D * 8),
              i_mem = add(in->memory_bytes, D * 8), i_rank = add(in->id_rank, D * 4),
              i_pt = add(in->p_t, DD * 8), i_lat = add(in->latency, DD * 8),
              i_bw = add(in->bandwidth, DD * 8), i_foff = add(in->fg_member_offset, (F + 1) * 4),
              i_fmem = add(in->fg_members, nfm * 4), i_fcap = add(in->fg_capacity, F * 8),
              i_fbwi = add(in->fg_min_bw, F * 8), i_fbw = add(in->fg_min_bw, F * 8),
              i_fhas = add(in->fg_has_min_bw, F), i_fsg = add(in->fg_sg_offset, (F + 1) * 4),
              i_soff = add(in->sg_member_offset, (nsg + 1) * 4), i_smem = add(in->sg_members, nsm * 4),
              i_scap = add(in->sg_capacity, nsg * 8);
    if (c->arena_ev) CUDA_TRY(cudaEventSynchronize(c->arena_ev));  // last H2D done
    if (off > c->h_arena_cap) {
        if (c->h_arena) cudaFreeHost(c->h_arena);
        c->h_arena = nullptr;
        c->h_arena_cap = 0;
        CUDA_TRY(cudaHostAlloc((void**)&c->h_arena, off, cudaHostAllocDefault));
        c->h_arena_cap = off;
    }
    for (int i = 0; i < ns; ++i)
        if (seg[i].bytes) memcpy(c->h_arena + seg[i].off, seg[i].src, seg[i].bytes);
    CUDA_TRY(c->arena.ensure(off));
    CUDA_TRY(cudaMemcpyAsync(c->arena.p, c->h_arena, off, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaEventRecord(c->arena_ev, s));
    unsigned char* A = c->arena.p;
    c->fwd.p = (double*)(A + seg[i_fwd].off);
    c->bwd_in.p = (double*)(A + seg[i_bwd].off);
    c->bwd_w.p = (double*)(A + seg[i_wgt].off);
    c->act.p = (double*)(A + seg[i_act].off);
    c->param.p = (double*)(A + seg[i_par].off);
    c->batch.p = (long long*)(A + seg[i_b].off);
    c->micro.p = (long long*)(A + seg[i_m].off);
    c->p_c.p = (double*)(A + seg[i_pc].off);
    c->mem.p = (double*)(A + seg[i_mem].off);
    c->id_rank.p = (uint32_t*)(A + seg[i_rank].off);
    c->p_t.p = (double*)(A + seg[i_pt].off);
    c->lat.p = (double*)(A + seg[i_lat].off);
    c->bw.p = (double*)(A + seg[i_bw].off);
    c->fg_off.p = (uint32_t*)(A + seg[i_foff].off);
    c->fg_mem.p = (uint32_t*)(A + seg[i_fmem].off);
    c->fg_cap.p = (double*)(A + seg[i_fcap].off);
    c->fg_minbw_in.p = (double*)(A + seg[i_fbwi].off);
    c->fg_minbw.p = (double*)(A + seg[i_fbw].off);
    c->fg_has.p = (uint8_t*)(A + seg[i_fhas].off);
    c->fg_sg_off.p = (uint32_t*)(A + seg[i_fsg].off);
    c->sg_off.p = (uint32_t*)(A + seg[i_soff].off);
    c->sg_mem.p = (uint32_t*)(A + seg[i_smem].off);
    c->sg_cap.p = (double*)(A + seg[i_scap].off);
    c->arena_bytes = off;
    size_t N2 = (size_t)(n + 1) * (n + 1);
    CUDA_TRY(c->S.ensure(5 * N2));
    CUDA_TRY(c->g_tp_ok.ensure(F));
    CUDA_TRY(c->g_rf.ensure(nfm));
    CUDA_TRY(c->g_cf.ensure(nfm));
    CUDA_TRY(c->g_dp.ensure(nsg ? nsg : 1));
    CUDA_TRY(c->g_minmem.ensure(F));
    CUDA_TRY(c->sg_minmem.ensure(nsg ? nsg : 1));
    CUDA_TRY(c->stg.ensure((size_t)c->nm * F * N2));
    CUDA_TRY(c->scode.ensure((size_t)F * N2));
    CUDA_TRY(c->skind.ensure((size_t)F * N2));
    CUDA_TRY(c->C1.ensure((size_t)F * N2));
    CUDA_TRY(c->fbws.ensure((size_t)F * N2));
    CUDA_TRY(c->vtab.ensure((size_t)c->nm * F * ((size_t)n * (n + 1) / 2)));
    CUDA_TRY(c->gw.ensure((size_t)F * F));
    CUDA_TRY(c->xt.ensure((size_t)c->nm * F * F * ((n + 1) & ~1u)));
    CUDA_TRY(c->tpk.ensure((size_t)c->nm * F * ((size_t)n * (n + 1) / 2)));
    CUDA_TRY(c->tcol.ensure((size_t)c->nm * F * (n + 1)));
    CUDA_TRY(c->flagsbuf.ensure(1));
    CUDA_TRY(c->counter.ensure(1));
    CUDA_TRY(c->result.ensure(1));
    CUDA_TRY(c->err_idx.ensure(1));
    CUDA_TRY(c->blk.ensure(4096));  // >= the generic fix-up grid (no realloc mid-stream)
    CUDA_TRY(cudaMemsetAsync(c->counter.p, 0, sizeof(unsigned int), s));
    if (!c->binom.p) {
        // C(nn, r) for nn < 257, r <= GP_MAX_STAGES (composition unranking)
        std::vector<unsigned long long> tab((size_t)BINOM_ROWS * (GP_MAX_STAGES + 1), 0ull);
        for (int nn = 0; nn < BINOM_ROWS; ++nn)
            for (int r = 0; r <= GP_MAX_STAGES; ++r) tab[(size_t)nn * (GP_MAX_STAGES + 1) + r] = h_binom(nn, r);
        CUDA_TRY(upload(s, c->binom, tab.data(), tab.size()));
    }
    int st = run_tables(c, true);
    if (st != GP_OK) return st;
    // enumeration helpers depend on (n, k) only: rebuild when those change
    if (c->cache_n == (int)n && c->cache_k == (int)F) {
        c->loaded = true;
        return GP_OK;
    }
    c->cache_n = (int)n;
    c->cache_k = (int)F;
    c->tiles_ok = false;  // K3 tile table: built lazily by the sub-range path
    // K3 sweep run groups (see k3_sweep): full K3_SEG runs by a, then partial
    // runs grouped by length, longest first
    c->sweep_ok = false;
    if ((int)F >= 3 && (int)F <= (int)n) {
        int k = (int)F, nn = (int)n;
        std::vector<uint4> g;
        unsigned long long start = 0;
        for (int a = k - 2; a <= nn - 2; ++a) {
            unsigned long long rows = h_binom(a - 1, k - 3);
            int L = nn - 1 - a, nf = L / K3_SEG;
            if (rows && nf) {
                g.push_back(make_uint4((unsigned)start, (unsigned)a | ((unsigned)K3_SEG << 16),
                                       (unsigned)rows, (unsigned)nf));
                start += rows * nf;
            }
        }
        for (int len = K3_SEG - 1; len >= 1; --len)
            for (int a = k - 2; a <= nn - 2; ++a) {
                int L = nn - 1 - a;
                if (L % K3_SEG != len) continue;
                unsigned long long rows = h_binom(a - 1, k - 3);
                if (!rows) continue;
                g.push_back(make_uint4((unsigned)start, (unsigned)a | ((unsigned)len << 16),
                                       (unsigned)rows, 0u));
                start += rows;
            }
        // colex list of (k-3)-subsets of [1, n-3]: the subsets of [1, a-1]
        // are exactly its first C(a-1, k-3) entries
        std::vector<uint8_t> pre;
        unsigned long long npre = (k > 3) ? h_binom(nn - 3, k - 3) : 1;
        bool pre_ok = npre <= (1ull << 22);
        if (pre_ok && k > 3) {
            int m = k - 3;
            std::vector<int> cmb(m);
            for (int i = 0; i < m; ++i) cmb[i] = i + 1;
            pre.assign((size_t)npre * 16, 0);
            for (unsigned long long r = 0; r < npre; ++r) {
                for (int i = 0; i < m; ++i) pre[r * 16 + i] = (uint8_t)cmb[i];
                // colex successor: smallest i with cmb[i] + 1 < cmb[i+1] (or last)
                int i = 0;
                while (i < m - 1 && cmb[i] + 1 == cmb[i + 1]) ++i;
                ++cmb[i];
                for (int j = 0; j < i; ++j) cmb[j] = j + 1;
            }
        }
        if (pre_ok && start < (1ull << 31) && !g.empty()) {
            if (k > 3) CUDA_TRY(upload(s, c->prefixes, pre.data(), pre.size()));
            std::vector<unsigned long long> bk((size_t)(nn + 1) * (k + 1) + 2, 0ull);
            for (int a = 0; a <= nn; ++a)
                for (int r = 0; r <= k; ++r) bk[(size_t)a * (k + 1) + r] = h_binom(a, r);
            CUDA_TRY(upload(s, c->bnk, bk.data(), bk.size()));
            CUDA_TRY(upload(s, c->groups, g.data(), g.size()));
            c->ngroups = (int)g.size();
            c->sweep_W = (unsigned)start;
            c->sweep_ok = true;
        }
    }
    c->loaded = true;
    return GP_OK;
}

static int ensure_tiles(gp_ctx* c) {
    if (c->tiles_ok) return GP_OK;
    int n = c->n, F = c->F;
    if (F >= 3 && F <= n) {
        unsigned long long NC = h_binom(n - 1, F - 1);
        unsigned long long ntiles = (NC + K3_TILE - 1) / K3_TILE;
        if (ntiles <= (1ull << 22)) {
            CUDA_TRY(c->tiles.ensure(ntiles * 16));
            k_tiles<<<(unsigned)((ntiles + 127) / 128), 128, 0, c->stream>>>(n, F, ntiles, c->tiles.p);
            CUDA_TRY(cudaGetLastError());
            c->tiles_ok = true;
        }
    }
    return GP_OK;
}

int gp_set_bandwidth(gp_ctx* c, const double* bandwidth) {
    if (!c || !c->loaded || !bandwidth) return fail(GP_ERR_INPUT, "context not loaded");
    CUDA_TRY(cudaSetDevice(c->device));
    size_t DD = (size_t)c->D * c->D;
    CUDA_TRY(cudaMemcpyAsync(c->bw.p, bandwidth, DD * sizeof(double), cudaMemcpyHostToDevice,
                             c->stream));
    DevInst I = c->view();
    k1_minbw<<<(c->F + 31) / 32, 32, 0, c->stream>>>(I, c->fg_minbw.p);
    CUDA_TRY(cudaGetLastError());
    return run_tables(c, false);
}

int gp_eval_batch_device(gp_ctx* c, uint32_t k, uint64_t n, const uint8_t* d_order,
                         const uint8_t* d_counts, const uint8_t* d_bm, double* d_cost,
                         uint8_t* d_status) {
    if (!c || !c->loaded) return fail(GP_ERR_INPUT, "context not loaded");
    if (k < 1 || k > GP_MAX_STAGES) return fail(GP_ERR_INPUT, "k=%u outside [1,%d]", k, GP_MAX_STAGES);
    if (n == 0) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    DevInst I = c->view();
    unsigned blocks = (unsigned)((n + 255) / 256);
    k2_eval_batch<<<blocks, 256, 0, c->stream>>>(I, (int)k, (long long)n, d_order, d_counts, d_bm,
                                                 d_cost, d_status);
    CUDA_TRY(cudaGetLastError());
    return GP_OK;
}

int gp_eval_batch(gp_ctx* c, uint32_t k, uint64_t n, const uint8_t* order, const uint8_t* counts,
                  const uint8_t* bm, double* cost, uint8_t* status) {
    if (!c || !c->loaded) return fail(GP_ERR_INPUT, "context not loaded");
    if (n == 0) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    CUDA_TRY(c->b_order.ensure(n * k));
    CUDA_TRY(c->b_counts.ensure(n * k));
    CUDA_TRY(c->b_bm.ensure(n));
    CUDA_TRY(c->b_cost.ensure(n));
    CUDA_TRY(c->b_status.ensure(n));
    CUDA_TRY(cudaMemcpyAsync(c->b_order.p, order, n * k, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->b_counts.p, counts, n * k, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->b_bm.p, bm, n, cudaMemcpyHostToDevice, s));
    int st = gp_eval_batch_device(c, k, n, c->b_order.p, c->b_counts.p, c->b_bm.p, c->b_cost.p,
                                  c->b_status.p);
    if (st != GP_OK) return st;
    CUDA_TRY(cudaMemcpyAsync(cost, c->b_cost.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(status, c->b_status.p, n, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return GP_OK;
}

static unsigned long long h_fact(int k) {
    unsigned long long f = 1;
    for (int i = 2; i <= k; ++i) f *= (unsigned long long)i;
    return f;
}

int gp_space_size(gp_ctx* c, uint64_t* out) {
    if (!c || !c->loaded || !out) return fail(GP_ERR_INPUT, "context not loaded");
    int k = c->F;
    *out = (k > c->n) ? 0 : (uint64_t)c->nb * c->nm * h_fact(k) * h_binom(c->n - 1, k - 1);
    return GP_OK;
}

// Sweep launch over items [item_lo, item_hi) of (mi * k! + order).
static int launch_sweep(gp_ctx* c, const RangeGeom& R, unsigned long long item_lo,
                        unsigned long long item_hi, int mode, const uint32_t* dflags) {
    cudaStream_t s = c->stream;
    const int k = R.k, n = c->n;
    size_t ntri = (size_t)n * (n + 1) / 2;
    size_t nxp = (size_t)((n + 1) & ~1);
    size_t smem0 = 16 + (((size_t)(n + 1) * (k + 1) * 8 + 15) & ~(size_t)15) + (size_t)c->ngroups * 16;
    size_t smem1 = smem0 + ntri * 16 + (n + 1) * 16 + 3 * nxp * 8 + (size_t)n * 16;
    size_t smem2 = smem1 + ntri * 16;
    if (mode == 2 && smem2 > (size_t)c->smem_max) mode = 1;
    if (mode == 1 && smem1 > (size_t)c->smem_max) mode = 0;
    size_t smem = mode == 2 ? smem2 : (mode == 1 ? smem1 : smem0);
    typedef void (*SwFn)(DevInst, SweepGeom, ArgminScratch, const unsigned long long*,
                         const uint32_t*);
    static const SwFn table[3][4] = {
        {k3_sweep<0, 1>, k3_sweep<0, 2>, k3_sweep<0, 3>, k3_sweep<0, 4>},
        {k3_sweep<1, 1>, k3_sweep<1, 2>, k3_sweep<1, 3>, k3_sweep<1, 4>},
        {k3_sweep<2, 1>, k3_sweep<2, 2>, k3_sweep<2, 3>, k3_sweep<2, 4>}};
    SwFn kern = table[mode][c->nb - 1];
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, K3S_THREADS, smem));
    unsigned long long resident = (unsigned long long)(per_sm > 0 ? per_sm : 1) * c->n_sms;
    unsigned long long items = item_hi - item_lo;
    unsigned long long tasks = (c->sweep_W + 31) / 32;
    unsigned long long cpi = items >= resident ? 1 : resident / items;
    unsigned long long cap = (tasks + (K3S_THREADS / 32) - 1) / (K3S_THREADS / 32);
    if (cpi > cap) cpi = cap;
    if (cpi < 1) cpi = 1;
    unsigned long long grid = items * cpi;
    if (grid > 0x7fffffffull) return fail(GP_ERR_INPUT, "item range too large for one launch");
    SweepGeom G;
    G.k = k;
    G.nbm = R.nbm;
    G.NC = R.NC;
    G.NP = R.NP;
    G.item0 = item_lo;
    G.cpi = cpi;
    G.W = c->sweep_W;
    G.ngroups = c->ngroups;
    G.groups = c->groups.p;
    G.prefixes = c->prefixes.p;
    G.bnk = c->bnk.p;
    G.items = (unsigned int)items;
    G.tpk = c->tpk.p;
    G.tcol = c->tcol.p;
    G.xt = c->xt.p;
    G.s_tpk = G.s_tcol = G.s_xt = 0;
    G.gsteps = 1;
    while (G.gsteps * 2 <= c->ngroups) G.gsteps *= 2;
    CUDA_TRY(c->item_ctr.ensure(items));
    CUDA_TRY(cudaMemsetAsync(c->item_ctr.p, 0, items * sizeof(unsigned int), s));
    G.item_ctr = c->item_ctr.p;
    CUDA_TRY(c->blk.ensure(grid));
    ArgminScratch S;
    S.blk = c->blk.p;
    S.counter = c->counter.p;
    S.result = c->result.p;
    S.err = nullptr;
    S.err_idx = c->err_idx.p;
    c->last_geom = R;
    DevInst I = c->view();
    kern<<<(unsigned)grid, K3S_THREADS, smem, s>>>(I, G, S, c->binom.p, dflags);
    CUDA_TRY(cudaGetLastError());
    return GP_OK;
}

// Generic status-tracking pass that runs only when the device flags are set.
static int launch_fixup(gp_ctx* c, const RangeGeom& G) {
    unsigned long long grid = (G.hi - G.lo + 255) / 256;
    unsigned long long gmax = (unsigned long long)c->n_sms * 16;
    if (grid > gmax) grid = gmax;
    if (grid < 1) grid = 1;
    CUDA_TRY(c->blk.ensure(grid));
    ArgminScratch S;
    S.blk = c->blk.p;
    S.counter = c->counter.p;
    S.result = c->result.p;
    S.err = nullptr;
    S.err_idx = c->err_idx.p;
    DevInst I = c->view();
    k3_argmin_generic<<<(unsigned)grid, 256, 0, c->stream>>>(I, G, S, c->flagsbuf.p);
    CUDA_TRY(cudaGetLastError());
    return GP_OK;
}

int gp_argmin_range_async(gp_ctx* c, uint64_t lo, uint64_t hi) {
    if (!c || !c->loaded) return fail(GP_ERR_INPUT, "context not loaded");
    int k = c->F;
    uint64_t total;
    gp_space_size(c, &total);
    if (hi > total) hi = total;
    if (lo > hi) lo = hi;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    RangeGeom G;
    G.k = k;
    G.nbm = c->nb * c->nm;
    G.NC = h_binom(c->n - 1, k - 1);
    G.NP = h_fact(k);
    G.lo = lo;
    G.hi = hi;
    G.items_mode = 0;
    G.it_lo = 0;
    G.it_span = 1;
    G.nm = c->nm;
    G.item_ctr = nullptr;
    G.tiles = nullptr;
    c->last_lo = lo;
    c->last_hi = hi;
    ArgminScratch S;
    CUDA_TRY(cudaMemsetAsync(c->err_idx.p, 0xFF, sizeof(unsigned long long), s));  // = ~0
    DevInst I = c->view();
    // table flags (error entries, overflow) force the status-tracking kernel;
    // while the async read-back is pending, launch the fast kernel with a
    // device-side check plus a generic fix-up that runs only if flagged
    const int fl = known_flags(c);
    bool generic = fl > 0 || k < 3 || c->force_mode == 3 || c->nb > 4;
    const bool pending = fl < 0 && !generic;
    const uint32_t* dflags = pending ? c->flagsbuf.p : nullptr;
    unsigned long long grid;
    // fast-path kernel variant by shared-memory fit (see k3_argmin)
    size_t ntri = (size_t)c->n * (c->n + 1) / 2;
    size_t nxp = (size_t)((c->n + 1) & ~1);
    size_t smem0 = 16 + (((size_t)(c->n + 1) * (k + 1) * 8 + 15) & ~(size_t)15);
    size_t smem1 = smem0 + ntri * 16 + (c->n + 1) * 16 + 3 * nxp * 8 + (size_t)c->n * 16;
    size_t smem2 = smem1 + ntri * 16;
    int mode = smem2 <= (size_t)c->smem_max ? 2 : (smem1 <= (size_t)c->smem_max ? 1 : 0);
    if (c->force_mode >= 0 && c->force_mode < mode) mode = c->force_mode;
    size_t smem = mode == 2 ? smem2 : (mode == 1 ? smem1 : smem0);
    typedef void (*K3Fn)(DevInst, RangeGeom, ArgminScratch, const unsigned long long*,
                         const uint32_t*);
    static const K3Fn table[3][4] = {
        {k3_argmin<0, 1>, k3_argmin<0, 2>, k3_argmin<0, 3>, k3_argmin<0, 4>},
        {k3_argmin<1, 1>, k3_argmin<1, 2>, k3_argmin<1, 3>, k3_argmin<1, 4>},
        {k3_argmin<2, 1>, k3_argmin<2, 2>, k3_argmin<2, 3>, k3_argmin<2, 4>}};
    K3Fn kern = generic ? nullptr : table[mode][c->nb - 1];
    if (!generic && lo == 0 && hi == total && hi > 0 && c->sweep_ok && c->force_mode != 4) {
        c->last_generic = false;
        CUDA_TRY(c->blk.ensure(1));
        int st = launch_sweep(c, G, 0, (unsigned long long)c->nm * G.NP, mode, dflags);
        if (st != GP_OK || !pending) return st;
        return launch_fixup(c, G);
    }
    if (hi == lo) {
        generic = true;
        grid = 1;
    } else if (generic) {
        grid = (hi - lo + 255) / 256;
        unsigned long long gmax = (unsigned long long)c->n_sms * 16;  // grid-stride
        if (grid > gmax) grid = gmax;
    } else {
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, K3_THREADS, smem));
        unsigned long long resident = (unsigned long long)(per_sm > 0 ? per_sm : 1) * c->n_sms;
        // items = (micro index, order); a range inside one batch block touches
        // a contiguous run of them, a wider range all of them
        unsigned long long per_b = (unsigned long long)c->nm * G.NP;
        unsigned long long blk_lo = lo / G.NC, blk_hi = (hi - 1) / G.NC;  // (bm, perm) blocks
        unsigned long long item_first, items;
        if (blk_lo / per_b == blk_hi / per_b) {
            item_first = blk_lo % per_b;
            items = blk_hi % per_b - item_first + 1;
        } else {
            item_first = 0;
            items = per_b;
        }
        // CTAs per item: fill the resident slots, at most one per 8 tiles
        unsigned long long tiles_per_item = (G.NC + K3_TILE - 1) / K3_TILE;
        unsigned long long cpi = items >= resident ? 1 : resident / items;
        unsigned long long cap = (tiles_per_item + 7) / 8;
        if (cpi > cap) cpi = cap;
        if (cpi < 1) cpi = 1;
        G.item0 = item_first;
        G.chunk = 0;
        G.chunks_per_item = cpi;
        grid = items * cpi;
        CUDA_TRY(c->item_ctr.ensure(items));
        CUDA_TRY(cudaMemsetAsync(c->item_ctr.p, 0, items * sizeof(unsigned int), s));
        G.item_ctr = c->item_ctr.p;
        int ts = ensure_tiles(c);
        if (ts != GP_OK) return ts;
        G.tiles = c->tiles_ok ? c->tiles.p : nullptr;
    }
    c->last_generic = generic;
    if (grid > 0x7fffffffull) return fail(GP_ERR_INPUT, "range too large for one launch");
    CUDA_TRY(c->blk.ensure(grid));
    S.blk = c->blk.p;
    S.counter = c->counter.p;
    S.result = c->result.p;
    S.err = nullptr;
    S.err_idx = c->err_idx.p;
    c->last_geom = G;
    if (generic) {
        if (hi == lo) G.hi = G.lo;  // one empty CTA writes the neutral key
        k3_argmin_generic<<<(unsigned)grid, 256, 0, s>>>(I, G, S, nullptr);
    } else {
        kern<<<(unsigned)grid, K3_THREADS, smem, s>>>(I, G, S, c->binom.p, dflags);
        CUDA_TRY(cudaGetLastError());
        if (pending) return launch_fixup(c, G);
    }
    CUDA_TRY(cudaGetLastError());
    return GP_OK;
}

static void h_unrank_perm(int k, unsigned long long r, uint8_t* perm) {
    uint8_t pool[GP_MAX_STAGES];
    for (int i = 0; i < k; ++i) pool[i] = (uint8_t)i;
    int left = k;
    for (int i = 0; i < k; ++i) {
        unsigned long long f = h_fact(k - 1 - i);
        unsigned long long q = r / f;
        r %= f;
        perm[i] = pool[q];
        for (int j = (int)q; j + 1 < left; ++j) pool[j] = pool[j + 1];
        --left;
    }
}

static void h_unrank_counts(int n, int k, unsigned long long r, uint8_t* counts) {
    int prev = 0;
    for (int j = 1; j < k; ++j) {
        for (int q = prev + 1;; ++q) {
            unsigned long long cnt = h_binom(n - q - 1, k - 1 - j);
            if (r < cnt) { counts[j - 1] = (uint8_t)(q - prev); prev = q; break; }
            r -= cnt;
        }
    }
    counts[k - 1] = (uint8_t)(n - prev);
}

int gp_argmin_fetch(gp_ctx* c, gp_best* out) {
    if (!c || !c->loaded || !out) return fail(GP_ERR_INPUT, "context not loaded");
    CUDA_TRY(cudaSetDevice(c->device));
    Key r;
    unsigned long long err;
    CUDA_TRY(cudaMemcpyAsync(&r, c->result.p, sizeof(Key), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaMemcpyAsync(&err, c->err_idx.p, sizeof(err), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    memset(out, 0, sizeof(*out));
    const RangeGeom& G = c->last_geom;
    out->k = (uint32_t)G.k;
    out->evaluated = c->last_hi - c->last_lo;
    if (err != ~0ull) {
        int code = (int)(err & 15ull);
        return fail(code, "candidate %llu raises status %d", err >> 4, code);
    }
    if (r.tie == ~0ull) return fail(GP_ERR_NO_FEASIBLE, "empty candidate range");
    unsigned long long bm = r.tie % (unsigned long long)G.nbm;
    unsigned long long pc = r.tie / (unsigned long long)G.nbm;
    unsigned long long comp = pc % G.NC, perm = pc / G.NC;
    out->cost = r.cost;
    out->index = (bm * G.NP + perm) * G.NC + comp;
    out->batch_index = (uint32_t)(bm / c->nm);
    out->micro_index = (uint32_t)(bm % c->nm);
    h_unrank_perm(G.k, perm, out->order);
    h_unrank_counts(c->n, G.k, comp, out->counts);
    return GP_OK;
}

int gp_argmin_range(gp_ctx* c, uint64_t lo, uint64_t hi, gp_best* out) {
    int st = gp_argmin_range_async(c, lo, hi);
    if (st != GP_OK) return st;
    return gp_argmin_fetch(c, out);
}

int gp_argmin_bnb_async(gp_ctx* c) {
    if (!c || !c->loaded) return fail(GP_ERR_INPUT, "context not loaded");
    const int k = c->F, n = c->n;
    uint64_t total;
    gp_space_size(c, &total);
    int fl = known_flags(c);
    if (fl < 0) {
        CUDA_TRY(cudaEventSynchronize(c->flags_ev));
        fl = known_flags(c);
    }
    if (fl != 0 || k < 2 || total == 0)  // error entries / trivial spaces: exhaustive path
        return gp_argmin_range_async(c, 0, total);
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    RangeGeom R;
    memset(&R, 0, sizeof(R));
    R.k = k; R.nbm = c->nb * c->nm; R.NC = h_binom(n - 1, k - 1); R.NP = h_fact(k);
    R.lo = 0; R.hi = total; R.nm = c->nm;
    c->last_geom = R;
    c->last_lo = 0;
    c->last_hi = total;
    const unsigned long long items = (unsigned long long)R.nbm * R.NP;
    if (items > 0x7fffffffull) return fail(GP_ERR_INPUT, "too many items for one launch");
    CUDA_TRY(c->gbest.ensure(1));
    // all-ones bits: above every finite cost as u64, a NaN bound as double
    // (prunes nothing until a finite cost is found)
    CUDA_TRY(cudaMemsetAsync(c->gbest.p, 0xFF, sizeof(unsigned long long), s));
    CUDA_TRY(cudaMemsetAsync(c->err_idx.p, 0xFF, sizeof(unsigned long long), s));
    CUDA_TRY(c->blk.ensure(items > 4096 ? items : 4096));
    ArgminScratch S;
    S.blk = c->blk.p; S.counter = c->counter.p; S.result = c->result.p; S.err = nullptr;
    S.err_idx = c->err_idx.p;
    BnbGeom G;
    G.k = k; G.nbm = R.nbm; G.NC = R.NC; G.NP = R.NP; G.gbest = c->gbest.p;
    DevInst I = c->view();
    const size_t smem = (size_t)k * (n + 1) * sizeof(double);
    k4_bnb<<<(unsigned)items, 32, smem, s>>>(I, G, S, c->binom.p);
    CUDA_TRY(cudaGetLastError());
    return GP_OK;
}

int gp_argmin_items_async(gp_ctx* c, uint64_t item_lo, uint64_t item_hi) {
    if (!c || !c->loaded) return fail(GP_ERR_INPUT, "context not loaded");
    const int k = c->F;
    uint64_t total;
    gp_space_size(c, &total);
    const unsigned long long NP = h_fact(k), NC = h_binom(c->n - 1, k - 1);
    const unsigned long long n_items = total ? (unsigned long long)c->nm * NP : 0;
    if (item_hi > n_items) item_hi = n_items;
    if (item_lo > item_hi) item_lo = item_hi;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    RangeGeom G;
    memset(&G, 0, sizeof(G));
    G.k = k;
    G.nbm = c->nb * c->nm;
    G.NC = NC;
    G.NP = NP;
    G.nm = c->nm;
    G.items_mode = 1;
    G.it_lo = item_lo;
    G.it_span = item_hi > item_lo ? item_hi - item_lo : 1;
    G.lo = 0;
    G.hi = (unsigned long long)c->nb * (item_hi - item_lo) * NC;
    c->last_lo = 0;
    c->last_hi = G.hi;
    c->last_geom = G;
    CUDA_TRY(cudaMemsetAsync(c->err_idx.p, 0xFF, sizeof(unsigned long long), s));
    const int fl = known_flags(c);
    const bool generic = fl > 0 || k < 3 || c->force_mode == 3 || c->force_mode == 4 ||
                         c->nb > 4 || !c->sweep_ok || G.hi == 0;
    if (!generic) {
        int mode = c->force_mode >= 0 && c->force_mode <= 2 ? c->force_mode : 2;
        const uint32_t* dflags = fl < 0 ? c->flagsbuf.p : nullptr;
        int st = launch_sweep(c, G, item_lo, item_hi, mode, dflags);
        if (st != GP_OK || fl >= 0) return st;
        return launch_fixup(c, G);
    }
    unsigned long long grid = G.hi ? (G.hi + 255) / 256 : 1;
    unsigned long long gmax = (unsigned long long)c->n_sms * 16;
    if (grid > gmax) grid = gmax;
    ArgminScratch S;
    S.blk = c->blk.p;
    S.counter = c->counter.p;
    S.result = c->result.p;
    S.err = nullptr;
    S.err_idx = c->err_idx.p;
    DevInst I = c->view();
    k3_argmin_generic<<<(unsigned)grid, 256, 0, s>>>(I, G, S, nullptr);
    CUDA_TRY(cudaGetLastError());
    return GP_OK;
}

// arg-min + on-device winner detail + D2H of the SolveOut record (no sync)
static int enqueue_solve(gp_ctx* c, uint64_t lo, uint64_t hi) {
    int st = gp_argmin_range_async(c, lo, hi);
    if (st != GP_OK) return st;
    const RangeGeom& G = c->last_geom;
    CUDA_TRY(c->dsolve.ensure(1));
    DevInst I = c->view();
    k_solve_detail<<<1, 32, 0, c->stream>>>(I, G.k, G.NC, G.NP, G.nbm, c->result.p, c->err_idx.p,
                                            c->binom.p, c->dsolve.p);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(c->h_solve, c->dsolve.p, sizeof(SolveOut), cudaMemcpyDeviceToHost,
                             c->stream));
    return GP_OK;
}

// decode the SolveOut record that landed in pinned memory
static int finish_solve(gp_ctx* c, gp_best* best, gp_plan_info* info) {
    const RangeGeom& G = c->last_geom;
    const SolveOut& o = *c->h_solve;
    memset(best, 0, sizeof(*best));
    best->k = (uint32_t)G.k;
    best->evaluated = c->last_hi - c->last_lo;
    if (o.err != ~0ull) {
        int code = (int)(o.err & 15ull);
        return fail(code, "candidate %llu raises status %d", o.err >> 4, code);
    }
    if (o.key.tie == ~0ull) return fail(GP_ERR_NO_FEASIBLE, "empty candidate range");
    unsigned long long bmv = o.key.tie % (unsigned long long)G.nbm;
    unsigned long long pc = o.key.tie / (unsigned long long)G.nbm;
    best->cost = o.key.cost;
    best->index = (bmv * G.NP + pc / G.NC) * G.NC + pc % G.NC;
    best->batch_index = (uint32_t)(bmv / c->nm);
    best->micro_index = (uint32_t)(bmv % c->nm);
    memcpy(best->order, o.order, sizeof(best->order));
    memcpy(best->counts, o.counts, sizeof(best->counts));
    if (info) *info = o.info;
    if (o.status != GP_OK) return fail(o.status, "winner raises status %d", o.status);
    return GP_OK;
}

int gp_solve(gp_ctx* c, uint64_t lo, uint64_t hi, gp_best* best, gp_plan_info* info) {
    if (!c || !c->loaded || !best) return fail(GP_ERR_INPUT, "context not loaded");
    int st = enqueue_solve(c, lo, hi);
    if (st != GP_OK) return st;
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return finish_solve(c, best, info);
}

// shape of an instance: everything the arena layout and the launch geometry
// depend on (a CUDA graph captured for one shape replays for any instance of
// the same shape)
static void instance_shape(const gp_instance* in, unsigned long long* key) {
    key[0] = in->n_layers; key[1] = in->n_devices; key[2] = in->n_fgs;
    key[3] = in->n_batch; key[4] = in->n_micro;
    key[5] = in->fg_member_offset[in->n_fgs];
    key[6] = in->fg_sg_offset[in->n_fgs];
    key[7] = in->sg_member_offset[in->fg_sg_offset[in->n_fgs]];
    unsigned long long h = 1469598103934665603ull;  // group structure (CSR offsets)
    for (uint32_t f = 0; f <= in->n_fgs; ++f) {
        h = (h ^ in->fg_member_offset[f]) * 1099511628211ull;
        h = (h ^ in->fg_sg_offset[f]) * 1099511628211ull;
    }
    for (uint32_t g = 0; g <= in->fg_sg_offset[in->n_fgs]; ++g)
        h = (h ^ in->sg_member_offset[g]) * 1099511628211ull;
    for (uint32_t i = 0; i < in->n_batch; ++i) h = (h ^ (unsigned long long)in->batch[i]) * 1099511628211ull;
    for (uint32_t i = 0; i < in->n_micro; ++i) h = (h ^ (unsigned long long)in->micro[i]) * 1099511628211ull;
    key[8] = h;
}

int gp_replan(gp_ctx* c, const gp_instance* in, gp_best* best, gp_plan_info* info) {
    if (!c || !in || !best) return fail(GP_ERR_INPUT, "null argument");
    unsigned long long key[10];
    instance_shape(in, key);
    memcpy(&key[9], &in->bottleneck_factor, sizeof(double));
    const bool same = c->graph_exec && memcmp(key, c->graph_key, sizeof(key)) == 0 &&
                      c->graph_gen == __atomic_load_n(&g_alloc_gen, __ATOMIC_RELAXED);
    cudaStream_t s = c->stream;
    if (!same) {
        // first instance of this shape: regular load (allocations, helpers),
        // then capture H2D + K1 + K3 + detail + D2H as one graph
        int st = gp_ctx_load(c, in);
        if (st != GP_OK) return st;
        CUDA_TRY(cudaStreamSynchronize(s));
        if (c->graph_exec) { cudaGraphExecDestroy(c->graph_exec); c->graph_exec = nullptr; }
        uint64_t total;
        gp_space_size(c, &total);
        // make every buffer the graph touches exist before capturing
        CUDA_TRY(c->dsolve.ensure(1));
        CUDA_TRY(c->item_ctr.ensure((size_t)c->nm * h_fact(c->F) + 1));
        c->capturing = true;
        CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
        cudaError_t ce = cudaMemcpyAsync(c->arena.p, c->h_arena, c->arena_bytes,
                                         cudaMemcpyHostToDevice, s);
        int st2 = ce == cudaSuccess ? GP_OK : fail(GP_ERR_CUDA, "capture: %s", cudaGetErrorString(ce));
        if (st2 == GP_OK) {
            DevInst I = c->view();
            cudaMemsetAsync(c->flagsbuf.p, 0, sizeof(uint32_t), s);
            const int gw_blocks = (c->F * c->F + 3) / 4;
            k1_phase1<<<5 + c->F + gw_blocks, 128, 0, s>>>(I);
            long long ns = (long long)c->F * (c->n + 1) * (c->n + 1);
            long long nx = (long long)c->nm * c->F * c->F * c->n;
            k1_phase2<<<(unsigned)((ns + nx + 127) / 128), 128, 0, s>>>(I, ns);
            cudaMemcpyAsync(c->h_flags, c->flagsbuf.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
            cudaEventRecord(c->flags_ev, s);
            c->flags_known = false;
            st2 = enqueue_solve(c, 0, total);
        }
        cudaGraph_t g = nullptr;
        cudaError_t ee = cudaStreamEndCapture(s, &g);
        c->capturing = false;
        if (st2 != GP_OK) { if (g) cudaGraphDestroy(g); return st2; }
        if (ee != cudaSuccess) return fail(GP_ERR_CUDA, "graph capture: %s", cudaGetErrorString(ee));
        ee = cudaGraphInstantiate(&c->graph_exec, g, 0);
        cudaGraphDestroy(g);
        if (ee != cudaSuccess) { c->graph_exec = nullptr; return fail(GP_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(ee)); }
        memcpy(c->graph_key, key, sizeof(key));
        c->graph_gen = __atomic_load_n(&g_alloc_gen, __ATOMIC_RELAXED);
        c->graph_geom = c->last_geom;
        c->graph_lo = c->last_lo;
        c->graph_hi = c->last_hi;
    } else {
        // same shape: refill the pinned arena in place (same offsets)
        if (c->arena_ev) CUDA_TRY(cudaEventSynchronize(c->arena_ev));
        const uint32_t n = in->n_layers, D = in->n_devices, F = in->n_fgs;
        const size_t DD = (size_t)D * D;
        const uint32_t nsg = in->fg_sg_offset[F];
        const void* src[23] = {in->fwd_flops, in->bwd_input_flops, in->bwd_weight_flops,
                               in->activation_out_bytes, in->param_bytes, in->batch, in->micro,
                               in->p_c, in->memory_bytes, in->id_rank, in->p_t, in->latency,
                               in->bandwidth, in->fg_member_offset, in->fg_members, in->fg_capacity,
                               in->fg_min_bw, in->fg_min_bw, in->fg_has_min_bw, in->fg_sg_offset,
                               in->sg_member_offset, in->sg_members, in->sg_capacity};
        const size_t bytes[23] = {n * 8ull, n * 8ull, n * 8ull, n * 8ull, n * 8ull,
                                  in->n_batch * 8ull, in->n_micro * 8ull, D * 8ull, D * 8ull,
                                  D * 4ull, DD * 8, DD * 8, DD * 8, (F + 1) * 4ull,
                                  in->fg_member_offset[F] * 4ull, F * 8ull, F * 8ull, F * 8ull,
                                  (size_t)F, (F + 1) * 4ull, (nsg + 1) * 4ull,
                                  in->sg_member_offset[nsg] * 4ull, nsg * 8ull};
        size_t off = 0;
        for (int i = 0; i < 23; ++i) {
            if (bytes[i]) memcpy(c->h_arena + off, src[i], bytes[i]);
            off += (bytes[i] + 15) & ~(size_t)15;
        }
        c->bf = in->bottleneck_factor;
        c->last_geom = c->graph_geom;
        c->last_lo = c->graph_lo;
        c->last_hi = c->graph_hi;
    }
    CUDA_TRY(cudaGraphLaunch(c->graph_exec, s));
    CUDA_TRY(cudaEventRecord(c->arena_ev, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    c->flags_known = false;
    c->loaded = true;
    return finish_solve(c, best, info);
}

int gp_plan_detail(gp_ctx* c, uint32_t k, const uint8_t* order, const uint8_t* counts, uint32_t bm,
                   gp_plan_info* out) {
    if (!c || !c->loaded || !out) return fail(GP_ERR_INPUT, "context not loaded");
    if (k < 1 || k > GP_MAX_STAGES || bm >= (uint32_t)(c->nb * c->nm))
        return fail(GP_ERR_INPUT, "bad candidate");
    int sum = 0;
    unsigned seen = 0;
    for (uint32_t s = 0; s < k; ++s) {
        if (order[s] >= c->F || ((seen >> order[s]) & 1u) || counts[s] == 0)
            return fail(GP_ERR_INPUT, "stage order must use distinct groups and positive counts");
        seen |= 1u << order[s];
        sum += counts[s];
    }
    if (sum > c->n) return fail(GP_ERR_INPUT, "counts exceed the layer count");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    CUDA_TRY(c->b_order.ensure(GP_MAX_STAGES));
    CUDA_TRY(c->b_counts.ensure(GP_MAX_STAGES));
    CUDA_TRY(c->info.ensure(1));
    CUDA_TRY(c->dstatus.ensure(1));
    CUDA_TRY(cudaMemcpyAsync(c->b_order.p, order, k, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->b_counts.p, counts, k, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemsetAsync(c->info.p, 0, sizeof(gp_plan_info), s));
    DevInst I = c->view();
    k_plan_detail<<<1, 32, 0, s>>>(I, (int)k, c->b_order.p, c->b_counts.p, (int)bm, c->info.p,
                                   c->dstatus.p);
    CUDA_TRY(cudaGetLastError());
    int status = 0;
    CUDA_TRY(cudaMemcpyAsync(out, c->info.p, sizeof(gp_plan_info), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&status, c->dstatus.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (status != GP_OK) return fail(status, "candidate raises status %d", status);
    return GP_OK;
}

__global__ void k_group_info(DevInst I, int f, gp_group_info* out) {
    if (threadIdx.x != 0) return;
    int m0 = I.fg_off[f], m1 = I.fg_off[f + 1];
    int s0 = I.fg_sg_off[f], s1 = I.fg_sg_off[f + 1];
    out->n_members = (uint32_t)(m1 - m0);
    out->n_sgs = (uint32_t)(s1 - s0);
    out->tp_ok = I.g_tp_ok[f];
    for (int x = m0; x < m1; ++x) { out->tp_row[x - m0] = I.g_rf[x]; out->tp_col[x - m0] = I.g_cf[x]; }
    for (int g = s0; g < s1; ++g) out->dp_fraction[g - s0] = I.g_dp[g];
}

int gp_group_splits(gp_ctx* c, uint32_t f, gp_group_info* out) {
    if (!c || !c->loaded || !out || f >= (uint32_t)c->F) return fail(GP_ERR_INPUT, "bad group");
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(c->ginfo.ensure(1));
    CUDA_TRY(cudaMemsetAsync(c->ginfo.p, 0, sizeof(gp_group_info), c->stream));
    DevInst I = c->view();
    k_group_info<<<1, 32, 0, c->stream>>>(I, (int)f, c->ginfo.p);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out, c->ginfo.p, sizeof(gp_group_info), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return GP_OK;
}

// ---- diagnostics: FP64 add issue-rate microbenchmark --------------------------------
// 8 independent DADD chains per thread so the FP64 pipe, not latency, bounds it.
__global__ void k_fp64_peak(double* sink, int iters, double step) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
           a6 = a0 + 6, a7 = a0 + 7;
    for (int i = 0; i < iters; ++i) {
        a0 = a0 + step; a1 = a1 + step; a2 = a2 + step; a3 = a3 + step;
        a4 = a4 + step; a5 = a5 + step; a6 = a6 + step; a7 = a7 + step;
    }
    double r = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (r == 12345.678) sink[blockIdx.x] = r;  // never true; keeps the chains live
}

int gp_sim_1f1b_device(gp_ctx* c, const gp_timing* d_timings, uint64_t n, uint32_t iterations,
                       double* d_makespan, uint8_t* d_status) {
    if (!c) return fail(GP_ERR_INPUT, "null context");
    if (n == 0) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    k5_sim_1f1b<<<(unsigned)((n + 127) / 128), 128, 0, c->stream>>>(d_timings, (long long)n,
                                                                   (int)iterations, d_makespan,
                                                                   d_status);
    CUDA_TRY(cudaGetLastError());
    return GP_OK;
}

int gp_sim_1f1b(gp_ctx* c, const gp_timing* timings, uint64_t n, uint32_t iterations,
                double* makespan, uint8_t* status) {
    if (!c) return fail(GP_ERR_INPUT, "null context");
    if (n == 0) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    CUDA_TRY(c->s_tim.ensure(n));
    CUDA_TRY(c->s_ms.ensure(n));
    CUDA_TRY(c->s_st.ensure(n));
    CUDA_TRY(cudaMemcpyAsync(c->s_tim.p, timings, n * sizeof(gp_timing), cudaMemcpyHostToDevice, s));
    int st = gp_sim_1f1b_device(c, c->s_tim.p, n, iterations, c->s_ms.p, c->s_st.p);
    if (st != GP_OK) return st;
    CUDA_TRY(cudaMemcpyAsync(makespan, c->s_ms.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(status, c->s_st.p, n, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return GP_OK;
}

int gp_replan_snapshots(gp_ctx* c, const double* bandwidth, uint32_t n_snap, gp_best* out,
                        int32_t* status) {
    if (!c || !c->loaded || !bandwidth || !out || !status) return fail(GP_ERR_INPUT, "bad arguments");
    if (n_snap == 0) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    const int k = c->F, n = c->n;
    uint64_t total;
    gp_space_size(c, &total);
    const unsigned long long NP = h_fact(k), NC = h_binom(n - 1, k - 1);
    const unsigned long long items = (unsigned long long)c->nm * NP;
    const size_t DD = (size_t)c->D * c->D;
    const size_t ntri = (size_t)n * (n + 1) / 2, nxp = (size_t)((n + 1) & ~1);
    const size_t s_tpk = (size_t)c->nm * c->F * ntri, s_tcol = (size_t)c->nm * c->F * (n + 1);
    const size_t s_xt = (size_t)c->nm * c->F * c->F * nxp;
    int fl_sync = known_flags(c);
    if (fl_sync < 0) {  // base tables must be error-free for the per-snapshot fast path
        CUDA_TRY(cudaEventSynchronize(c->flags_ev));
        fl_sync = known_flags(c);
    }
    const bool fast = k >= 3 && c->sweep_ok && c->nb <= 4 && total > 0 && c->force_mode != 3 &&
                      c->force_mode != 4;
    // batch size: keep the per-snapshot tables around 256 MB
    size_t per = (s_tpk + s_tcol) * 16 + s_xt * 8 + DD * 8;
    uint32_t SB = (uint32_t)((256ull << 20) / (per ? per : 1));
    if (SB < 1) SB = 1;
    if (SB > 4096) SB = 4096;
    if (SB > n_snap) SB = n_snap;
    std::vector<uint32_t> h_fl(SB);
    std::vector<Key> h_res(SB);
    std::vector<uint32_t> slow;
    for (uint32_t b0 = 0; b0 < n_snap; b0 += SB) {
        const uint32_t nb = (n_snap - b0) < SB ? (n_snap - b0) : SB;
        if (!(fast && fl_sync == 0)) {
            for (uint32_t i = 0; i < nb; ++i) slow.push_back(b0 + i);
            continue;
        }
        CUDA_TRY(c->z_bw.ensure((size_t)SB * DD));
        CUDA_TRY(c->z_mbw.ensure((size_t)SB * c->F));
        CUDA_TRY(c->z_flags.ensure(SB));
        CUDA_TRY(c->z_tpk.ensure((size_t)SB * s_tpk));
        CUDA_TRY(c->z_tcol.ensure((size_t)SB * s_tcol));
        CUDA_TRY(c->z_xt.ensure((size_t)SB * s_xt));
        CUDA_TRY(c->z_res.ensure(SB));
        CUDA_TRY(c->z_cnt.ensure(SB));
        CUDA_TRY(cudaMemcpyAsync(c->z_bw.p, bandwidth + (size_t)b0 * DD, (size_t)nb * DD * 8,
                                 cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemsetAsync(c->z_flags.p, 0, nb * sizeof(uint32_t), s));
        CUDA_TRY(cudaMemsetAsync(c->z_cnt.p, 0, nb * sizeof(unsigned int), s));
        SnapGeom Z;
        Z.nsnap = (int)nb;
        Z.bw = c->z_bw.p; Z.mbw = c->z_mbw.p; Z.flags = c->z_flags.p;
        Z.tpk = c->z_tpk.p; Z.tcol = c->z_tcol.p; Z.xt = c->z_xt.p;
        Z.s_tpk = s_tpk; Z.s_tcol = s_tcol; Z.s_xt = s_xt;
        DevInst I = c->view();
        k6_minbw<<<(unsigned)((nb * c->F + 127) / 128), 128, 0, s>>>(I, Z);
        const long long work = (long long)(s_tpk + (size_t)c->nm * c->F * c->F * n);
        dim3 pg((unsigned)((work + 255) / 256), nb);
        k6_patch<<<pg, 256, 0, s>>>(I, Z);
        CUDA_TRY(cudaGetLastError());
        // sweep over (snapshot, item)
        size_t smem0 = 16 + (((size_t)(n + 1) * (k + 1) * 8 + 15) & ~(size_t)15) + (size_t)c->ngroups * 16;
        size_t smem1 = smem0 + ntri * 16 + (n + 1) * 16 + 3 * nxp * 8 + (size_t)n * 16;
        size_t smem2 = smem1 + ntri * 16;
        int mode = smem2 <= (size_t)c->smem_max ? 2 : (smem1 <= (size_t)c->smem_max ? 1 : 0);
        if (c->force_mode >= 0 && c->force_mode < mode) mode = c->force_mode;
        size_t smem = mode == 2 ? smem2 : (mode == 1 ? smem1 : smem0);
        typedef void (*SwFn)(DevInst, SweepGeom, ArgminScratch, const unsigned long long*,
                             const uint32_t*);
        static const SwFn table[3][4] = {
            {k3_sweep<0, 1>, k3_sweep<0, 2>, k3_sweep<0, 3>, k3_sweep<0, 4>},
            {k3_sweep<1, 1>, k3_sweep<1, 2>, k3_sweep<1, 3>, k3_sweep<1, 4>},
            {k3_sweep<2, 1>, k3_sweep<2, 2>, k3_sweep<2, 3>, k3_sweep<2, 4>}};
        SwFn kern = table[mode][c->nb - 1];
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, K3S_THREADS, smem));
        unsigned long long resident = (unsigned long long)(per_sm > 0 ? per_sm : 1) * c->n_sms;
        unsigned long long cpi = (items * nb) >= resident ? 1 : resident / (items * nb);
        unsigned long long tasks = (c->sweep_W + 31) / 32;
        unsigned long long cap = (tasks + (K3S_THREADS / 32) - 1) / (K3S_THREADS / 32);
        if (cpi > cap) cpi = cap;
        if (cpi < 1) cpi = 1;
        unsigned long long grid = (unsigned long long)nb * items * cpi;
        if (grid > 0x7fffffffull) return fail(GP_ERR_INPUT, "snapshot batch too large");
        SweepGeom G;
        G.k = k; G.nbm = c->nb * c->nm; G.NC = NC; G.NP = NP; G.item0 = 0; G.cpi = cpi;
        G.W = c->sweep_W; G.ngroups = c->ngroups; G.groups = c->groups.p;
        G.prefixes = c->prefixes.p;
        G.bnk = c->bnk.p;
        G.gsteps = 1;
        while (G.gsteps * 2 <= c->ngroups) G.gsteps *= 2;
        G.items = (unsigned int)items;
        G.tpk = c->z_tpk.p; G.tcol = c->z_tcol.p; G.xt = c->z_xt.p;
        G.s_tpk = s_tpk; G.s_tcol = s_tcol; G.s_xt = s_xt;
        CUDA_TRY(c->item_ctr.ensure((size_t)nb * items));
        CUDA_TRY(cudaMemsetAsync(c->item_ctr.p, 0, (size_t)nb * items * sizeof(unsigned int), s));
        G.item_ctr = c->item_ctr.p;
        CUDA_TRY(c->blk.ensure(grid > 4096 ? grid : 4096));
        ArgminScratch S;
        S.blk = c->blk.p;
        S.counter = c->z_cnt.p;
        S.result = c->z_res.p;
        S.err = nullptr;
        S.err_idx = c->err_idx.p;
        kern<<<(unsigned)grid, K3S_THREADS, smem, s>>>(I, G, S, c->binom.p, c->z_flags.p);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(h_res.data(), c->z_res.p, nb * sizeof(Key), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(h_fl.data(), c->z_flags.p, nb * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        for (uint32_t i = 0; i < nb; ++i) {
            gp_best& o = out[b0 + i];
            memset(&o, 0, sizeof(o));
            o.k = (uint32_t)k;
            o.evaluated = total;
            if (h_fl[i]) { slow.push_back(b0 + i); continue; }
            const Key& r = h_res[i];
            if (r.tie == ~0ull) { status[b0 + i] = GP_ERR_NO_FEASIBLE; continue; }
            const int nbm = c->nb * c->nm;
            unsigned long long bmv = r.tie % (unsigned long long)nbm, pc = r.tie / (unsigned long long)nbm;
            o.cost = r.cost;
            o.index = (bmv * NP + pc / NC) * NC + pc % NC;
            o.batch_index = (uint32_t)(bmv / c->nm);
            o.micro_index = (uint32_t)(bmv % c->nm);
            h_unrank_perm(k, pc / NC, o.order);
            h_unrank_counts(n, k, pc % NC, o.counts);
            status[b0 + i] = GP_OK;
        }
    }
    if (!slow.empty()) {
        // exact status-tracking path, one snapshot at a time on the context
        std::vector<double> base((size_t)DD);
        CUDA_TRY(cudaMemcpyAsync(base.data(), c->bw.p, DD * 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        for (uint32_t sn : slow) {
            int st = gp_set_bandwidth(c, bandwidth + (size_t)sn * DD);
            if (st == GP_OK) st = gp_argmin_range(c, 0, total, &out[sn]);
            status[sn] = st;
        }
        int st = gp_set_bandwidth(c, base.data());
        if (st != GP_OK) return st;
    }
    return GP_OK;
}

int gp_sim_candidates(gp_ctx* c, uint32_t k, uint64_t n, const uint8_t* order,
                      const uint8_t* counts, const uint8_t* bm, uint32_t iterations,
                      double opt_seconds, double* makespan, uint8_t* status) {
    if (!c || !c->loaded) return fail(GP_ERR_INPUT, "context not loaded");
    if (k < 1 || k > GP_MAX_STAGES) return fail(GP_ERR_INPUT, "k=%u outside [1,%d]", k, GP_MAX_STAGES);
    if (n == 0) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    CUDA_TRY(c->b_order.ensure(n * k));
    CUDA_TRY(c->b_counts.ensure(n * k));
    CUDA_TRY(c->b_bm.ensure(n));
    CUDA_TRY(c->b_cost.ensure(n));
    CUDA_TRY(c->b_status.ensure(n));
    CUDA_TRY(cudaMemcpyAsync(c->b_order.p, order, n * k, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->b_counts.p, counts, n * k, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->b_bm.p, bm, n, cudaMemcpyHostToDevice, s));
    DevInst I = c->view();
    k5_sim_candidates<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(I, (int)k, (long long)n, c->b_order.p,
                                                                 c->b_counts.p, c->b_bm.p,
                                                                 (int)iterations, opt_seconds,
                                                                 c->b_cost.p, c->b_status.p);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(makespan, c->b_cost.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(status, c->b_status.p, n, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return GP_OK;
}

int gp_ctx_set_k3_mode(gp_ctx* c, int mode) {
    if (!c || mode < -1 || mode > 4) return fail(GP_ERR_INPUT, "bad mode");
    c->force_mode = mode;
    return GP_OK;
}

int gp_diag_fp64_peak(int device, double* dadd_per_second) {
    if (!dadd_per_second) return fail(GP_ERR_INPUT, "null output");
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 1 << 14;
    double* sink = nullptr;
    CUDA_TRY(cudaMalloc(&sink, blocks * sizeof(double)));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_fp64_peak<<<blocks, threads>>>(sink, iters, 1e-9);  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_fp64_peak<<<blocks, threads>>>(sink, iters, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (err != cudaSuccess) return fail(GP_ERR_CUDA, "fp64 peak: %s", cudaGetErrorString(err));
    double ops = (double)blocks * threads * iters * 8.0;
    *dadd_per_second = ops / (best * 1e-3);
    return GP_OK;
}

}  // extern "C"
