// common.cuh - shared device-side pieces of the engine: error plumbing,
// the device view of a loaded instance (DevInst), arg-min keys and their
// warp / CTA / grid reduction, exact scalar helpers, enumeration decode,
// and the TMA bulk-copy + mbarrier primitives.
#pragma once
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

// ----------------------------------------------------------------------------
// checked build (make checked -> libgeopipe_b200_chk.so, -DGP_CHECKS): device
// index / invariant checks record the first failing source line in a device
// word instead of trapping (a trap would leave the context unusable);
// gp_diag_checks() reads and clears it.  The stand-in for compute-sanitizer,
// which this GPU pool does not allow.  Production builds compile them out.
// ----------------------------------------------------------------------------
#if defined(GP_CHECKS)
static __device__ unsigned int g_chk_line = 0u;
#define GP_DCHECK(cond) do { if (!(cond)) atomicCAS(&g_chk_line, 0u, (unsigned)__LINE__); } while (0)
#else
#define GP_DCHECK(cond) do {} while (0)
#endif

// stage-table codes (per group, layer range)
enum : uint8_t { SC_OK = 0, SC_INFEASIBLE = 1, SC_DEGENERATE = 4, SC_TOPOLOGY = 5 };
// context flags that force the generic (status-tracking) range kernel
enum : uint32_t { FLAG_STAGE_ERROR = 1, FLAG_OVERFLOW = 2, FLAG_GATEWAY_ERROR = 4 };
#define K3_THREADS 256
#define K3_TILE 256
#ifndef K3_SEG
#define K3_SEG 32
#endif
#ifndef K3_QPAIR
#define K3_QPAIR 1  // k3_sweep: two q steps per iteration where the warp's runs allow
#endif
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

// Per-group constants of the stage-table build, one 128-byte record per
// first-level group written by K1 phase 1 (k1_group_block) so that a phase-2
// thread reads its group in one round trip.  `fast` = the register path of
// k1_stage_t applies (<= 2 second-level groups); tp_thr = the TP memory
// threshold (see tp_threshold), valid when thr_ok.
struct __align__(16) K1Grp {
    double cap, mbw, minmem, tp_thr;  // fg capacity, min intra bw, min member memory
    double sgcap[4], sgmin[4];        // second-level capacities / min memories
    int nmem, s0, nsg;
    uint8_t has, tp_ok, thr_ok, sgne;  // sgne bit j: SG j has members
    int fast, pad[3];
};

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
    double* mtab;   // [nb*nm] (double)(batch / micro) per (b, m) index (K1)
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
    K1Grp* grp;                  // [F] packed per-group constants (phase 1 -> phase 2)
    uint8_t* sshare0;            // [F][(n+1)^2] first ASYMMETRIC_PP share (winner detail)
    uint8_t* gwbad;              // [F*F] gateway bandwidth not > 0 (winner detail)
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

// interval-sum table S[col] is stored b-major (transposed) so that K1's
// per-a sweeps write coalesced
__device__ __forceinline__ int s_idx(int n, int a, int b) { return b * (n + 1) + a; }

__device__ __forceinline__ double Ssum(const DevInst& I, int col, int a, int b) {
    size_t N2 = (size_t)(I.n + 1) * (I.n + 1);
    return I.S[col * N2 + s_idx(I.n, a, b)];
}


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


// ----------------------------------------------------------------------------
// Verify sink (parity tests): when `out` is set, the verify instantiations of
// the K3 / K6 kernels store every evaluated candidate's cost at its global
// position g = snapshot * stride + enumeration index, g in [lo, lo + n).
// Production launches carry out = nullptr and use the plain instantiations
// (same arithmetic source, no stores).  Error candidates (generic kernel)
// store a quiet NaN whose low bits hold the status code.
// ----------------------------------------------------------------------------
struct VerifySink {
    double* out = nullptr;
    unsigned long long lo = 0, n = 0, stride = 0;
};
__device__ __forceinline__ void vput(const VerifySink& V, unsigned long long snap,
                                     unsigned long long idx, double c) {
    const unsigned long long g = snap * V.stride + idx;
    if (g - V.lo < V.n) V.out[g - V.lo] = c;
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
    VerifySink vs;                     // parity tests only (out = nullptr otherwise)
};

static __device__ unsigned long long d_binom(int n, int r) {
    if (r < 0 || r > n) return 0ull;
    unsigned long long res = 1;
    for (int i = 1; i <= r; ++i) res = res * (unsigned long long)(n - r + i) / (unsigned long long)i;
    return res;
}

static __device__ void d_unrank_perm(int k, unsigned long long r, uint8_t* perm) {
    if (k <= 12 && r < 479001600ull) {
        // 32-bit arithmetic (12! < 2^32) and the pool as 4-bit fields of one
        // register (no local-memory array, no 64-bit division)
        unsigned long long pool = 0xfedcba9876543210ull;  // field i = i
        unsigned int f = 1, rr = (unsigned int)r;
        for (int i = 2; i < k; ++i) f *= (unsigned int)i;     // (k-1)!
        for (int i = 0; i < k; ++i) {
            const unsigned int q = rr / f;
            rr -= q * f;
            perm[i] = (uint8_t)((pool >> (4 * q)) & 15ull);
            // remove field q: keep fields below, shift the ones above down
            const unsigned long long lowmask = q ? ((1ull << (4 * q)) - 1ull) : 0ull;
            pool = (pool & lowmask) | ((pool >> 4) & ~lowmask);
            if (k - 1 - i > 0) f /= (unsigned int)(k - 1 - i);
        }
        return;
    }
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
static __device__ void d_unrank_cuts(int n, int k, unsigned long long r, int* p) {
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
    unsigned int* rearm = nullptr;  // [nrearm] work counters the group's last CTA zeroes
    unsigned int nrearm = 0;
};

// CTA-wide reduction of per-thread keys, then last-block grid reduction.
// Reduction over a group of `nblk` CTAs (the whole grid, or one snapshot's
// CTAs): CTA `bidx` of the group writes its key; the last one to finish
// reduces the group's keys into *S.result and re-arms the counter.
static __device__ void block_argmin_finish(Key mine, const ArgminScratch& S, unsigned int nblk,
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
    // every CTA of the group has finished its last atomicAdd on the work
    // counters before it reached the group counter: zero them for the next
    // launch (saves a memset node per launch)
    for (unsigned int i = threadIdx.x; i < S.nrearm; i += blockDim.x) S.rearm[i] = 0u;
}

__device__ __forceinline__ void block_argmin_finish(Key mine, const ArgminScratch& S) {
    block_argmin_finish(mine, S, gridDim.x, blockIdx.x);
}


// packed triangle: row a of a stage table holds b = a+1..n
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




// ---- per-CTA timeline (diagnostic builds, -DGP_TIMELINE) --------------------------
// Thread 0 of each CTA of the instrumented kernels appends {kernel id, CTA,
// SM, entry, after pdl_wait, exit} (globaltimer ns) to a device log that
// gp_diag_timeline() drains.  Compiled out of the shipped library.
struct TlRec { unsigned long long t0, tw, t1; unsigned int kid, blk, smid, pad; };
#if defined(GP_TIMELINE)
#define GP_TL_CAP 65536
__device__ TlRec g_tl[GP_TL_CAP];
__device__ unsigned int g_tl_n;
__device__ __forceinline__ unsigned long long tl_now() {
    unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}
#define TL_START() const unsigned long long _tl0 = tl_now(); unsigned long long _tlw = _tl0
#define TL_WAITED() _tlw = tl_now()
#define TL_STOP(kid) do { if (threadIdx.x == 0) { \
    unsigned int _i = atomicAdd(&g_tl_n, 1u); unsigned int _sm; \
    asm volatile("mov.u32 %0, %%smid;" : "=r"(_sm)); \
    if (_i < GP_TL_CAP) g_tl[_i] = TlRec{_tl0, _tlw, tl_now(), (unsigned)(kid), blockIdx.x, _sm, 0u}; \
    } } while (0)
#else
#define TL_START() do {} while (0)
#define TL_WAITED() do {} while (0)
#define TL_STOP(kid) do {} while (0)
#endif

// ---- programmatic dependent launch ----------------------------------------------
// Kernels of the gp_replan graph are launched with programmatic stream
// serialisation: a dependent grid is scheduled once every CTA of the
// preceding grid has called pdl_trigger(), and pdl_wait() blocks until the
// preceding grid has completed and its writes are visible.  Without the
// launch attribute both are no-ops, so the same kernels serve every path.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

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
// bulk copy multicast to the same shared-memory offset of every CTA in
// ctamask (thread-block cluster); each destination's mbarrier at `bar`'s
// offset receives the complete_tx
__device__ __forceinline__ void tma_bulk_g2s_mc(void* dst, const void* src, uint32_t bytes,
                                                uint64_t* bar, uint16_t ctamask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(ctamask) : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
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
