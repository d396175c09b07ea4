// k2_eval.cuh - K2: per-candidate evaluation from the tables (explicit batches, status-tracking path).
#pragma once
#include "k1_tables.cuh"

// ----------------------------------------------------------------------------
// generic evaluation of one candidate from the tables (status-tracking path)
// ----------------------------------------------------------------------------
struct EvalOut {
    double cost;
    int status;
};

// p[0..k] are cut positions (p[0] = 0); order[s] group of stage s.
static __device__ EvalOut eval_tables(const DevInst& I, int k, const uint8_t* order, const int* p,
                               int mi, long long M) {
    int n = I.n;
    size_t N2 = (size_t)(n + 1) * (n + 1);
    EvalOut out{0.0, GP_OK};
    bool feas = true;
    GP_DCHECK(k >= 1 && k <= I.F && p[0] == 0 && mi >= 0 && mi < I.nm);
    for (int s = 0; s < k; ++s) GP_DCHECK(order[s] < I.F && p[s] < p[s + 1] && p[s + 1] <= n);
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

static __global__ void k2_eval_batch(DevInst I, int k, long long ncand, const uint8_t* __restrict__ order,
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
    if (*I.flags == 0u && p[k] == I.n && k >= 2 && k <= 6) {
        const double Md = __ldg(&I.mtab[b]);  // (double)(batch / micro), tabulated by K1
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
    EvalOut r = eval_tables(I, k, o, p, mi, I.batch[b / I.nm] / I.micro[mi]);
    cost[i] = r.status == GP_OK ? r.cost : NAN;
    status[i] = (uint8_t)r.status;
}


// ---- K2 for large batches: stage codes in shared memory ---------------------
// Persistent grid-stride variant for batches of many candidates on tables
// without error entries.  Every CTA copies the stage-code table scode[f][a][b]
// (F * (n+1)^2 bytes, 26 KB at C4) into shared memory once; a candidate with a
// memory-infeasible stage (SC_INFEASIBLE, whose stage-table entry is +inf by
// construction, so its cost is exactly +inf: no inf - inf can arise) is
// decided from shared memory, and only the others gather their k stage entries
// and k-1 boundary values from L2 (84 % of random C4 candidates are
// infeasible).  k = 4 reads order and counts as one 32-bit word each.
#ifndef K2_U
#define K2_U 2
#endif
template <int K>
__global__ void __launch_bounds__(256) k2_eval_batch_sc(DevInst I, long long ncand,
                                                        const uint8_t* __restrict__ order,
                                                        const uint8_t* __restrict__ counts,
                                                        const uint8_t* __restrict__ bm,
                                                        double* __restrict__ cost,
                                                        uint8_t* __restrict__ status) {
    extern __shared__ __align__(16) uint8_t sc_s[];
    const int n = I.n;
    const int N2 = (n + 1) * (n + 1);
    const int nbytes = I.F * N2;
    {
        int done = 0;
        if ((reinterpret_cast<uintptr_t>(I.scode) & 15u) == 0) {
            const uint4* src = reinterpret_cast<const uint4*>(I.scode);
            uint4* dst = reinterpret_cast<uint4*>(sc_s);
            for (int i = threadIdx.x; i < nbytes / 16; i += blockDim.x) dst[i] = __ldg(&src[i]);
            done = nbytes & ~15;
        }
        for (int i = done + threadIdx.x; i < nbytes; i += blockDim.x) sc_s[i] = __ldg(&I.scode[i]);
    }
    __syncthreads();
    const bool fast_tables = *I.flags == 0u;
    const long long stride = (long long)gridDim.x * blockDim.x;
    // K2_U candidates per thread and iteration: their input words are loaded
    // before any of them is evaluated (memory-level parallelism)
    for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < ncand;
         i0 += stride * K2_U) {
        uint32_t ow[K2_U], cw[K2_U];
        int bv[K2_U];
#pragma unroll
        for (int u = 0; u < K2_U; ++u) {
            const long long i = i0 + u * stride;
            ow[u] = cw[u] = 0u;
            bv[u] = 0;
            if (i < ncand) {
                if (K == 4) {
                    ow[u] = __ldg(reinterpret_cast<const uint32_t*>(order) + i);
                    cw[u] = __ldg(reinterpret_cast<const uint32_t*>(counts) + i);
                }
                bv[u] = __ldg(&bm[i]);
            }
        }
#pragma unroll
        for (int u = 0; u < K2_U; ++u) {
            const long long i = i0 + u * stride;
            if (i >= ncand) break;
            uint8_t o[K];
            int p[K + 1];
            p[0] = 0;
            int st = GP_OK;
            unsigned seen = 0;
#pragma unroll
            for (int s = 0; s < K; ++s) {
                int c;
                if (K == 4) {
                    o[s] = (uint8_t)(ow[u] >> (8 * s));
                    c = (int)((cw[u] >> (8 * s)) & 0xffu);
                } else {
                    o[s] = __ldg(&order[i * K + s]);
                    c = __ldg(&counts[i * K + s]);
                }
                if (o[s] >= I.F || (seen >> o[s]) & 1u || c == 0) st = GP_ERR_INPUT;
                seen |= 1u << (o[s] & 31);
                p[s + 1] = p[s] + c;
            }
            const int b = bv[u];
            if (b >= I.nb * I.nm || p[K] > n) st = GP_ERR_INPUT;
            if (st != GP_OK) { cost[i] = NAN; status[i] = (uint8_t)st; continue; }
            const int mi = b % I.nm;
            if (fast_tables && p[K] == n) {
                bool inf = false;
#pragma unroll
                for (int s = 0; s < K; ++s)
                    inf |= sc_s[o[s] * N2 + tri_idx(n, p[s], p[s + 1])] == SC_INFEASIBLE;
                double c = INFINITY;
                if (!inf) c = eval_fast<K>(I, o, p, mi, __ldg(&I.mtab[b]));
                cost[i] = c;
                status[i] = GP_OK;
                continue;
            }
            EvalOut r = eval_tables(I, K, o, p, mi, I.batch[b / I.nm] / I.micro[mi]);
            cost[i] = r.status == GP_OK ? r.cost : NAN;
            status[i] = (uint8_t)r.status;
        }
    }
}

// ---- K2, k = 4, large batches: warp-compacted evaluation -------------------
// As k2_eval_batch_sc, but the candidates that need the stage-table gathers
// (feasible ones, ~16 % of random C4 candidates) are queued per warp in
// shared memory and evaluated 32 at a time, so eval_fast runs with every lane
// busy instead of once per warp under a mostly-idle mask.
#define K2Q_THREADS 256
#ifndef K2Q_MINB
#define K2Q_MINB 1
#endif
static __global__ void __launch_bounds__(K2Q_THREADS, K2Q_MINB) k2_eval_batch_q4(DevInst I, long long ncand,
                                                                const uint8_t* __restrict__ order,
                                                                const uint8_t* __restrict__ counts,
                                                                const uint8_t* __restrict__ bm,
                                                                double* __restrict__ cost,
                                                                uint8_t* __restrict__ status) {
    extern __shared__ __align__(16) uint8_t q4_s[];
    uint4* queue = reinterpret_cast<uint4*>(q4_s);  // [warps][64] {index, order, counts, bm}
    uint8_t* sc_s = q4_s + (K2Q_THREADS / 32) * 64 * sizeof(uint4);
    const int n = I.n;
    const int N2 = (n + 1) * (n + 1);
    const int nbytes = I.F * N2;
    {
        int done = 0;
        if ((reinterpret_cast<uintptr_t>(I.scode) & 15u) == 0) {
            const uint4* src = reinterpret_cast<const uint4*>(I.scode);
            uint4* dst = reinterpret_cast<uint4*>(sc_s);
            for (int i = threadIdx.x; i < nbytes / 16; i += blockDim.x) dst[i] = __ldg(&src[i]);
            done = nbytes & ~15;
        }
        for (int i = done + threadIdx.x; i < nbytes; i += blockDim.x) sc_s[i] = __ldg(&I.scode[i]);
    }
    __syncthreads();
    const bool fast_tables = *I.flags == 0u;
    const int lane = threadIdx.x & 31;
    uint4* wq = queue + (threadIdx.x >> 5) * 64;
    const unsigned lt = (1u << lane) - 1u;
    auto decode = [&](uint32_t ow, uint32_t cw, uint8_t* o, int* p) {
        p[0] = 0;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            o[s] = (uint8_t)(ow >> (8 * s));
            p[s + 1] = p[s] + (int)((cw >> (8 * s)) & 0xffu);
        }
    };
    auto eval_entry = [&](const uint4 e) {
        uint8_t o[4];
        int p[5];
        decode(e.y, e.z, o, p);
        const int b = (int)e.w;
        cost[e.x] = eval_fast<4>(I, o, p, b % I.nm, __ldg(&I.mtab[b]));
    };
    int q = 0;  // warp-uniform queue length
    const long long stride = (long long)gridDim.x * blockDim.x;
    // the next iteration's input words are loaded before this one is decided
    auto load_in = [&](long long i, uint32_t& ow, uint32_t& cw, int& b) {
        ow = cw = 0u;
        b = 0;
        if (i < ncand) {
            ow = __ldg(reinterpret_cast<const uint32_t*>(order) + i);
            cw = __ldg(reinterpret_cast<const uint32_t*>(counts) + i);
            b = __ldg(&bm[i]);
        }
    };
    long long base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    uint32_t ow_n, cw_n;
    int b_n;
    load_in(base + lane, ow_n, cw_n, b_n);
    for (; base < ncand; base += stride) {
        const long long i = base + lane;
        const bool valid = i < ncand;
        const uint32_t ow = ow_n, cw = cw_n;
        const int b = b_n;
        load_in(base + stride + lane, ow_n, cw_n, b_n);
        bool need = false;
        if (valid) {
            uint8_t o[4];
            int p[5];
            decode(ow, cw, o, p);
            int st = GP_OK;
            unsigned seen = 0;
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                if (o[s] >= I.F || (seen >> o[s]) & 1u || p[s + 1] == p[s]) st = GP_ERR_INPUT;
                seen |= 1u << (o[s] & 31);
            }
            if (b >= I.nb * I.nm || p[4] > n) st = GP_ERR_INPUT;
            if (st != GP_OK) {
                cost[i] = NAN;
                status[i] = (uint8_t)st;
            } else if (fast_tables && p[4] == n) {
                bool inf = false;
#pragma unroll
                for (int s = 0; s < 4; ++s)
                    inf |= sc_s[o[s] * N2 + tri_idx(n, p[s], p[s + 1])] == SC_INFEASIBLE;
                status[i] = GP_OK;
                if (inf) cost[i] = INFINITY;
                else need = true;
            } else {
                const int mi = b % I.nm;
                EvalOut r = eval_tables(I, 4, o, p, mi, I.batch[b / I.nm] / I.micro[mi]);
                cost[i] = r.status == GP_OK ? r.cost : NAN;
                status[i] = (uint8_t)r.status;
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, need);
        if (need) wq[q + __popc(m & lt)] = make_uint4((unsigned)i, ow, cw, (unsigned)b);
        q += __popc(m);
        __syncwarp();
        if (q >= 32) {
            const uint4 e = wq[q - 32 + lane];
            __syncwarp();
            q -= 32;
            eval_entry(e);
        }
    }
    __syncwarp();
    if (lane < q) eval_entry(wq[lane]);
}

// ---- K2, k = 4, large batches: TMA-fed chunks --------------------------------
// Every warp owns a private pipeline: chunks of K2T_WCHUNK candidates (warp
// chunk = global warp id + j * total warps), streamed by the warp's lane 0
// into the warp's own K2T_STAGES-deep shared-memory ring with bulk async
// copies (cp.async.bulk + mbarrier complete_tx), so input loads leave the
// warps' critical path and no CTA-wide barrier paces the warps.  A warp
// classifies 32 candidates at a time from shared memory with SIMD byte
// arithmetic on the packed words (range, distinctness and zero checks on all
// four bytes at once, the cut positions as the byte-wise prefix sums of
// counts * 0x01010101) and the stage codes (shared by the CTA, in shared
// memory): errors and memory-infeasible candidates (+inf) are written at
// once, the feasible ones queued and evaluated 32 at a time (eval_fast: k
// stage entries + k-1 boundary values from L2), as in k2_eval_batch_q4.
#ifndef K2T_WCHUNK
#define K2T_WCHUNK 256
#endif
#ifndef K2T_STAGES
#define K2T_STAGES 3
#endif
#define K2T_THREADS 256
#ifndef K2T_MINB
#define K2T_MINB 2
#endif
#ifndef K2T_ILP
#define K2T_ILP 4
#endif
#define K2T_WARPS (K2T_THREADS / 32)
#define K2T_SLOT (K2T_WCHUNK * 9)  // order u32 + counts u32 + bm u8 per candidate

__host__ __device__ inline size_t k2t_smem(size_t sc_bytes) {
    return 16 * K2T_WARPS * K2T_STAGES / 2 + 64 + sc_bytes +
           (size_t)K2T_WARPS * K2T_STAGES * K2T_SLOT + (size_t)K2T_WARPS * 64 * 16;
}

static __global__ void __launch_bounds__(K2T_THREADS, K2T_MINB) k2_eval_batch_t4(DevInst I, long long ncand,
                                                              const uint8_t* __restrict__ order,
                                                              const uint8_t* __restrict__ counts,
                                                              const uint8_t* __restrict__ bm,
                                                              double* __restrict__ cost,
                                                              uint8_t* __restrict__ status,
                                                              unsigned sc_bytes) {
    extern __shared__ __align__(16) uint8_t t4_s[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t bar_bytes = ((size_t)K2T_WARPS * K2T_STAGES * 8 + 63) & ~(size_t)63;
    uint64_t* bar = reinterpret_cast<uint64_t*>(t4_s) + warp * K2T_STAGES;  // this warp's
    uint8_t* sc_s = t4_s + bar_bytes;
    uint8_t* ring = sc_s + sc_bytes + (size_t)warp * K2T_STAGES * K2T_SLOT;
    uint4* wq = reinterpret_cast<uint4*>(sc_s + sc_bytes + (size_t)K2T_WARPS * K2T_STAGES * K2T_SLOT) +
                warp * 64;
    const int n = I.n;
    const int N2 = (n + 1) * (n + 1);
    const long long nchunks = (ncand + K2T_WCHUNK - 1) / K2T_WCHUNK;
    const long long wstride = (long long)gridDim.x * K2T_WARPS;
    const long long wfirst = (long long)blockIdx.x * K2T_WARPS + warp;
    auto issue = [&](long long c, int slot) {  // lane 0
        const long long left = ncand - c * K2T_WCHUNK;
        const int cnt = (left < K2T_WCHUNK ? (int)left : K2T_WCHUNK) & ~15;  // ragged tail: direct loads
        uint8_t* dst = ring + (size_t)slot * K2T_SLOT;
        mbar_expect_tx(&bar[slot], (uint32_t)cnt * 9u);
        if (cnt) {
            tma_bulk_g2s(dst, order + c * K2T_WCHUNK * 4, (uint32_t)cnt * 4, &bar[slot]);
            tma_bulk_g2s(dst + K2T_WCHUNK * 4, counts + c * K2T_WCHUNK * 4, (uint32_t)cnt * 4, &bar[slot]);
            tma_bulk_g2s(dst + K2T_WCHUNK * 8, bm + c * K2T_WCHUNK, (uint32_t)cnt, &bar[slot]);
        }
    };
    if (lane == 0) {
        for (int s = 0; s < K2T_STAGES; ++s) mbar_init(&bar[s], 1);
        for (int s = 0; s < K2T_STAGES; ++s) {
            const long long c = wfirst + (long long)s * wstride;
            if (c < nchunks) issue(c, s);
        }
    }
    {
        const unsigned nbytes = (unsigned)(I.F * N2);
        const uint4* src = reinterpret_cast<const uint4*>(I.scode);
        uint4* dst = reinterpret_cast<uint4*>(sc_s);
        for (unsigned i = threadIdx.x; i < nbytes / 16; i += blockDim.x) dst[i] = __ldg(&src[i]);
        for (unsigned i = (nbytes & ~15u) + threadIdx.x; i < nbytes; i += blockDim.x)
            sc_s[i] = __ldg(&I.scode[i]);
    }
    __syncthreads();
    const bool fast_tables = *I.flags == 0u;
    const unsigned lt = (1u << lane) - 1u;
    const int nbm = I.nb * I.nm;
    auto eval_entry = [&](const uint4 e) {
        uint8_t o[4];
        int p[5];
        const unsigned pw = e.z * 0x01010101u;  // byte-wise prefix sums of the counts
        p[0] = 0;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            o[s] = (uint8_t)(e.y >> (8 * s));
            p[s + 1] = (int)((pw >> (8 * s)) & 0xffu);
        }
        const int b = (int)e.w;
        cost[e.x] = eval_fast<4>(I, o, p, b % I.nm, __ldg(&I.mtab[b]));
    };
    int q = 0;  // warp-uniform queue length
    int j = 0;
    for (long long c = wfirst; c < nchunks; c += wstride, ++j) {
        const int slot = j % K2T_STAGES;
        mbar_wait(&bar[slot], (uint32_t)((j / K2T_STAGES) & 1));
        const uint32_t* so = reinterpret_cast<const uint32_t*>(ring + (size_t)slot * K2T_SLOT);
        const uint32_t* scn = so + K2T_WCHUNK;
        const uint8_t* sb = reinterpret_cast<const uint8_t*>(so + 2 * K2T_WCHUNK);
        const long long c0 = c * K2T_WCHUNK;
        const long long left = ncand - c0;
        const int cnt = left < K2T_WCHUNK ? (int)left : K2T_WCHUNK;
        const int cnt16 = cnt & ~15;
        double* cc = cost + c0;
        uint8_t* sc = status + c0;
        // one candidate: write its result or report it for the warp's batch
        auto classify = [&](int r, uint32_t ow, uint32_t cw, int b) -> bool {
            // input checks on the packed words: groups < F and distinct (a
            // 4-bit set of 4 members), counts > 0 (no zero byte), sum of
            // counts <= n, (b, m) index in range
            const unsigned o0 = ow & 0xffu, o1 = (ow >> 8) & 0xffu, o2 = (ow >> 16) & 0xffu,
                           o3 = ow >> 24;
            const unsigned msk = (1u << (o0 & 31u)) | (1u << (o1 & 31u)) | (1u << (o2 & 31u)) |
                                 (1u << (o3 & 31u));
            const bool ok = ((ow & 0xE0E0E0E0u) == 0u) && (__popc(msk) == 4) &&
                            ((msk >> I.F) == 0u) &&
                            (((cw - 0x01010101u) & ~cw & 0x80808080u) == 0u);
            const int total = (int)__vsadu4(cw, 0u);
            if (!ok || b >= nbm || total > n) {
                cc[r] = NAN;
                sc[r] = (uint8_t)GP_ERR_INPUT;
                return false;
            }
            if (fast_tables && total == n) {
                const unsigned pw = cw * 0x01010101u;  // p1..p4 (exact: sums <= n <= 255)
                const int p1 = (int)(pw & 0xffu), p2 = (int)((pw >> 8) & 0xffu),
                          p3 = (int)((pw >> 16) & 0xffu);
                const bool inf = (sc_s[(int)o0 * N2 + p1] == SC_INFEASIBLE) |
                                 (sc_s[(int)o1 * N2 + tri_idx(n, p1, p2)] == SC_INFEASIBLE) |
                                 (sc_s[(int)o2 * N2 + tri_idx(n, p2, p3)] == SC_INFEASIBLE) |
                                 (sc_s[(int)o3 * N2 + tri_idx(n, p3, n)] == SC_INFEASIBLE);
                sc[r] = GP_OK;
                if (inf) cc[r] = INFINITY;
                return !inf;
            }
            uint8_t o[4];
            int p[5];
            p[0] = 0;
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                o[s] = (uint8_t)(ow >> (8 * s));
                p[s + 1] = p[s] + (int)((cw >> (8 * s)) & 0xffu);
            }
            const int mi = b % I.nm;
            EvalOut e = eval_tables(I, 4, o, p, mi, I.batch[b / I.nm] / I.micro[mi]);
            cc[r] = e.status == GP_OK ? e.cost : NAN;
            sc[r] = (uint8_t)e.status;
            return false;
        };
        auto enqueue = [&](bool need, int r, uint32_t ow, uint32_t cw, int b) {
            const unsigned m = __ballot_sync(0xffffffffu, need);
            if (need) wq[q + __popc(m & lt)] = make_uint4((unsigned)(c0 + r), ow, cw, (unsigned)b);
            q += __popc(m);
            __syncwarp();
            if (q >= 32) {
                const uint4 e = wq[q - 32 + lane];
                __syncwarp();
                q -= 32;
                eval_entry(e);
            }
        };
        if (cnt == K2T_WCHUNK) {  // full chunk: every input word in shared memory
            // K2T_ILP candidates per lane classified together (independent
            // chains: shared-memory round trips overlap), then queued in order
            for (int r0 = lane; r0 < K2T_WCHUNK; r0 += 32 * K2T_ILP) {
                uint32_t ow[K2T_ILP], cw[K2T_ILP];
                int b[K2T_ILP];
                bool need[K2T_ILP];
#pragma unroll
                for (int u = 0; u < K2T_ILP; ++u) {
                    ow[u] = so[r0 + 32 * u];
                    cw[u] = scn[r0 + 32 * u];
                    b[u] = sb[r0 + 32 * u];
                }
#pragma unroll
                for (int u = 0; u < K2T_ILP; ++u) need[u] = classify(r0 + 32 * u, ow[u], cw[u], b[u]);
#pragma unroll
                for (int u = 0; u < K2T_ILP; ++u) enqueue(need[u], r0 + 32 * u, ow[u], cw[u], b[u]);
            }
        } else {
            for (int r = lane; r < ((cnt + 31) & ~31); r += 32) {
                bool need = false;
                uint32_t ow = 0, cw = 0;
                int b = 0;
                if (r < cnt) {
                    if (r < cnt16) { ow = so[r]; cw = scn[r]; b = sb[r]; }
                    else {
                        ow = __ldg(reinterpret_cast<const uint32_t*>(order) + c0 + r);
                        cw = __ldg(reinterpret_cast<const uint32_t*>(counts) + c0 + r);
                        b = __ldg(&bm[c0 + r]);
                    }
                    need = classify(r, ow, cw, b);
                }
                enqueue(need, r, ow, cw, b);
            }
        }
        __syncwarp();  // the warp is done with the slot
        if (lane == 0) {
            const long long cn = c + (long long)K2T_STAGES * wstride;
            if (cn < nchunks) issue(cn, slot);
        }
    }
    __syncwarp();
    if (lane < q) eval_entry(wq[lane]);
}

// ---- K2, k = 4, large batches: vector lanes -----------------------------------
// As k2_eval_batch_t4 (per-warp TMA rings of input chunks, feasible
// candidates queued and evaluated 32 at a time), but a lane classifies FOUR
// CONSECUTIVE candidates per round: their order / counts words arrive in one
// 16-byte shared-memory load each and their four bm bytes in one 32-bit
// load, the classification is branch-free, and the four costs and four
// status bytes leave in two 16-byte and one 4-byte store.  Memory-infeasible
// stages come from a bit table (one bit per (group, a, b), 3.3 KB at C4,
// built from the stage codes by each CTA) instead of the byte table, so more
// CTAs fit an SM.  Queued (feasible) candidates get a placeholder cost in the
// vector store and their cost from eval_fast later (same warp, after a
// __syncwarp); candidates the fast tables cannot decide (an error status may
// follow) go through eval_tables.
#ifndef K2V_WCHUNK
#define K2V_WCHUNK 256
#endif
#ifndef K2V_STAGES
#define K2V_STAGES 2
#endif
#define K2V_QCAP 160  // queue entries per warp: < 32 left + 128 of one round
#define K2V_THREADS 256
#ifndef K2V_NW
#define K2V_NW 16  // warps per CTA of the shared-memory-table variant
#endif
#ifndef K2V_MINB
#define K2V_MINB 2
#endif
#define K2V_WARPS (K2V_THREADS / 32)
#define K2V_SLOT (K2V_WCHUNK * 9)  // order u32 | counts u32 | bm u8 per candidate

// infeasible-stage bit rows: row r = (f, a) = 4 words, bit b <=> stage [a, b)
// of group f is memory-infeasible (n + 1 <= 128), at word 4r + w.  Then F
// last-stage columns of 4 words: bit a of column f <=> stage [a, n) of group f
// is infeasible (4F consecutive words: a conflict-free lookup for F <= 8).
__host__ __device__ inline size_t k2v_bits_bytes(int F, int n) { return (size_t)F * (n + 2) * 16; }
__device__ __forceinline__ unsigned k2v_row_word(unsigned r, unsigned w) { return (r << 2) + w; }
// word e of the bit image (rows, then columns) from the stage codes
__device__ inline uint32_t k2v_bits_word(const DevInst& I, int e) {
    const int n = I.n, np = n + 1, N2 = np * np;
    uint32_t bits = 0;
    if (e < I.F * np * 4) {
        const int r = e >> 2, w = e & 3;  // r = f * np + a
        const uint8_t* src = I.scode + (size_t)(r / np) * N2 + (size_t)(r % np) * np;
        for (int j = 0; j < 32; ++j) {
            const int b = 32 * w + j;
            if (b <= n) bits |= (uint32_t)(__ldg(&src[b]) == SC_INFEASIBLE) << j;
        }
    } else {
        const int f = (e - I.F * np * 4) >> 2, w = e & 3;
        const uint8_t* src = I.scode + (size_t)f * N2 + n;
        for (int j = 0; j < 32; ++j) {
            const int a = 32 * w + j;
            if (a <= n) bits |= (uint32_t)(__ldg(&src[(size_t)a * np]) == SC_INFEASIBLE) << j;
        }
    }
    return bits;
}
// SMT: the first-stage rows [0, b), last-stage columns [a, n) and boundary
// rows of every (micro-batch, group) in shared memory, so a feasible
// candidate gathers only its two middle stage entries from L2
__host__ __device__ inline size_t k2v_tab_bytes(int F, int n, int nm, int nxp) {
    return (size_t)nm * F * (n + 1) * 16 * 2 + (((size_t)nm * F * F * nxp * 8 + 15) & ~(size_t)15);
}
__host__ __device__ inline size_t k2v_bar_bytes(int nwarps) { return ((size_t)nwarps * K2V_STAGES * 8 + 8 + 63) & ~(size_t)63; }
__host__ __device__ inline size_t k2v_smem(int F, int n, int nm, int nxp, int nwarps, bool smt) {
    return k2v_bar_bytes(nwarps) + k2v_bits_bytes(F, n) +
           (smt ? k2v_tab_bytes(F, n, nm, nxp) : 0) + (size_t)nwarps * K2V_STAGES * K2V_SLOT +
           (size_t)nwarps * K2V_QCAP * 16;
}

template <int NW, bool SMT>
static __global__ void __launch_bounds__(NW * 32, (NW >= 16 ? 1 : K2V_MINB)) k2_eval_batch_v4(DevInst I, long long ncand,
                                                              const uint8_t* __restrict__ order,
                                                              const uint8_t* __restrict__ counts,
                                                              const uint8_t* __restrict__ bm,
                                                              double* __restrict__ cost,
                                                              uint8_t* __restrict__ status,
                                                              const uint8_t* __restrict__ img) {
    extern __shared__ __align__(16) uint8_t v4_s[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = I.n, np = n + 1, F = I.F;
    const int nm = I.nm, nxp = I.nxp;
    const size_t bar_bytes = k2v_bar_bytes(NW);
    uint64_t* img_bar = reinterpret_cast<uint64_t*>(v4_s) + NW * K2V_STAGES;
    const size_t bits_bytes = k2v_bits_bytes(F, n) + (SMT ? k2v_tab_bytes(F, n, nm, nxp) : 0);
    uint64_t* bar = reinterpret_cast<uint64_t*>(v4_s) + warp * K2V_STAGES;
    uint32_t* ibits = reinterpret_cast<uint32_t*>(v4_s + bar_bytes);
    double2* t0s = reinterpret_cast<double2*>(v4_s + bar_bytes + k2v_bits_bytes(F, n));  // [nm][F][np]
    double2* t3s = t0s + (size_t)nm * F * np;                                              // [nm][F][np]
    double* xs = reinterpret_cast<double*>(t3s + (size_t)nm * F * np);                   // [nm][F][F][nxp]
    uint8_t* ring = v4_s + bar_bytes + bits_bytes + (size_t)warp * K2V_STAGES * K2V_SLOT;
    uint4* wq = reinterpret_cast<uint4*>(v4_s + bar_bytes + bits_bytes +
                                         (size_t)NW * K2V_STAGES * K2V_SLOT) + warp * K2V_QCAP;
    const int N2 = np * np;
    const long long nchunks = (ncand + K2V_WCHUNK - 1) / K2V_WCHUNK;
    const long long wstride = (long long)gridDim.x * NW;
    const long long wfirst = (long long)blockIdx.x * NW + warp;
    auto issue = [&](long long c, int slot) {  // lane 0
        const long long left = ncand - c * K2V_WCHUNK;
        const int cnt = (left < K2V_WCHUNK ? (int)left : K2V_WCHUNK) & ~15;  // ragged tail: direct loads
        uint8_t* dst = ring + (size_t)slot * K2V_SLOT;
        mbar_expect_tx(&bar[slot], (uint32_t)cnt * 9u);
        if (cnt) {
            tma_bulk_g2s(dst, order + c * K2V_WCHUNK * 4, (uint32_t)cnt * 4, &bar[slot]);
            tma_bulk_g2s(dst + K2V_WCHUNK * 4, counts + c * K2V_WCHUNK * 4, (uint32_t)cnt * 4, &bar[slot]);
            tma_bulk_g2s(dst + K2V_WCHUNK * 8, bm + c * K2V_WCHUNK, (uint32_t)cnt, &bar[slot]);
        }
    };
    if (lane == 0) {
        for (int s = 0; s < K2V_STAGES; ++s) mbar_init(&bar[s], 1);
        for (int s = 0; s < K2V_STAGES; ++s) {
            const long long c = wfirst + (long long)s * wstride;
            if (c < nchunks) issue(c, s);
        }
    }
    // bit rows (and SMT tables): one bulk copy of the image k2_image_build
    // made from this table generation, else from the stage codes
    const uint32_t img_bytes = (uint32_t)bits_bytes;
    if (img && threadIdx.x == 0) {
        mbar_init(img_bar, 1);
        mbar_expect_tx(img_bar, img_bytes);
        tma_bulk_g2s(ibits, img, img_bytes, img_bar);
    }
    if (!img)
    for (int rw = threadIdx.x; rw < F * (np + 1) * 4; rw += blockDim.x) ibits[rw] = k2v_bits_word(I, rw);
    if (SMT && !img) {
        for (int e = threadIdx.x; e < nm * F * np; e += blockDim.x) {
            const int a = e % np, mf = e / np;  // (mi, f) = mf
            const double2* T = I.stg + (size_t)mf * N2;
            t0s[e] = __ldg(&T[a]);                            // stage [0, a)
            t3s[e] = __ldg(&T[(size_t)a * np + n]);           // stage [a, n)
        }
        for (int e = threadIdx.x; e < nm * F * F * nxp; e += blockDim.x) xs[e] = __ldg(&I.xt[e]);
    }
    __syncthreads();  // (img_bar initialised)
    if (img) mbar_wait(img_bar, 0);
    const bool fast_tables = *I.flags == 0u;
    const unsigned lt = (1u << lane) - 1u;
    const int nbm = I.nb * I.nm;
    const unsigned fbias = (unsigned)(128 - (F < 128 ? F : 128)) * 0x01010101u;
    // bit b of row (f, a)
    auto inf_bit = [&](unsigned f, unsigned a, unsigned b) -> unsigned {
        const uint32_t w = ibits[k2v_row_word(f * (unsigned)np + a, b >> 5)];
        return __funnelshift_r(w, 0u, b) & 1u;
    };
    const uint32_t* icol = ibits + F * np * 4;
    auto inf_last = [&](unsigned f, unsigned a) -> unsigned {  // stage [a, n)
        return __funnelshift_r(icol[(f << 2) + (a >> 5)], 0u, a) & 1u;
    };
    // feasible candidates, 32 at a time, software-pipelined: a batch's table
    // entries (k stage entries, k-1 boundary values, M) are loaded when it
    // leaves the queue and its cost formed when the next batch leaves (or at
    // the end), so the L2 round trip overlaps the next round's classification
    bool pend = false;
    unsigned pidx = 0;
    double2 pe[4];
    double px[3], pM = 0.0;
    auto load_entry = [&](const uint4 e) {
        const unsigned pw = e.z * 0x01010101u;  // byte-wise prefix sums of the counts
        int p[5];
        p[0] = 0;
#pragma unroll
        for (int s = 0; s < 4; ++s) p[s + 1] = (int)((pw >> (8 * s)) & 0xffu);
        const int b = (int)e.w, mi = b % I.nm;
        const double2* T = I.stg + (size_t)mi * F * N2;
        const double* X = I.xt + (size_t)mi * F * F * I.nxp;
#if !defined(K2V_NOLOAD)
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const unsigned os = (e.y >> (8 * s)) & 0xffu;
            if (SMT && s == 0) pe[s] = t0s[((size_t)mi * F + os) * np + p[1]];
            else if (SMT && s == 3) pe[s] = t3s[((size_t)mi * F + os) * np + p[3]];
            else pe[s] = __ldg(&T[(size_t)os * N2 + tri_idx(n, p[s], p[s + 1])]);
            if (s < 3) {
                const unsigned on = (e.y >> (8 * (s + 1))) & 0xffu;
                px[s] = SMT ? xs[(((size_t)mi * F + os) * F + on) * nxp + (p[s + 1] - 1)]
                            : __ldg(&X[((size_t)os * F + on) * I.nxp + (p[s + 1] - 1)]);
            }
        }
#else
        (void)T; (void)X;
#endif
        pM = __ldg(&I.mtab[b]);
#if defined(K2V_NOLOAD)  // diagnostic build: no table gathers
        pe[0] = pe[1] = pe[2] = pe[3] = make_double2(pM, pM);
        px[0] = px[1] = px[2] = pM;
#endif
        pidx = e.x;
        pend = true;
    };
    auto finish_entry = [&]() {  // eval_fast's arithmetic on the loaded entries
        if (!pend) return;
        double fill = 0.0, res = 0.0, best = 0.0;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            if (s > 0) res = res + max0f(px[s - 1] - pe[s].x);
            const double total = ((fill + pM * pe[s].x) + res) + pe[s].y;
            best = (s == 0 || total > best) ? total : best;
            if (s + 1 < 4) fill = fill + (pe[s].x + px[s]);
        }
#if defined(K2V_NOSTORE)  // diagnostic build: evaluate, store only an impossible value
        if (best == -1.0) cost[pidx] = best;
#else
        cost[pidx] = best;
#endif
        pend = false;
    };
    auto eval_entry = [&](const uint4 e) {
        finish_entry();
        load_entry(e);
    };
    int q = 0;  // warp-uniform queue length
    auto push = [&](bool need, long long gi, uint32_t ow, uint32_t cw, int b) {
        const unsigned m = __ballot_sync(0xffffffffu, need);
        if (need) wq[q + __popc(m & lt)] = make_uint4((unsigned)gi, ow, cw, (unsigned)b);
        q += __popc(m);
    };
    auto drain = [&]() {  // full batches of 32 (one eval site: small code)
        __syncwarp();
        while (q >= 32) {
            const uint4 e = wq[q - 32 + lane];
            __syncwarp();
            q -= 32;
#if !defined(K2V_NOEVAL)  // diagnostic build: queue without evaluation
            eval_entry(e);
#else
            (void)e;
#endif
        }
    };
    // one candidate: 0 = error, 1 = +inf, 2 = queue (feasible), 3 =
    // status-tracking evaluation.  Packed-word checks: groups < F and
    // distinct (a 4-member bit set), no zero count, sum of counts <= n, (b, m)
    // index in range; the cut positions are the byte-wise prefix sums.
    auto classify = [&](uint32_t ow, uint32_t cw, unsigned b) -> int {
        const unsigned om = ow & 0x0f0f0f0fu;  // groups < 16: in-range table rows for any input
        const unsigned o0 = om & 0xffu, o1 = __byte_perm(om, 0u, 0x4441), o2 = __byte_perm(om, 0u, 0x4442),
                       o3 = om >> 24;
        const unsigned total = __vsadu4(cw, 0u);
        // groups: every byte < F (bytes < 128 first, then byte + 128 - F has
        // its top bit clear), pairwise distinct (no zero byte in the
        // differences to the byte-rotated words: the 6 pairs)
        const unsigned d8 = __vabsdiffu4(ow, __byte_perm(ow, 0u, 0x0321)),
                       d16 = __vabsdiffu4(ow, __byte_perm(ow, 0u, 0x1032));
        const unsigned z = ((d8 - 0x01010101u) & ~d8) | ((d16 - 0x01010101u) & ~d16) |
                           (cw - 0x01010101u) & ~cw | (ow & 0x80808080u) | (ow + fbias);
        const bool ok = ((z & 0x80808080u) == 0u) & (b < (unsigned)nbm) & (total <= (unsigned)n);
        const bool fast = ok & fast_tables & (total == (unsigned)n);
        // p1..p3 (exact when fast: sums <= n <= 127)
        const unsigned pw = (cw * 0x01010101u) & 0x7f7f7f7fu;
        const unsigned p1 = pw & 0xffu, p2 = __byte_perm(pw, 0u, 0x4441), p3 = __byte_perm(pw, 0u, 0x4442);
        // unconditional lookups (rows < 16 * 128, in the allocation), no branches
        const unsigned inf = (inf_bit(o0, 0u, p1) | inf_bit(o1, p1, p2) | inf_bit(o2, p2, p3) |
                              inf_last(o3, p3)) & (unsigned)fast;
#if defined(K2V_STREAM)  // diagnostic build: inputs in, outputs out, no classification
        return ((ow ^ cw ^ b) & 1u) ? 1 : 1;
#endif
        return !ok ? 0 : (!fast ? 3 : (inf ? 1 : 2));
    };
    auto slow_eval = [&](long long gi, uint32_t ow, uint32_t cw, int b) {
        uint8_t o[4];
        int p[5];
        p[0] = 0;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            o[s] = (uint8_t)(ow >> (8 * s));
            p[s + 1] = p[s] + (int)((cw >> (8 * s)) & 0xffu);
        }
        const int mi = b % I.nm;
        EvalOut e = eval_tables(I, 4, o, p, mi, I.batch[b / I.nm] / I.micro[mi]);
        cost[gi] = e.status == GP_OK ? e.cost : NAN;
        status[gi] = (uint8_t)e.status;
    };
    int j = 0;
    for (long long c = wfirst; c < nchunks; c += wstride, ++j) {
        const int slot = j % K2V_STAGES;
        mbar_wait(&bar[slot], (uint32_t)((j / K2V_STAGES) & 1));
        const uint8_t* sl = ring + (size_t)slot * K2V_SLOT;
        const long long c0 = c * K2V_WCHUNK;
        const long long left = ncand - c0;
        const int cnt = left < K2V_WCHUNK ? (int)left : K2V_WCHUNK;
        if (cnt == K2V_WCHUNK) {
#pragma unroll 1
            for (int r = 0; r < K2V_WCHUNK / 128; ++r) {
                const int i0 = 128 * r + 4 * lane;  // this lane's four candidates
                const uint4 ow4 = *reinterpret_cast<const uint4*>(sl + 4 * i0);
                const uint4 cw4 = *reinterpret_cast<const uint4*>(sl + K2V_WCHUNK * 4 + 4 * i0);
                const uint32_t bw4 = *reinterpret_cast<const uint32_t*>(sl + K2V_WCHUNK * 8 + i0);
                const uint32_t ow[4] = {ow4.x, ow4.y, ow4.z, ow4.w};
                const uint32_t cw[4] = {cw4.x, cw4.y, cw4.z, cw4.w};
                const unsigned bb[4] = {bw4 & 0xffu, __byte_perm(bw4, 0u, 0x4441), __byte_perm(bw4, 0u, 0x4442),
                                        bw4 >> 24};
                int cl[4];
#pragma unroll
                for (int s = 0; s < 4; ++s) cl[s] = classify(ow[s], cw[s], bb[s]);
                double cv[4];
                uint32_t sv = 0;
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    cv[s] = cl[s] == 0 ? NAN : (cl[s] == 1 ? INFINITY : 0.0);
                    sv |= (uint32_t)(cl[s] == 0 ? GP_ERR_INPUT : GP_OK) << (8 * s);
                }
                double2* cd = reinterpret_cast<double2*>(cost + c0 + i0);
                cd[0] = make_double2(cv[0], cv[1]);
                cd[1] = make_double2(cv[2], cv[3]);
                *reinterpret_cast<uint32_t*>(status + c0 + i0) = sv;
                if ((cl[0] == 3) | (cl[1] == 3) | (cl[2] == 3) | (cl[3] == 3)) {
#pragma unroll
                    for (int s = 0; s < 4; ++s)
                        if (cl[s] == 3) slow_eval(c0 + i0 + s, ow[s], cw[s], (int)bb[s]);
                }
#pragma unroll
                for (int s = 0; s < 4; ++s) push(cl[s] == 2, c0 + i0 + s, ow[s], cw[s], (int)bb[s]);
                drain();
            }
        } else {  // ragged last chunk: one candidate per lane per round
            const int cnt16 = cnt & ~15;
            for (int r = lane; r < ((cnt + 31) & ~31); r += 32) {
                int cl = -1;
                uint32_t ow = 0, cw = 0;
                int b = 0;
                if (r < cnt) {
                    if (r < cnt16) {
                        ow = reinterpret_cast<const uint32_t*>(sl)[r];
                        cw = reinterpret_cast<const uint32_t*>(sl + K2V_WCHUNK * 4)[r];
                        b = sl[K2V_WCHUNK * 8 + r];
                    } else {
                        ow = __ldg(reinterpret_cast<const uint32_t*>(order) + c0 + r);
                        cw = __ldg(reinterpret_cast<const uint32_t*>(counts) + c0 + r);
                        b = __ldg(&bm[c0 + r]);
                    }
                    cl = classify(ow, cw, (unsigned)b);
                    if (cl == 3) {
                        slow_eval(c0 + r, ow, cw, b);
                    } else {
                        cost[c0 + r] = cl == 0 ? NAN : (cl == 1 ? INFINITY : 0.0);
                        status[c0 + r] = (uint8_t)(cl == 0 ? GP_ERR_INPUT : GP_OK);
                    }
                }
                push(cl == 2, c0 + r, ow, cw, b);
                drain();
            }
        }
        __syncwarp();  // the warp is done with the slot
        if (lane == 0) {
            const long long cn = c + (long long)K2V_STAGES * wstride;
            if (cn < nchunks) issue(cn, slot);
        }
    }
    __syncwarp();
    finish_entry();
    if (lane < q) {
        load_entry(wq[lane]);
        finish_entry();
    }
}

// The shared-memory image of k2_eval_batch_v4<*, true>: infeasible-stage bit
// rows, first-stage rows, last-stage columns, boundary rows - built once per
// table generation, bulk-copied by every CTA.
static __global__ void k2_image_build(DevInst I, uint8_t* __restrict__ img) {
    const int n = I.n, np = n + 1, F = I.F, nm = I.nm, nxp = I.nxp, N2 = np * np;
    uint32_t* bits = reinterpret_cast<uint32_t*>(img);
    double2* t0 = reinterpret_cast<double2*>(img + k2v_bits_bytes(F, n));
    double2* t3 = t0 + (size_t)nm * F * np;
    double* xs = reinterpret_cast<double*>(t3 + (size_t)nm * F * np);
    const long long nb = (long long)F * (np + 1) * 4, nt = (long long)nm * F * np, nx = (long long)nm * F * F * nxp;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nb + nt + nx;
         e += (long long)gridDim.x * blockDim.x) {
        if (e < nb) {
            bits[e] = k2v_bits_word(I, (int)e);
        } else if (e < nb + nt) {
            const long long q = e - nb;
            const int a = (int)(q % np);
            const double2* T = I.stg + (size_t)(q / np) * N2;
            t0[q] = T[a];
            t3[q] = T[(size_t)a * np + n];
        } else {
            xs[e - nb - nt] = I.xt[e - nb - nt];
        }
    }
}

// Arg-min over an evaluated batch (gp_argmin_batch_device): the least
// (cost, key) over the candidates with status 0, key = keys[i] (e.g. the
// enumeration index of a sampled candidate) or i; {+inf, ~0} when none.
// Grid-stride scan, then the CTA / last-CTA reduction of common.cuh.
static __global__ void __launch_bounds__(256) k2_batch_argmin(unsigned long long n,
                                                               const double* __restrict__ cost,
                                                               const uint8_t* __restrict__ status,
                                                               const unsigned long long* __restrict__ keys,
                                                               ArgminScratch S) {
    Key mine{INFINITY, ~0ull};
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        if (__ldg(&status[i])) continue;
        const Key o{__ldg(&cost[i]), keys ? __ldg(&keys[i]) : i};
        if (key_less(o, mine)) mine = o;
    }
    block_argmin_finish(mine, S);
}
