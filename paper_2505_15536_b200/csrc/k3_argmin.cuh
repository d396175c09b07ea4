// k3_argmin.cuh - K3: exhaustive arg-min kernels (sub-range tile queue, full-item sweep, generic).
#pragma once
#include "k2_eval.cuh"

// Sub-range fast path (all stage entries error-free, k >= 3).
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
template <int MODE, int NB, bool VER = false>
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
                        if constexpr (VER)
                            vput(G.vs, 0, (((unsigned long long)bi * I.nm + mi) * G.NP + perm_rank) * G.NC + rabs, c);
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
    ArgminScratch Sr = S;  // the launch's item counters, zeroed by the last CTA
    Sr.rearm = G.item_ctr;
    Sr.nrearm = (unsigned int)(gridDim.x / G.chunks_per_item);
    block_argmin_finish(mine, Sr);
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
// record sweep (k3_sweep_rec.cuh) run table entry: prefix cuts p1..p(k-3),
// a = p(k-2), the run's length n-1-a, the longest padded length in its 32-run
// task and the composition rank of (prefix, a, q = a+1); host-built per
// (n, k), runs ordered by length
struct __align__(16) K3Run {
    uint8_t p[4];
    uint8_t a, len;
    uint8_t tmax;  // longest padded run of its 32-run task
    uint8_t pad;
    unsigned long long rpre;
};

struct SweepGeom {
    int k, nbm;
    unsigned long long NC, NP;
    unsigned long long item0;       // first (mi * NP + perm) item
    unsigned long long cpi;         // CTAs per item
    unsigned int W;                 // runs per item
    int ngroups;                    // uint4 slots staged: the run groups + the task table
    int ng;                         // run groups
    const uint4* groups;            // [ng] groups, then u16 task -> group of its first run
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
    int csize;                      // thread-block cluster size (CTAs of one item), 1 = none
    int interleave;                 // CTA -> item map: 1 = item-minor (b % items), 0 = item-major
    unsigned long long* gbound = nullptr;  // k3_sweep_rec: per-snapshot shared bound (~bits, 0 = none)
    const K3Run* runs = nullptr;    // k3_sweep_rec: run table ([W] runs)
    const uint32_t* rowstart = nullptr;  // k3_sweep_rec: padded record row starts [n]
    int nrecp = 0;                  // k3_sweep_rec: padded row records
    int b0;                         // first batch index of the NB evaluated together
    VerifySink vs;                  // parity tests only (VER instantiations)
};

#if defined(K3_PROFILE)
__device__ __forceinline__ unsigned __nv_smid_k3() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
#endif
// KS > 0 fixes the stage count at compile time (cut arrays in registers,
// no local memory); KS = 0 is the generic kernel.
template <int MODE, int NB, int KS, bool VER = false>
__global__ void __launch_bounds__(K3S_THREADS, K3S_MINB) k3_sweep(DevInst I, SweepGeom G, ArgminScratch S,
                                                          const unsigned long long* __restrict__ binom,
                                                          const uint32_t* skip_if_flags) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
#if defined(K3_PROFILE)
    unsigned long long t0p; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0p));
#endif
    TL_START();
    pdl_trigger();
    pdl_wait();  // K1's tables (gp_replan graph); no-op on plain launches
    TL_WAITED();
    const int n = I.n, k = KS > 0 ? KS : G.k;
    const int ntri = n * (n + 1) / 2;
    const int KB = k + 1;
    const unsigned int per_snap = G.items * (unsigned int)G.cpi;
    const unsigned int snap = blockIdx.x / per_snap, local = blockIdx.x % per_snap;
    // Item-minor map: CTAs are dispatched in blockIdx order, one per SM first,
    // and the SM's warp scheduler favours its older CTA, so an item-major map
    // (an item's CTAs adjacent) gives whole items only first-wave or only
    // second-wave CTAs and they finish ~15 % apart.  Item-minor spreads each
    // item's CTAs over both waves; with clusters the map is cluster-minor (a
    // cluster's CTAs stay on one item: measured 32.8 vs 30.7 us unclustered).
    const unsigned long long islot =
        !G.interleave ? local / G.cpi
                      : (G.csize == 1 ? local % G.items : (local / G.csize) % G.items);
    const unsigned long long item = G.item0 + islot;
    const int mi = (int)(item / G.NP);
    const unsigned long long perm_rank = item % G.NP;
    uint8_t order[GP_MAX_STAGES];
    d_unrank_perm(k, perm_rank, order);
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
    // every table this CTA reads arrives by bulk async copy on one mbarrier;
    // with a cluster (the CTAs of one item), the cluster's rank 0 issues each
    // copy once, multicast into every member's shared memory
    const uint32_t bn_bytes = (uint32_t)(((size_t)(n + 1) * KB * 8 + 15) & ~(size_t)15);
    uint32_t bytes = bn_bytes + (uint32_t)G.ngroups * 16;
    if (MODE >= 1)
        bytes += (uint32_t)(ntri * 16 + (n + 1) * 16 + 3 * I.nxp * 8 + n * 16) +
                 (MODE == 2 ? (uint32_t)ntri * 16 : 0u);
    const bool mc = G.csize > 1;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_expect_tx(bar, bytes);
    }
    if (mc) { cluster_arrive(); cluster_wait(); }  // every member's mbarrier is armed
    if (threadIdx.x == 0 && (!mc || cluster_ctarank() == 0)) {
        const uint16_t mask = (uint16_t)((1u << G.csize) - 1u);
        auto copy = [&](void* dst, const void* src, uint32_t nb) {
            if (mc) tma_bulk_g2s_mc(dst, src, nb, bar, mask);
            else tma_bulk_g2s(dst, src, nb, bar);
        };
        copy(bn, G.bnk, bn_bytes);
        copy(grp, G.groups, (uint32_t)G.ngroups * 16);
        if (MODE >= 1) {
            copy(tri2, P2, (uint32_t)ntri * 16);
            copy(col3, C3, (uint32_t)(n + 1) * 16);
            copy(x12s, X12, (uint32_t)I.nxp * 8);
            copy(x23s, X23, (uint32_t)I.nxp * 8);
            copy(row0, P0, (uint32_t)n * 16);
            copy(x01s, X01, (uint32_t)I.nxp * 8);
            if (MODE == 2) copy(tri1, P1, (uint32_t)ntri * 16);
        }
    }
    const int lane = threadIdx.x & 31;
    double best_c = INFINITY;
    unsigned long long best_t = ~0ull;  // R * NB + bi
#if defined(K3_NOTASK)
    const bool skip = true;  // diagnostic: staging + reduction only
#else
    const bool skip = skip_if_flags && skip_if_flags[snap];  // generic kernel decides
#endif
    unsigned int* const ctr = &G.item_ctr[(size_t)snap * G.items + islot];
    unsigned int t_next = 0;
#if defined(K3_STATIC)
    // diagnostic: round-robin tasks over the item's warps, no queue
    const unsigned int wstride = (unsigned int)G.cpi * (blockDim.x >> 5);
    const unsigned int wfirst = (unsigned int)((G.interleave && G.csize == 1) ? local / G.items
                                                                               : local % G.cpi) *
                                    (blockDim.x >> 5) + (threadIdx.x >> 5);
    t_next = wfirst;
#else
    if (lane == 0 && !skip) t_next = atomicAdd(ctr, 1u);  // (its latency overlaps the staging)
#endif
    // micro-batch counts M = B / m (loaded after the copies are issued: on a
    // cold L2 their latency would otherwise delay the TMA issue)
    double Mv[NB];
#pragma unroll
    for (int bi = 0; bi < NB; ++bi) Mv[bi] = (double)(I.batch[G.b0 + bi] / I.micro[mi]);
    __syncthreads();
    mbar_wait(bar, 0);
    if (mc) cluster_arrive();  // this CTA's copies have landed (waited on before exit)
#if defined(K3_PROFILE)
    unsigned long long t1p; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1p));
#endif

    for (; !skip;) {
#if defined(K3_STATIC)
        const unsigned int t = t_next;
        if ((unsigned long long)t * 32 >= G.W) break;
        t_next += wstride;
#else
        const unsigned int t = __shfl_sync(0xffffffffu, t_next, 0);
        if ((unsigned long long)t * 32 >= G.W) break;
        if (lane == 0) t_next = atomicAdd(ctr, 1u);  // next task, latency hidden by this one
#endif
        const unsigned int u = t * 32 + lane;
        int len = 0, a = 1, q0 = 2;  // idle lanes keep in-range table addresses
        double fill2 = 0.0, res1 = 0.0, x1 = 0.0;
        double mx1[NB];
        unsigned long long rpre = 0;  // comp rank of (prefix, a, q = a + 1)
        if (u < G.W) {
            // run id -> group (from the task's first group, a few steps at
            // most), prefix row, segment; full-length groups are segment-major
            // so the lanes of a warp share (a, q) and read the same shared-
            // memory words (broadcast)
            int gi = ((const uint16_t*)(grp + G.ng))[t];
            while (gi + 1 < G.ng && grp[gi + 1].x <= u) ++gi;
            const uint4 g = grp[gi];
            const unsigned int local = u - g.x;
            a = (int)(g.y & 0xffffu);
            len = (int)(g.y >> 16);
            unsigned int row;
            if (g.w) { const unsigned seg = local / g.z; row = local - seg * g.z; q0 = a + 1 + (int)seg * K3_SEG; }
            else { row = local; q0 = n - len; }
            // prefix cuts p[1..k-3]: colex row `row` (subsets of [1, a-1] come first)
            int p[GP_MAX_STAGES + 1];
            p[0] = 0;
            if (k == 4) {
                p[1] = (int)row + 1;  // colex 1-subsets of [1, n-3]: row r is {r + 1}
            } else if (k > 3) {
                const uint8_t* pr = G.prefixes + (size_t)row * 16;
                for (int j = 1; j <= k - 3; ++j) p[j] = pr[j - 1];
            }
            p[k - 2] = a;
            GP_DCHECK(gi < G.ng && a >= k - 2 && a <= n - 2 && len >= 1 && len <= K3_SEG &&
                      q0 >= a + 1 && q0 + len - 1 <= n - 1);
            for (int j = 1; j <= k - 2; ++j) GP_DCHECK(p[j - 1] < p[j]);
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
        int lmax = len, lmin = len;
#if defined(K3_NOLOOP)
        len = 0; lmax = 0; lmin = 0;  // diagnostic: prologue + staging cost only
#endif
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            int o = __shfl_xor_sync(0xffffffffu, lmax, off);
            lmax = o > lmax ? o : lmax;
            o = __shfl_xor_sync(0xffffffffu, lmin, off);
            lmin = o < lmin ? o : lmin;
        }
        // walk q: per-run minimum with strict < (ranks increase with q, and
        // with the batch index inside one q), merged into the lane's best
        // under the full key (cost, rank, batch) when the run ends
        const double2* e2p = (MODE >= 1 ? tri2 : P2) + (rowoff(n, a) - a - 1) + q0;
        const double2* e3p = (MODE >= 1 ? col3 : C3) + q0;
        const double* x2p = (MODE >= 1 ? x23s : X23) + (q0 - 1);
        double run_c = INFINITY;
        int run_i = -1, run_b = 0;
        // candidate q = q0 + i of the run: (cost min over the batch sizes, its batch)
        auto eval_q = [&](int i, double& cmin, int& bmin) {
            GP_DCHECK(i >= 0 && i < len && rowoff(n, a) - a - 1 + q0 + i < ntri && q0 + i <= n);
            double2 e2, e3;
            double x2;
            if (MODE >= 1) { e2 = e2p[i]; e3 = e3p[i]; x2 = x2p[i]; }
            else { e2 = __ldg(&e2p[i]); e3 = __ldg(&e3p[i]); x2 = __ldg(&x2p[i]); }
            // stages k-2 = [a, q) and k-1 = [q, n) (src/costmodel.py:68-81)
            const double res2 = res1 + max0f(x1 - e2.x);
            const double fill3 = fill2 + (e2.x + x2);
            const double res3 = res2 + max0f(x2 - e3.x);
            cmin = INFINITY;
            bmin = 0;
#pragma unroll
            for (int bi = 0; bi < NB; ++bi) {
                double t2 = ((fill2 + Mv[bi] * e2.x) + res2) + e2.y;
                double t3 = ((fill3 + Mv[bi] * e3.x) + res3) + e3.y;
                double c = gtsel(t2, mx1[bi]);
                c = gtsel(t3, c);
                if constexpr (VER)
                    vput(G.vs, snap,
                         ((((unsigned long long)(G.b0 + bi) * I.nm + mi) * G.NP + perm_rank) * G.NC) +
                             rpre + (unsigned long long)(q0 + i - a - 1), c);
                if (bi == 0 || c < cmin) { cmin = c; bmin = bi; }
            }
        };
        // steps every lane of the warp has (runs are sorted by length, so
        // usually all of them): two independent q evaluations per iteration
        // (ILP 2 for the fixed-latency FP64 chains), merged in q order
        int i0 = 0;
#if K3_QPAIR
        for (; i0 + 1 < lmin; i0 += 2) {
            double c0, c1;
            int b0, b1;
            eval_q(i0, c0, b0);
            eval_q(i0 + 1, c1, b1);
            if (run_i < 0 || c0 < run_c) { run_c = c0; run_i = i0; run_b = b0; }
            if (c1 < run_c) { run_c = c1; run_i = i0 + 1; run_b = b1; }
        }
#endif
        for (int i = i0; i < lmax; ++i) {
            if (i < len) {
                double cmin; int bmin;
                eval_q(i, cmin, bmin);
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
        GP_DCHECK(rr < G.NC);
        mine.cost = best_c;
        mine.tie = ((perm_rank * G.NC) + rr) * (unsigned long long)G.nbm +
                   (unsigned long long)((G.b0 + bi) * I.nm + mi);
    }
    ArgminScratch Ss = S;
    Ss.blk = S.blk + (size_t)snap * per_snap;
    Ss.counter = S.counter + snap;
    Ss.result = S.result + snap;
    Ss.rearm = ctr - islot;  // this snapshot's item counters
    Ss.nrearm = G.items;
#if defined(K3_PROFILE)
    unsigned long long t2p; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2p));
#endif
    block_argmin_finish(mine, Ss, per_snap, local);
    if (mc) cluster_wait();  // no CTA leaves while a multicast into a peer may be in flight
    TL_STOP(30);
#if defined(K3_PROFILE)
    { unsigned long long t3; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t3));
      if (threadIdx.x == 0) printf("K3P %d %d %llu %llu %llu %llu\n", blockIdx.x, (int)__nv_smid_k3(), t0p, t1p, t2p, t3); }
#endif
}

// Tile table: cut positions p[1..k-1] (u8) of every K3_TILE-th composition
// rank (16-byte records); depends on (n, k) only.
static __global__ void k_tiles(int n, int k, unsigned long long ntiles, uint8_t* out) {
    unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    int p[GP_MAX_STAGES + 1];
    d_unrank_cuts(n, k, t * K3_TILE, p);
    for (int j = 1; j < 16; ++j) out[t * 16 + j - 1] = j < k ? (uint8_t)p[j] : 0;
    out[t * 16 + 15] = 0;
}

// Generic range kernel (status-tracking): one thread per index; records the
// first erroring candidate in enumeration order.
static __global__ void __launch_bounds__(256) k3_argmin_generic(DevInst I, RangeGeom G, ArgminScratch S,
                                                         const uint32_t* only_if_flags) {
    // fix-up launch behind a fast-path kernel: do nothing unless the table
    // build raised a flag (then this kernel's result replaces the fast one)
    TL_START();
    pdl_trigger();
    pdl_wait();
    TL_WAITED();
    if (only_if_flags && *only_if_flags == 0u) { TL_STOP(40); return; }
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
        if (G.vs.out)
            vput(G.vs, 0, idx, e.status != GP_OK
                 ? __longlong_as_double(0x7ff8000000000000ll | (long long)e.status) : e.cost);
        if (e.status != GP_OK) {
            atomicMin(S.err_idx, (idx << 4) | (unsigned long long)e.status);
        } else {
            Key o{e.cost, ((perm_rank * G.NC) + comp) * (unsigned long long)G.nbm + (unsigned long long)bmi};
            if (key_less(o, mine)) mine = o;
        }
    }
    block_argmin_finish(mine, S);
}

// r[0] = the smallest of the keys r[0..n) (range split into launches)
static __global__ void k_key_combine(Key* r, int n) {
    Key b = r[0];
    for (int i = 1; i < n; ++i) if (key_less(r[i], b)) b = r[i];
    r[0] = b;
}
