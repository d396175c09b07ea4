// k3_sweep_rec.cuh - K3 sweep with per-item (a, q) records (the hot kernel of
// the exhaustive and snapshot re-plans for k = 3..6 stage groups).
#pragma once
#include "k3_argmin.cuh"

// Same enumeration, run structure, task queue and reduction as k3_sweep
// (k3_argmin.cuh).  What changes is the q walk.  Along a run the prefix
// stages are fixed and only the last two stages [a, q) and [q, n) vary, and
// several terms of their Eq. 1 chains (src/costmodel.py:68-81) depend on
// (a, q) or on q alone - not on the run:
//     D2 = max(0, x1 - c2)   x1 = x(a) of boundary k-3, c2 = C1*m of [a, q)
//     G2 = c2 + x2           x2 = x(q) of boundary k-2
//     D3 = max(0, x2 - c3)   c3 = C1*m of [q, n)
// so each CTA tabulates them once per item, in shared memory, as records
//     row (a, q): {D2, G2, c2, AL2}      col q: {D3, c3, AL3}
// and a q step of a run is, for the run's res1 / fill2 / mx1[b],
//     res2 = res1 + D2,  fill3 = fill2 + G2,  res3 = res2 + D3
//     t2_b = ((fill2 + M_b*c2) + res2) + AL2,  t3_b = ((fill3 + M_b*c3) + res3) + AL3
//     cost_b = max(mx1_b, t2_b, t3_b)          (first-max)
// - every value the same IEEE operation on the same operands as the
// reference's order (the records hold the very sums and maxima the chains
// would compute), so the costs are bit-identical; the q step drops from 6
// adds + 2 integer max0 + 2 NB multiplies + 6 NB adds to 3 + 2 NB + 6 NB
// with no integer work.  Rows hold only a in [k-2, n-2], q in [a+1, n-1]
// (the pairs a sweep visits): (n-k+1)(n-k+2)/2 records of 32 B.  The run
// minimum is kept per batch size (shorter select chains) and merged under
// the reference key at the end of the run.
#ifndef K3R_UNROLL
#define K3R_UNROLL 2
#endif

struct __align__(16) K3RowRec { double D2, G2, c2, al2; };
struct __align__(16) K3ColRec { double D3, c3, al3, pad; };

// records of the compact (a, q) triangle before row a (a >= A0 = k-2)
__device__ __forceinline__ int k3r_rowbase(int n, int A0, int a) {
    // sum_{j=A0}^{a-1} (n-1-j)
    return (a - A0) * (n - 1) - ((a - 1) * a / 2 - (A0 - 1) * A0 / 2);
}

__host__ __device__ inline size_t k3r_smem(int n, int k, int ngroups) {
    const size_t nrec = (size_t)(n - k + 1) * (n - k + 2) / 2;
    const size_t nxp = (size_t)((n + 1) & ~1);
    return 16 + (((size_t)(n + 1) * (k + 1) * 8 + 15) & ~(size_t)15) + (size_t)ngroups * 16 +
           nrec * sizeof(K3RowRec) + (size_t)(n + 1) * sizeof(K3ColRec) + (size_t)n * 16 +
           nxp * 8;
}

template <int NB, int KS, bool VER = false>
__global__ void __launch_bounds__(K3S_THREADS, K3S_MINB) k3_sweep_rec(DevInst I, SweepGeom G, ArgminScratch S,
                                                              const unsigned long long* __restrict__ binom,
                                                              const uint32_t* skip_if_flags) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TL_START();
    pdl_trigger();
    pdl_wait();  // K1's tables (gp_replan graph); no-op on plain launches
    TL_WAITED();
    constexpr int k = KS;
    const int n = I.n;
    const int ntri = n * (n + 1) / 2;
    constexpr int KB = k + 1;
    const int A0 = k - 2;
    const unsigned int per_snap = G.items * (unsigned int)G.cpi;
    const unsigned int snap = blockIdx.x / per_snap, local = blockIdx.x % per_snap;
    const unsigned long long islot = !G.interleave ? local / G.cpi : local % G.items;
    const unsigned long long item = G.item0 + islot;
    const int mi = (int)(item / G.NP);
    const unsigned long long perm_rank = item % G.NP;
    uint8_t order[GP_MAX_STAGES];
    d_unrank_perm(k, perm_rank, order);
    double Mv[NB];
#pragma unroll
    for (int bi = 0; bi < NB; ++bi) Mv[bi] = (double)(I.batch[G.b0 + bi] / I.micro[mi]);
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

    // shared: mbarrier | binom | groups | row records | col records | row0 | x01
    uint64_t* bar = (uint64_t*)smem_raw;
    unsigned long long* bn = (unsigned long long*)(smem_raw + 16);
    const uint32_t bn_bytes = (uint32_t)(((size_t)(n + 1) * KB * 8 + 15) & ~(size_t)15);
    uint4* grp = (uint4*)(smem_raw + 16 + bn_bytes);
    K3RowRec* rrec = (K3RowRec*)(grp + G.ngroups);
    const int nrec = (n - k + 1) * (n - k + 2) / 2;
    K3ColRec* crec = (K3ColRec*)(rrec + nrec);
    double2* row0 = (double2*)(crec + (n + 1));
    double* x01s = (double*)(row0 + n);
    const uint32_t bytes = bn_bytes + (uint32_t)G.ngroups * 16 + (uint32_t)n * 16 +
                           (uint32_t)I.nxp * 8;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_expect_tx(bar, bytes);
        tma_bulk_g2s(bn, G.bnk, bn_bytes, bar);
        tma_bulk_g2s(grp, G.groups, (uint32_t)G.ngroups * 16, bar);
        tma_bulk_g2s(row0, P0, (uint32_t)n * 16, bar);
        tma_bulk_g2s(x01s, X01, (uint32_t)I.nxp * 8, bar);
    }
    // records, one warp per row a (lanes over q), straight from L2
    {
        const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
        for (int a = A0 + wid; a <= n - 2; a += nw) {
            const double x1 = __ldg(&X12[a - 1]);
            const double2* prow = P2 + (rowoff(n, a) - a - 1);
            K3RowRec* rr = rrec + (k3r_rowbase(n, A0, a) - a - 1);
            for (int q = a + 1 + lane; q <= n - 1; q += 32) {
                GP_DCHECK(k3r_rowbase(n, A0, a) - a - 1 + q < nrec);
                const double2 e2 = __ldg(&prow[q]);
                const double x2 = __ldg(&X23[q - 1]);
                K3RowRec r;
                r.D2 = max0f(x1 - e2.x);
                r.G2 = e2.x + x2;
                r.c2 = e2.x;
                r.al2 = e2.y;
                rr[q] = r;
            }
        }
        for (int q = threadIdx.x; q <= n; q += blockDim.x) {
            K3ColRec cr;
            const double2 e3 = __ldg(&C3[q]);
            const double x2 = q >= 1 ? __ldg(&X23[q - 1]) : 0.0;
            cr.D3 = max0f(x2 - e3.x);
            cr.c3 = e3.x;
            cr.al3 = e3.y;
            cr.pad = 0.0;
            crec[q] = cr;
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
        int len = 0, a = A0 > 0 ? A0 : 1, q0 = a + 1;  // idle lanes keep in-range addresses
        double fill2 = 0.0, res1 = 0.0;
        double mx1[NB];
#pragma unroll
        for (int bi = 0; bi < NB; ++bi) mx1[bi] = -INFINITY;
        unsigned long long rpre = 0;  // comp rank of (prefix, a, q = a + 1)
        if (u < G.W) {
            int gi = ((const uint16_t*)(grp + G.ng))[t];
            while (gi + 1 < G.ng && grp[gi + 1].x <= u) ++gi;
            const uint4 g = grp[gi];
            const unsigned int lo = u - g.x;
            a = (int)(g.y & 0xffffu);
            len = (int)(g.y >> 16);
            unsigned int row;
            if (g.w) { const unsigned seg = lo / g.z; row = lo - seg * g.z; q0 = a + 1 + (int)seg * K3_SEG; }
            else { row = lo; q0 = n - len; }
            int p[k + 1];
            p[0] = 0;
            if (k == 4) {
                p[1] = (int)row + 1;
            } else if (k > 3) {
                const uint8_t* pr = G.prefixes + (size_t)row * 16;
#pragma unroll
                for (int j = 1; j <= k - 3; ++j) p[j] = pr[j - 1];
            }
            p[k - 2] = a;
            GP_DCHECK(gi < G.ng && a >= k - 2 && a <= n - 2 && len >= 1 && len <= K3_SEG &&
                      q0 >= a + 1 && q0 + len - 1 <= n - 1);
#pragma unroll
            for (int j = 1; j <= k - 2; ++j)
                rpre += bn[(n - p[j - 1] - 1) * KB + (k - j)] - bn[(n - p[j]) * KB + (k - j)];
            // stages 0..k-4 (fixed by the prefix)
            double fill = 0.0, res = 0.0, xprev = 0.0;
            double mx[NB];
#pragma unroll
            for (int bi = 0; bi < NB; ++bi) mx[bi] = -INFINITY;
#pragma unroll
            for (int s = 0; s + 3 < k; ++s) {
                double2 e;
                double x;
                if (s == 0) {
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
            const double2 e1 = __ldg(&P1[rowoff(n, pk3) - pk3 - 1 + a]);
            const double x1 = __ldg(&X12[a - 1]);
            res1 = (k > 3) ? res + max0f(xprev - e1.x) : res;
#pragma unroll
            for (int bi = 0; bi < NB; ++bi) {
                double t1 = ((fill + Mv[bi] * e1.x) + res1) + e1.y;
                mx1[bi] = (k > 3) ? gtsel(t1, mx[bi]) : t1;
            }
            fill2 = fill + (e1.x + x1);
        }
        int lmax = len, lmin = len;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            int o = __shfl_xor_sync(0xffffffffu, lmax, off);
            lmax = o > lmax ? o : lmax;
            o = __shfl_xor_sync(0xffffffffu, lmin, off);
            lmin = o < lmin ? o : lmin;
        }
        const K3RowRec* rp = rrec + (k3r_rowbase(n, A0, a) - a - 1) + q0;
        const K3ColRec* cp = crec + q0;
        // per batch size: the run minimum (strict <: earliest q wins; the first
        // q stands when every cost is +inf)
        double run_c[NB];
        int run_q[NB];
#pragma unroll
        for (int bi = 0; bi < NB; ++bi) { run_c[bi] = INFINITY; run_q[bi] = 0; }
        auto eval_q = [&](int i) {
            GP_DCHECK(i >= 0 && i < len && k3r_rowbase(n, A0, a) - a - 1 + q0 + i < nrec);
            const K3RowRec R = rp[i];
            const K3ColRec Cq = cp[i];
            const double res2 = res1 + R.D2;
            const double fill3 = fill2 + R.G2;
            const double res3 = res2 + Cq.D3;
#pragma unroll
            for (int bi = 0; bi < NB; ++bi) {
                const double t2 = ((fill2 + Mv[bi] * R.c2) + res2) + R.al2;
                const double t3 = ((fill3 + Mv[bi] * Cq.c3) + res3) + Cq.al3;
                double c = gtsel(t2, mx1[bi]);
                c = gtsel(t3, c);
                if constexpr (VER)
                    vput(G.vs, snap,
                         ((((unsigned long long)(G.b0 + bi) * I.nm + mi) * G.NP + perm_rank) * G.NC) +
                             rpre + (unsigned long long)(q0 + i - a - 1), c);
                if (c < run_c[bi]) { run_c[bi] = c; run_q[bi] = i; }
            }
        };
        int i0 = 0;
        for (; i0 + K3R_UNROLL - 1 < lmin; i0 += K3R_UNROLL) {
#pragma unroll
            for (int uu = 0; uu < K3R_UNROLL; ++uu) eval_q(i0 + uu);
        }
        for (int i = i0; i < lmax; ++i)
            if (i < len) eval_q(i);
        if (len > 0) {
#pragma unroll
            for (int bi = 0; bi < NB; ++bi) {
                const unsigned long long tk =
                    (rpre + (unsigned long long)(q0 + run_q[bi] - a - 1)) * NB + bi;
                if (run_c[bi] < best_c || (run_c[bi] == best_c && tk < best_t)) {
                    best_c = run_c[bi];
                    best_t = tk;
                }
            }
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
    block_argmin_finish(mine, Ss, per_snap, local);
    TL_STOP(31);
}
