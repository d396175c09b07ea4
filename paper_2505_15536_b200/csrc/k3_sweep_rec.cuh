// k3_sweep_rec.cuh - K3 sweep with per-item (a, q) records: the hot kernel of
// the snapshot re-plans (K6) for k = 3..6 stage groups.
#pragma once
#include "k3_argmin.cuh"

// Candidates of one (m, order) item are grouped into RUNS = (prefix cuts
// p1..p(k-3), a = p(k-2)); a run walks every last cut q in (a, n-1].  Along
// a run the stages 0..k-3 are fixed, and several terms of the last two
// stages' Eq. 1 chains (src/costmodel.py:68-81) depend on (a, q) or on q
// alone - not on the run:
//     D2 = max(0, x1 - c2)   x1 = x(a) of boundary k-3, c2 = C1*m of [a, q)
//     G2 = c2 + x2           x2 = x(q) of boundary k-2
//     D3 = max(0, x2 - c3)   c3 = C1*m of [q, n)
// so each CTA (one (snapshot, item) unit) tabulates them once, in shared
// memory, as
//     row records (a, q): {D2, G2, c2, AL2}     col records q: {D3, AL3, M_b*c3}
// and a q step of a run is, for the run's res1 / fill2 / mx1[b] (formed once
// per run from stage 0..k-3 entries),
//     res2 = res1 + D2,  fill3 = fill2 + G2,  res3 = res2 + D3
//     t2_b = ((fill2 + M_b*c2) + res2) + AL2,  t3_b = ((fill3 + M_b*c3) + res3) + AL3
//     cost_b = max(mx1_b, t2_b, t3_b)          (first-max)
// - every value the same IEEE operation on the same operands as the
// reference's order (the records hold the very sums, products and maxima the
// chains would compute), so every cost is bit-identical.
//
// Arg-min: a lane keeps the best (cost, key) of the candidates that meet a
// bound T - a cost some evaluated candidate has (the warp's, the CTA's and
// the snapshot's best so far), so a candidate above T cannot be the arg-min.
// cost <= T  <=>  t2 <= Tb && t3 <= Tb with Tb = T when mx1 <= T (else a
// negative bound): two compares per candidate instead of two first-max
// selects and a running minimum; the exact cost and the reference key are
// formed only for the rare candidates within the bound.  Every candidate's
// t2 and t3 are computed (the verify instantiation stores each cost).
//
// Runs come from a host-built table (prefix cuts, a, length, composition
// rank), ordered by length, in 32-run tasks; a warp's lanes therefore walk in
// lock step and read the same records (shared-memory broadcast).  Tasks go
// to the warps in snake order (lengths balance); a warp loads its next
// task's run entry and stage k-3 entry while it walks the current one, and
// the next q step's records while it computes the current one.  Rows of
// records are padded to a multiple of the q unroll with records whose totals
// are +inf (no remainder loop).
#ifndef K3R_UNROLL
#define K3R_UNROLL 2
#endif
#ifndef K3R_RB
#define K3R_RB 4  // row-record (row, lane chunk) pairs per warp in flight
#endif
#ifndef K3R_PF
#define K3R_PF 1  // next iteration's records loaded while this one computes
#endif
#ifndef K3R_GT
#define K3R_GT 1  // share the bound across the snapshot's CTAs (G.gbound)
#endif

struct __align__(16) K3RowRec { double D2, G2, c2, al2; };
// col q: D3, AL3 and M_b * c3 per batch size (the product the reference
// forms, tabulated once per item)
template <int NB>
struct __align__(16) K3ColRecN { double D3, al3, Mc3[NB]; };

__host__ __device__ inline size_t k3r_colrec_bytes(int nb) { return ((size_t)(2 + nb) * 8 + 15) & ~(size_t)15; }

// padded row length and row starts: rows a in [k-2, n-2], q in (a, n-1]
__host__ __device__ __forceinline__ int k3r_lenp(int n, int a) {
    return ((n - 1 - a) + K3R_UNROLL - 1) / K3R_UNROLL * K3R_UNROLL;
}
__host__ __device__ inline int k3r_nrecp(int n, int k) {
    int s = 0;
    for (int a = k - 2; a <= n - 2; ++a) s += k3r_lenp(n, a);
    return s;
}
// shared layout: bar 16 | rows [nrecp] | cols [n + K3R_UNROLL] | rowstart [n] u32
// (16-aligned) | row0 [n] double2 | x01 | x12 | x23 [nxp]
__host__ __device__ inline size_t k3r_rowstart_bytes(int n) { return ((size_t)n * 4 + 15) & ~(size_t)15; }
__host__ __device__ inline size_t k3r_smem(int n, int k, int nb) {
    const size_t nxp = (size_t)((n + 1) & ~1);
    return 16 + (size_t)k3r_nrecp(n, k) * sizeof(K3RowRec) + (size_t)(n + K3R_UNROLL) * k3r_colrec_bytes(nb) +
           k3r_rowstart_bytes(n) + (size_t)n * 16 + 3 * nxp * 8;
}

template <int NB, int KS, bool VER = false>
__global__ void __launch_bounds__(K3S_THREADS, K3S_MINB) k3_sweep_rec(DevInst I, SweepGeom G, ArgminScratch S,
                                                              const unsigned long long* __restrict__ binom,
                                                              const uint32_t* skip_if_flags) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ unsigned long long s_thr;  // the CTA's bound (bits of a non-negative double)
    TL_START();
    pdl_trigger();
    pdl_wait();  // K1's tables (gp_replan graph); no-op on plain launches
    TL_WAITED();
    (void)binom;
    constexpr int k = KS;
    const int n = I.n;
    const int ntri = n * (n + 1) / 2;
    const int A0 = k - 2;
    const int nrecp = G.nrecp;
    const unsigned int per_snap = G.items * (unsigned int)G.cpi;
    // CTA -> (snapshot, unit): snapshot-minor (K3R_SNAPMINOR), so a
    // snapshot's items run in different waves and the later ones start from
    // the bound the earlier ones published (fewer slow-path steps)
#ifndef K3R_SNAPMINOR
#define K3R_SNAPMINOR 1
#endif
    const unsigned int nsnap = gridDim.x / per_snap;
    const unsigned int snap = K3R_SNAPMINOR ? blockIdx.x % nsnap : blockIdx.x / per_snap;
    const unsigned int local = K3R_SNAPMINOR ? blockIdx.x / nsnap : blockIdx.x % per_snap;
    const unsigned int islot = local % G.items, csub = local / G.items;
    const unsigned long long item = G.item0 + islot;
    const int mi = (int)(item / G.NP);
    const unsigned long long perm_rank = item % G.NP;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint8_t order[GP_MAX_STAGES];
    d_unrank_perm(k, perm_rank, order);
    double Mv[NB];
#pragma unroll
    for (int bi = 0; bi < NB; ++bi) Mv[bi] = (double)(I.batch[G.b0 + bi] / I.micro[mi]);
    const double2* TPm = G.tpk + snap * G.s_tpk + (size_t)mi * I.F * ntri;
    const double* X = G.xt + snap * G.s_xt + (size_t)mi * I.F * I.F * I.nxp;
    const int f1 = order[k - 3], f2 = order[k - 2], f3 = order[k - 1];
    const double2* P1 = TPm + (size_t)f1 * ntri;
    const double2* P2 = TPm + (size_t)f2 * ntri;
    const double2* C3 = G.tcol + snap * G.s_tcol + ((size_t)mi * I.F + f3) * (n + 1);

    uint64_t* bar = (uint64_t*)smem_raw;
    K3RowRec* rrec = (K3RowRec*)(smem_raw + 16);
    K3ColRecN<NB>* crec = (K3ColRecN<NB>*)(rrec + nrecp);
    uint32_t* rstart = (uint32_t*)(crec + (n + K3R_UNROLL));
    double2* row0 = (double2*)((unsigned char*)rstart + k3r_rowstart_bytes(n));
    double* x01s = (double*)(row0 + n);
    double* x12s = x01s + I.nxp;
    double* x23s = x12s + I.nxp;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        const uint32_t rsb = (uint32_t)k3r_rowstart_bytes(n);
        mbar_expect_tx(bar, rsb + (uint32_t)(n * 16 + 3 * I.nxp * 8));
        tma_bulk_g2s(rstart, G.rowstart, rsb, bar);
        tma_bulk_g2s(row0, TPm + (size_t)order[0] * ntri, (uint32_t)n * 16, bar);
        tma_bulk_g2s(x01s, X + ((size_t)order[0] * I.F + order[1]) * I.nxp, (uint32_t)I.nxp * 8, bar);
        tma_bulk_g2s(x12s, X + ((size_t)f1 * I.F + f2) * I.nxp, (uint32_t)I.nxp * 8, bar);
        tma_bulk_g2s(x23s, X + ((size_t)f2 * I.F + f3) * I.nxp, (uint32_t)I.nxp * 8, bar);
        s_thr = 0x7FEFFFFFFFFFFFFFull;  // DBL_MAX
    }
    // the first tasks' run entries (independent of the tables)
    const int ntask = (int)((G.W + 31) / 32);
    const int wg = (int)csub * nw + wid, wstride = (int)G.cpi * nw;
    auto task_of = [&](int j) {  // snake order over the warps
        return j * wstride + ((j & 1) ? (wstride - 1 - wg) : wg);
    };
    auto load_run = [&](int j, K3Run& r) {
        const int t = task_of(j);
        const unsigned int u = (unsigned int)t * 32u + lane;
        if (t < ntask && u < G.W) {
            r = G.runs[u];
        } else {
            r.a = (uint8_t)A0;
            r.len = 0;
            r.tmax = 0;
            r.rpre = 0;
            r.p[0] = r.p[1] = r.p[2] = r.p[3] = 0;
        }
    };
    K3Run ri_a, ri_b;
    load_run(0, ri_a);
    load_run(1, ri_b);
    __syncthreads();  // mbarrier initialised
    mbar_wait(bar, 0);

    // ---- row records (a, q): one warp per row, lanes over q; padding
    // records (q > n-1) have +inf totals
    // (the (row, lane-chunk) pairs of a warp in batches of K3R_RB, loads
    // first: several L2 round trips in flight)
    {
        const int rows = n - 1 - A0;
        int a = A0 + wid, i = lane;  // the warp's first pair
        while (a <= n - 2) {
            int ba[K3R_RB], bi[K3R_RB];
            double2 e2[K3R_RB];
#pragma unroll
            for (int v = 0; v < K3R_RB; ++v) {
                ba[v] = a;
                bi[v] = i;
                if (a <= n - 2 && i < n - 1 - a) e2[v] = __ldg(&P2[rowoff(n, a) + i]);
                // next pair: next lane chunk of this row, else the warp's next row
                if (a <= n - 2) {
                    i += 32;
                    if (i >= k3r_lenp(n, a)) { a += nw; i = lane; }
                }
            }
#pragma unroll
            for (int v = 0; v < K3R_RB; ++v) {
                const int ra = ba[v], ri_ = bi[v];
                if (ra > n - 2 || ri_ >= k3r_lenp(n, ra)) continue;
                GP_DCHECK(rstart[ra] + ri_ < (uint32_t)nrecp);
                K3RowRec r;
                if (ri_ < n - 1 - ra) {
                    r.D2 = max0f(x12s[ra - 1] - e2[v].x);
                    r.G2 = e2[v].x + x23s[ra + ri_];
                    r.c2 = e2[v].x;
                    r.al2 = e2[v].y;
                } else {
                    r.D2 = r.G2 = r.c2 = 0.0;
                    r.al2 = INFINITY;
                }
                rrec[rstart[ra] + ri_] = r;
            }
        }
        (void)rows;
    }
    // ---- col records q (padding past n: +inf totals)
    for (int q = threadIdx.x; q < n + K3R_UNROLL; q += blockDim.x) {
        K3ColRecN<NB> cr;
        if (q <= n) {
            const double2 e3 = __ldg(&C3[q]);
            const double x2 = q >= 1 ? x23s[q - 1] : 0.0;
            cr.D3 = max0f(x2 - e3.x);
            cr.al3 = e3.y;
#pragma unroll
            for (int bi = 0; bi < NB; ++bi) cr.Mc3[bi] = Mv[bi] * e3.x;
        } else {
            cr.D3 = 0.0;
            cr.al3 = INFINITY;
#pragma unroll
            for (int bi = 0; bi < NB; ++bi) cr.Mc3[bi] = 0.0;
        }
        crec[q] = cr;
    }
    // stage k-3 entry of a run (L2), loaded one task ahead
    auto load_e1 = [&](const K3Run& r) -> double2 {
        const int a = r.a, pk3 = (k > 3) ? r.p[k > 3 ? k - 4 : 0] : 0;
        return r.len ? __ldg(&P1[rowoff(n, pk3) + (a - pk3 - 1)]) : make_double2(0.0, 0.0);
    };
    double2 e1_a = load_e1(ri_a);
    __syncthreads();  // records complete

    double best_c = INFINITY;  // lane best (cost, R * NB + bi) within the bound
    unsigned long long best_t = ~0ull, inf_t = ~0ull;
    double T = __longlong_as_double((long long)0x7FEFFFFFFFFFFFFFull);
    const bool skip = skip_if_flags && skip_if_flags[snap];  // generic kernel decides
    unsigned long long* const gbound = G.gbound ? G.gbound + snap : nullptr;
    unsigned long long gb_prev = (K3R_GT && gbound) ? *(volatile unsigned long long*)gbound : 0ull;
    for (int j = 0; !skip && task_of(j) < ntask; ++j) {
        const K3Run ri = ri_a;
        const double2 e1 = e1_a;
        // in flight during this task's walk: the next task's stage k-3 entry
        // and the run entries of the one after
        ri_a = ri_b;
        e1_a = load_e1(ri_a);
        load_run(j + 2, ri_b);
        {
            unsigned long long ct = *(volatile unsigned long long*)&s_thr;
            if (K3R_GT && gb_prev != 0ull && ~gb_prev < ct) ct = ~gb_prev;
            if (ct < (unsigned long long)__double_as_longlong(T)) T = __longlong_as_double((long long)ct);
            // the snapshot's bound, consumed at the next task
            if (K3R_GT && gbound) gb_prev = *(volatile unsigned long long*)gbound;
        }
        const int len = ri.len;
        const int a = ri.a;
        const unsigned long long rpre = ri.rpre;  // comp rank of (prefix, a, q = a + 1)
        // stages 0..k-3 of the run: fill2, res1 and the first-max mx1
        double fill2, res1, mx1[NB];
        {
            int p[k + 1];
            p[0] = 0;
#pragma unroll
            for (int jj = 1; jj <= k - 3; ++jj) p[jj] = ri.p[jj - 1];
            p[k - 2] = a;
            double fill = 0.0, res = 0.0, xprev = 0.0;
            double mx[NB];
#pragma unroll
            for (int bi = 0; bi < NB; ++bi) mx[bi] = -INFINITY;
#pragma unroll
            for (int s = 0; s + 3 < k; ++s) {
                double2 e;
                double x;
                if (s == 0) {
                    e = row0[p[1] > 0 ? p[1] - 1 : 0];
                    x = x01s[p[1] > 0 ? p[1] - 1 : 0];
                } else {
                    e = __ldg(&TPm[(size_t)order[s] * ntri + rowoff(n, p[s]) + (p[s + 1] - p[s] - 1)]);
                    x = __ldg(&X[((size_t)order[s] * I.F + order[s + 1]) * I.nxp + (p[s + 1] - 1)]);
                }
                if (s > 0) res = res + max0f(xprev - e.x);
#pragma unroll
                for (int bi = 0; bi < NB; ++bi) {
                    const double tot = ((fill + Mv[bi] * e.x) + res) + e.y;
                    mx[bi] = (s == 0) ? tot : gtsel(tot, mx[bi]);
                }
                fill = fill + (e.x + x);
                xprev = x;
            }
            res1 = (k > 3) ? res + max0f(xprev - e1.x) : res;
#pragma unroll
            for (int bi = 0; bi < NB; ++bi) {
                const double t1 = ((fill + Mv[bi] * e1.x) + res1) + e1.y;
                mx1[bi] = (k > 3) ? gtsel(t1, mx[bi]) : t1;
            }
            fill2 = fill + (e1.x + x12s[a - 1]);
        }
        const int lenp = len ? k3r_lenp(n, a) : 0;
        const int lmax = __shfl_sync(0xffffffffu, ri.tmax, 0);  // the task's longest (lane 0 holds a run)
        const K3RowRec* rp = rrec + rstart[a];
        const K3ColRecN<NB>* cp = crec + (a + 1);
        // the run's first key: the lane's answer when none of its candidates
        // is finite (every cost +inf: the earliest key wins)
        if (len > 0) inf_t = rpre * NB < inf_t ? rpre * NB : inf_t;
        // per batch size: cost = max(mx1, t2, t3) <= T  <=>  t2 <= Tb && t3 <= Tb
        // with Tb = T when mx1 <= T, else a negative bound
        double Tb[NB];
        auto set_bounds = [&]() {
#pragma unroll
            for (int bi = 0; bi < NB; ++bi) Tb[bi] = (len > 0 && mx1[bi] <= T) ? T : -1.0;
        };
        set_bounds();
        auto step_rc = [&](int i, const K3RowRec& R, const K3ColRecN<NB>& Cq, double* t2, double* t3) -> bool {
            const double res2 = res1 + R.D2;
            const double fill3 = fill2 + R.G2;
            const double res3 = res2 + Cq.D3;
            bool p = false;
#pragma unroll
            for (int bi = 0; bi < NB; ++bi) {
                t2[bi] = ((fill2 + Mv[bi] * R.c2) + res2) + R.al2;
                t3[bi] = ((fill3 + Cq.Mc3[bi]) + res3) + Cq.al3;
                p |= (t2[bi] <= Tb[bi]) & (t3[bi] <= Tb[bi]);
                if constexpr (VER)
                    if (i < len)
                        vput(G.vs, snap,
                             ((((unsigned long long)(G.b0 + bi) * I.nm + mi) * G.NP + perm_rank) * G.NC) +
                                 rpre + (unsigned long long)i,
                             gtsel(t3[bi], gtsel(t2[bi], mx1[bi])));
            }
            return p;
        };
        auto step = [&](int i, double* t2, double* t3) -> bool {
            GP_DCHECK(rstart[a] + i < (uint32_t)nrecp && a + 1 + i < n + K3R_UNROLL);
            return step_rc(i, rp[i], cp[i], t2, t3);
        };
        // a candidate within the bound: its exact cost (first-max, the
        // reference's order) against the lane's best under the full key
        auto take = [&](int i, const double* t2, const double* t3) {
#pragma unroll
            for (int bi = 0; bi < NB; ++bi) {
                const double c = gtsel(t3[bi], gtsel(t2[bi], mx1[bi]));
                const unsigned long long tk = (rpre + (unsigned long long)i) * NB + bi;
                if (c < best_c || (c == best_c && tk < best_t)) { best_c = c; best_t = tk; }
            }
        };
        // the warp's bound: min of its lanes' best costs, shared with the CTA
        // and the snapshot
        auto refresh = [&]() {
            unsigned long long m = __double_as_longlong(best_c);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const unsigned long long o = __shfl_xor_sync(0xffffffffu, m, off);
                m = o < m ? o : m;
            }
            if (m < (unsigned long long)__double_as_longlong(T)) {
                if (lane == 0) {
                    atomicMin(&s_thr, m);
                    if (K3R_GT && gbound) atomicMax(gbound, ~m);
                }
                T = __longlong_as_double((long long)m);
            }
            set_bounds();
        };
#if K3R_PF
        // records of the next iteration loaded while this one computes
        K3RowRec Rn[K3R_UNROLL];
        K3ColRecN<NB> Cn[K3R_UNROLL];
#pragma unroll
        for (int uu = 0; uu < K3R_UNROLL; ++uu) { Rn[uu] = rp[uu]; Cn[uu] = cp[uu]; }
#endif
        for (int i0 = 0; i0 < lmax; i0 += K3R_UNROLL) {
            // lanes past their (padded) row: no candidate (in-range reads)
            const bool act = i0 < lenp;
            const int ib = act ? i0 : 0;
            double t2[K3R_UNROLL][NB], t3[K3R_UNROLL][NB];
            bool p[K3R_UNROLL], any = false;
#if K3R_PF
            K3RowRec Rc[K3R_UNROLL];
            K3ColRecN<NB> Cc[K3R_UNROLL];
#pragma unroll
            for (int uu = 0; uu < K3R_UNROLL; ++uu) { Rc[uu] = Rn[uu]; Cc[uu] = Cn[uu]; }
            {
                const int inx = i0 + K3R_UNROLL;
                const int ibn = inx < lenp ? inx : 0;
                if (inx < lmax) {
#pragma unroll
                    for (int uu = 0; uu < K3R_UNROLL; ++uu) { Rn[uu] = rp[ibn + uu]; Cn[uu] = cp[ibn + uu]; }
                }
            }
#pragma unroll
            for (int uu = 0; uu < K3R_UNROLL; ++uu) {
                p[uu] = step_rc(ib + uu, Rc[uu], Cc[uu], t2[uu], t3[uu]) & act;
                any |= p[uu];
            }
#else
#pragma unroll
            for (int uu = 0; uu < K3R_UNROLL; ++uu) {
                p[uu] = step(ib + uu, t2[uu], t3[uu]) & act;
                any |= p[uu];
            }
#endif
            if (__any_sync(0xffffffffu, any)) {
#pragma unroll
                for (int uu = 0; uu < K3R_UNROLL; ++uu)
                    if (p[uu]) take(i0 + uu, t2[uu], t3[uu]);
                refresh();
            }
        }
    }
    Key mine{INFINITY, ~0ull};
    if (best_t == ~0ull) best_t = inf_t;  // nothing finite within the bound
    if (best_t != ~0ull) {
        const unsigned long long rr = best_t / NB, bi = best_t % NB;
        GP_DCHECK(rr < G.NC);
        mine.cost = best_c;
        mine.tie = ((perm_rank * G.NC) + rr) * (unsigned long long)G.nbm +
                   (unsigned long long)((G.b0 + bi) * I.nm + mi);
    }
    ArgminScratch Ss = S;
    Ss.blk = S.blk + (size_t)snap * per_snap;
    Ss.counter = S.counter + snap;
    Ss.result = S.result + snap;
    Ss.rearm = nullptr;
    Ss.nrearm = 0;
    block_argmin_finish(mine, Ss, per_snap, local);
    TL_STOP(31);
}
