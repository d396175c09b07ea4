// k4_bnb.cuh - K4: exact branch-and-bound arg-min with the exact-in-reals DP bound.
#pragma once
#include "k2_eval.cuh"

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

