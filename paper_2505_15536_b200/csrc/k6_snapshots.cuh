// k6_snapshots.cuh - K6: per-snapshot table patch for batched bandwidth-snapshot re-plans.
#pragma once
#include "k2_eval.cuh"

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

// One warp per (snapshot, group): the min over member pairs of the
// snapshot's bandwidth (lanes over pairs, warp min), and the gateway check
// of the group's ordered pairs (f, g).  Flags OR into the snapshot's word.
__global__ void k6_minbw(DevInst I, SnapGeom Z) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= Z.nsnap * I.F) return;
    const int sn = w / I.F, f = w % I.F;
    const double* bw = Z.bw + (size_t)sn * I.D * I.D;
    const int m0 = I.fg_off[f], nmem = I.fg_off[f + 1] - m0;
    const int npairs = nmem * (nmem - 1) / 2;
    double mn = INFINITY;
    for (int t = lane; t < npairs; t += 32) {
        // pair t -> (x, y), x < y, row-major over x
        const double h = 2.0 * nmem - 1.0;
        int x = (int)((h - sqrt(h * h - 8.0 * (double)t)) * 0.5);
        if (x < 0) x = 0;
        while (x > 0 && x * (2 * nmem - x - 1) / 2 > t) --x;
        while ((x + 1) * (2 * nmem - x - 2) / 2 <= t) ++x;
        const int y = x + 1 + (t - x * (2 * nmem - x - 1) / 2);
        GP_DCHECK(x >= 0 && x < y && y < nmem);
        const double v = bw[(size_t)I.fg_mem[m0 + x] * I.D + I.fg_mem[m0 + y]];
        mn = v < mn ? v : mn;
    }
    for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, mn, off);
        mn = o < mn ? o : mn;
    }
    bool stage_bad = false, gw_bad = false;
    if (lane == 0) {
        Z.mbw[(size_t)sn * I.F + f] = npairs ? mn : 0.0;
        stage_bad = I.fg_has_minbw[f] && !(npairs && mn > 0);
    }
    for (int g = lane; g < I.F; g += 32)
        if (g != f && !(bw[I.gw[f * I.F + g]] > 0)) gw_bad = true;
    const bool any_gw = __any_sync(0xffffffffu, gw_bad);
    if (lane == 0 && (stage_bad || any_gw))
        atomicOr(&Z.flags[sn], (stage_bad ? FLAG_STAGE_ERROR : 0u) | (any_gw ? FLAG_GATEWAY_ERROR : 0u));
}

// Per-snapshot copies of the packed stage triangles (AL = V / min_bw of the
// snapshot) and boundary rows x = lat + (act*m)/bw; grid.y = snapshot,
// 32-bit index arithmetic (one table entry per thread).
__global__ void k6_patch(DevInst I, SnapGeom Z) {
    const int n = I.n;
    const unsigned ntri = (unsigned)(n * (n + 1) / 2);
    const unsigned per_snap_tri = (unsigned)I.nm * I.F * ntri;
    const unsigned per_snap_x = (unsigned)I.nm * I.F * I.F * n;
    const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
    const int sn = blockIdx.y;
    const double* mbw = Z.mbw + (size_t)sn * I.F;
    if (t < per_snap_tri) {
        const unsigned row = t / ntri;      // mi * F + f
        const int f = (int)(row % (unsigned)I.F);
        const int e = (int)(t - row * ntri);
        // packed entry e -> (a, b): row a holds n - a entries and starts at
        // rowoff(n, a) = a*n - a(a-1)/2; invert the quadratic, then fix the
        // estimate by one step either way (exact integer checks)
        const double h = 2.0 * n + 1.0;
        int a = (int)((h - sqrt(h * h - 8.0 * (double)e)) * 0.5);
        if (a < 0) a = 0;
        if (a > n - 1) a = n - 1;
        while (a > 0 && rowoff(n, a) > e) --a;
        while (a + 1 < n && rowoff(n, a + 1) <= e) ++a;
        const int b = a + 1 + (e - rowoff(n, a));
        GP_DCHECK(a >= 0 && a < n && b > a && b <= n && rowoff(n, a) + (b - a - 1) == e);
        double2 v = I.tpk[t];
        const double V = I.vtab[t];
        const double mb = mbw[f];
        v.y = (V != 0.0 && I.fg_has_minbw[f] && mb > 0) ? V / mb : 0.0;
        Z.tpk[sn * Z.s_tpk + t] = v;
        if (b == n) Z.tcol[sn * Z.s_tcol + (size_t)row * (n + 1) + a] = v;
        if (a == 0 && b == 1)
            Z.tcol[sn * Z.s_tcol + (size_t)row * (n + 1) + n] = make_double2(INFINITY, 0.0);
    } else if (t < per_snap_tri + per_snap_x) {
        const unsigned u = t - per_snap_tri;
        const unsigned r = u / (unsigned)n;  // mi * F * F + pair
        const int j = (int)(u - r * (unsigned)n);
        const int pair = (int)(r % (unsigned)(I.F * I.F));
        const int mi = (int)(r / (unsigned)(I.F * I.F));
        const int g = I.gw[pair];
        const double md = (double)I.micro[mi];
        const double bw = Z.bw[(size_t)sn * I.D * I.D + g];
        Z.xt[sn * Z.s_xt + (size_t)r * I.nxp + j] = I.lat[g] + (I.act[j] * md) / bw;
    }
}
