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

