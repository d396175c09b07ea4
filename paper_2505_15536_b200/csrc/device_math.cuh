// device_math.cuh - scalar rules of the reference's arithmetic, on the device.
//
// Every function here reproduces one CPython / reference rule bit for bit.
// The translation unit is compiled with -fmad=false and IEEE division
// (-prec-div=true, the default without --use_fast_math): each + - * / is one
// correctly rounded double operation, as in CPython.
#pragma once
#include <cstdint>

#include "../../include/geopipe_b200.h"

namespace gpd {

// ---- CPython 3.12 builtin sum over floats (Neumaier), streaming form ----
// State after the first element x0 is (f = 0 + x0, c = 0); each further
// element updates (f, c); the value is f + c when c is a finite non-zero.
struct NeumaierSum {
    double f, c;
    __host__ __device__ void start(double x0) { f = 0.0 + x0; c = 0.0; }
    __host__ __device__ void add(double x) {
        // c += (big - t) + small with big the operand of larger magnitude
        // (selects instead of a divergent branch; identical arithmetic)
        const double t = f + x;
        const bool fb = fabs(f) >= fabs(x);
        const double big = fb ? f : x, small = fb ? x : f;
        c += (big - t) + small;
        f = t;
    }
    __host__ __device__ double value() const {
        return (c != 0.0 && isfinite(c)) ? f + c : f;
    }
};

__host__ __device__ inline double psum(const double* x, int n) {
    if (n <= 0) return 0.0;
    NeumaierSum s;
    s.start(x[0]);
    for (int i = 1; i < n; ++i) s.add(x[i]);
    return s.value();
}

// math.isclose(a, b, rel_tol=rel, abs_tol=0)
__host__ __device__ inline bool py_isclose(double a, double b, double rel) {
    if (a == b) return true;
    if (isinf(a) || isinf(b)) return false;
    double diff = fabs(b - a);
    return (diff <= fabs(rel * b)) || (diff <= fabs(rel * a));
}

// proportional_split(total, weights, minimum) (src/planner.py:65-87).
// Returns false where the reference raises InfeasibleSplitError.
__host__ __device__ inline bool proportional_split(int total, const double* w, int n,
                                                   int minimum, int* shares) {
    double wsum = psum(w, n);
    double rem[GP_MAX_SGS];
    int idx[GP_MAX_SGS];
    long long ssum = 0;
    for (int i = 0; i < n; ++i) {
        double raw = ((double)total * w[i]) / wsum;
        double fl = floor(raw);
        shares[i] = (int)fl;
        rem[i] = raw - fl;
        ssum += shares[i];
        idx[i] = i;
    }
    long long leftover = (long long)total - ssum;
    // sorted(range(n), key=(-rem[i], i)): stable insertion sort on -rem
    for (int i = 1; i < n; ++i) {
        int v = idx[i];
        int j = i - 1;
        while (j >= 0 && (-rem[idx[j]] > -rem[v])) { idx[j + 1] = idx[j]; --j; }
        idx[j + 1] = v;
    }
    long long take = leftover >= 0 ? (leftover < n ? leftover : n)
                                   : (n + leftover > 0 ? n + leftover : 0);
    for (long long t = 0; t < take; ++t) shares[idx[t]] += 1;
    if (minimum > 0) {
        for (int i = 0; i < n; ++i) {
            while (shares[i] < minimum) {
                int donor = 0;
                for (int j = 1; j < n; ++j)
                    if (shares[j] > shares[donor]) donor = j;
                if (shares[donor] <= minimum) return false;
                shares[donor] -= 1;
                shares[i] += 1;
            }
        }
    }
    return true;
}

// split_asymmetric_tp_dp (src/planner.py:116-154) on device capacities in
// member order.  Returns true and fills rf/cf when a rank-1 grid exists.
__host__ __device__ inline bool tp_grid(const double* caps, int n, double* rf, double* cf) {
    // candidate shapes (r, n/r), r in [2, n), stably sorted by |r - c|
    int shp[64], ns = 0;
    for (int r = 2; r < n && ns < 64; ++r)
        if (n % r == 0 && n / r >= 2) shp[ns++] = r;
    for (int i = 1; i < ns; ++i) {
        int r = shp[i], j = i - 1;
        int key = r - n / r; key = key < 0 ? -key : key;
        while (j >= 0) {
            int kj = shp[j] - n / shp[j]; kj = kj < 0 ? -kj : kj;
            if (kj <= key) break;
            shp[j + 1] = shp[j];
            --j;
        }
        shp[j + 1] = r;
    }
    for (int s = 0; s < ns; ++s) {
        int r = shp[s], c = n / r;
        bool ok = true;
        for (int i = 0; i < r && ok; ++i)
            for (int j = 0; j < c && ok; ++j)
                ok = py_isclose(caps[j * r + i] * caps[0], caps[i] * caps[j * r], 1e-9);
        if (!ok) continue;
        // rows = grid[i][0] = caps[i]; cols = grid[0][j] = caps[j*r]
        NeumaierSum rs, cs;
        rs.start(caps[0]);
        for (int i = 1; i < r; ++i) rs.add(caps[i]);
        cs.start(caps[0]);
        for (int j = 1; j < c; ++j) cs.add(caps[j * r]);
        double rsum = rs.value(), csum = cs.value();
        for (int k = 0; k < n; ++k) {
            rf[k] = caps[k % r] / rsum;
            cf[k] = caps[(k / r) * r] / csum;
        }
        return true;
    }
    return false;
}

// split_asymmetric_dp (src/planner.py:107-113)
__host__ __device__ inline void dp_fractions(const double* caps, int n, double* fr) {
    double total = psum(caps, n);
    for (int i = 0; i < n; ++i) fr[i] = caps[i] / total;
    fr[n - 1] = 1.0 - psum(fr, n - 1);
}

// Python max(0.0, x)
__host__ __device__ inline double max0(double x) { return x > 0.0 ? x : 0.0; }

}  // namespace gpd
