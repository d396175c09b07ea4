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

