/*
 * oracle.c - CPU restatement of the reference planner's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline - never as the product path.
 *
 * It re-states, candidate by candidate and in the reference's operation
 * order, what `_evaluate` (src/planner.py:313-327) computes, so that it is an
 * independent check of the table-driven CUDA engine.  src/ =
 * /root/reference/pkg/src/geopipe/.  Parity pinning: tests/test_oracle.py
 * checks this file bit-for-bit against the live reference (in the build
 * container) and against the committed fixtures in tests/golden/ generated
 * from the reference by scripts/make_golden.py.
 *
 * Compile with -ffp-contract=off (no FMA contraction): every + - * / below is
 * one IEEE double operation, exactly as CPython performs it.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/geopipe_b200.h"

#define OR_MAX_DEV GP_MAX_MEMBERS

/* ------------------------------------------------------------------------
 * CPython 3.12 builtin sum() over floats: Neumaier compensation
 * (Python/bltinmodule.c, builtin_sum_impl).  Start value is int 0, so the
 * first element enters as 0 + x0.
 * ---------------------------------------------------------------------- */
double or_psum(const double *x, size_t n)
{
    if (n == 0)
        return 0.0;
    double f = 0.0 + x[0];
    double c = 0.0;
    for (size_t i = 1; i < n; ++i) {
        double xi = x[i];
        double t = f + xi;
        if (fabs(f) >= fabs(xi))
            c += (f - t) + xi;
        else
            c += (xi - t) + f;
        f = t;
    }
    if (c != 0.0 && isfinite(c))
        f += c;
    return f;
}

/* sum over a strided generator: sum(model.layers[i].<field> for i in [a,b)) */
static double psum_range(const double *x, uint32_t a, uint32_t b)
{
    return or_psum(x + a, (size_t)(b - a));
}

/* math.isclose(a, b, rel_tol, abs_tol=0) (Modules/mathmodule.c) */
static int py_isclose(double a, double b, double rel_tol)
{
    if (a == b)
        return 1;
    if (isinf(a) || isinf(b))
        return 0;
    double diff = fabs(b - a);
    return (diff <= fabs(rel_tol * b)) || (diff <= fabs(rel_tol * a));
}

/* ------------------------------------------------------------------------
 * proportional_split (src/planner.py:65-87).  Returns 0 or
 * GP_ERR_INFEASIBLE_SPLIT.
 * ---------------------------------------------------------------------- */
int or_proportional_split(int64_t total, const double *w, int n, int minimum,
                          int64_t *shares)
{
    double wsum = or_psum(w, (size_t)n);
    double rem[GP_MAX_SGS];
    int idx[GP_MAX_SGS];
    int64_t ssum = 0;
    for (int i = 0; i < n; ++i) {
        double raw = ((double)total * w[i]) / wsum;
        shares[i] = (int64_t)floor(raw);
        rem[i] = raw - (double)shares[i];
        ssum += shares[i];
        idx[i] = i;
    }
    int64_t leftover = total - ssum;
    /* sorted(range(n), key=lambda i: (-rem[i], i)) - stable insertion sort */
    for (int i = 1; i < n; ++i) {
        int v = idx[i];
        int j = i - 1;
        while (j >= 0 && (-rem[idx[j]] > -rem[v])) {
            idx[j + 1] = idx[j];
            --j;
        }
        idx[j + 1] = v;
    }
    /* python slice [:leftover] */
    int64_t take = leftover >= 0 ? (leftover < n ? leftover : n)
                                 : (n + leftover > 0 ? n + leftover : 0);
    for (int64_t t = 0; t < take; ++t)
        shares[idx[t]] += 1;
    if (minimum > 0) {
        for (int i = 0; i < n; ++i) {
            while (shares[i] < minimum) {
                int donor = 0;
                for (int j = 1; j < n; ++j)
                    if (shares[j] > shares[donor])
                        donor = j;
                if (shares[donor] <= minimum)
                    return GP_ERR_INFEASIBLE_SPLIT;
                shares[donor] -= 1;
                shares[i] += 1;
            }
        }
    }
    return GP_OK;
}

/* ------------------------------------------------------------------------
 * split_asymmetric_tp_dp (src/planner.py:116-154).  Returns 1 and fills
 * rf/cf when a rank-1 grid exists (FactorizationError otherwise -> 0).
 * ---------------------------------------------------------------------- */
int or_tp_grid(const double *caps, int n, double *rf, double *cf)
{
    int shp_r[64], shp_c[64], ns = 0;
    for (int r = 2; r < n && ns < 64; ++r)
        if (n % r == 0 && n / r >= 2) {
            shp_r[ns] = r;
            shp_c[ns] = n / r;
            ++ns;
        }
    /* sorted(..., key=|r-c|): stable */
    for (int i = 1; i < ns; ++i) {
        int r = shp_r[i], c = shp_c[i], j = i - 1;
        while (j >= 0 && abs(shp_r[j] - shp_c[j]) > abs(r - c)) {
            shp_r[j + 1] = shp_r[j];
            shp_c[j + 1] = shp_c[j];
            --j;
        }
        shp_r[j + 1] = r;
        shp_c[j + 1] = c;
    }
    for (int s = 0; s < ns; ++s) {
        int r = shp_r[s], c = shp_c[s];
#define GRID(i, j) caps[(j) * r + (i)]
        int ok = 1;
        for (int i = 0; i < r && ok; ++i)
            for (int j = 0; j < c && ok; ++j)
                ok = py_isclose(GRID(i, j) * GRID(0, 0), GRID(i, 0) * GRID(0, j), 1e-9);
        if (!ok)
            continue;
        double rows[OR_MAX_DEV], cols[OR_MAX_DEV];
        for (int i = 0; i < r; ++i)
            rows[i] = GRID(i, 0);
        for (int j = 0; j < c; ++j)
            cols[j] = GRID(0, j);
#undef GRID
        double rsum = or_psum(rows, (size_t)r), csum = or_psum(cols, (size_t)c);
        for (int k = 0; k < n; ++k) {
            rf[k] = rows[k % r] / rsum;
            cf[k] = cols[k / r] / csum;
        }
        return 1;
    }
    return 0;
}

/* split_asymmetric_dp (src/planner.py:107-113) */
void or_dp_fractions(const double *caps, int n, double *fr)
{
    double total = or_psum(caps, (size_t)n);
    for (int i = 0; i < n; ++i)
        fr[i] = caps[i] / total;
    fr[n - 1] = 1.0 - or_psum(fr, (size_t)(n - 1));
}

/* ------------------------------------------------------------------------
 * per-candidate evaluation
 * ---------------------------------------------------------------------- */
typedef struct {
    int kind;
    int n_parts;
    uint32_t pp_start[GP_MAX_SGS], pp_end[GP_MAX_SGS];
} stage_split;

static double total_flops(const gp_instance *I, uint32_t i)
{
    /* LayerSpec.total_flops (src/plans.py:28-30) */
    return (I->fwd_flops[i] + I->bwd_input_flops[i]) + I->bwd_weight_flops[i];
}

static double psum_total_flops(const gp_instance *I, uint32_t a, uint32_t b)
{
    double buf[GP_MAX_LAYERS + 1];
    for (uint32_t i = a; i < b; ++i)
        buf[i - a] = total_flops(I, i);
    return or_psum(buf, b - a);
}

/* choose_intra_split (src/planner.py:157-200) */
static void choose_split(const gp_instance *I, uint32_t f, uint32_t a, uint32_t b,
                         stage_split *out, double *tp_rf, double *tp_cf)
{
    uint32_t m0 = I->fg_member_offset[f], m1 = I->fg_member_offset[f + 1];
    uint32_t s0 = I->fg_sg_offset[f], s1 = I->fg_sg_offset[f + 1];
    uint32_t nmem = m1 - m0, nsg = s1 - s0;
    out->n_parts = 0;
    if (nmem == 1 || nsg == 1) {
        out->kind = GP_UNIFORM;
        return;
    }
    const double *caps = I->sg_capacity + s0;
    /* split_asymmetric_pp (src/planner.py:90-104) */
    uint32_t n = b - a;
    if (nsg <= n) {
        int64_t shares[GP_MAX_SGS];
        if (or_proportional_split((int64_t)n, caps, (int)nsg, 1, shares) == GP_OK) {
            double times[GP_MAX_SGS];
            uint32_t pos = a;
            for (uint32_t j = 0; j < nsg; ++j) {
                out->pp_start[j] = pos;
                out->pp_end[j] = pos + (uint32_t)shares[j];
                pos += (uint32_t)shares[j];
                double flops = psum_total_flops(I, out->pp_start[j], out->pp_end[j]);
                times[j] = flops / caps[j];
            }
            double mean = or_psum(times, nsg) / (double)nsg;
            double mx = times[0];
            for (uint32_t j = 1; j < nsg; ++j)
                if (times[j] > mx)
                    mx = times[j];
            if (mx <= I->bottleneck_factor * mean) {
                out->kind = GP_ASYM_PP;
                out->n_parts = (int)nsg;
                return;
            }
        }
    }
    double dcaps[OR_MAX_DEV];
    for (uint32_t j = 0; j < nmem; ++j)
        dcaps[j] = I->p_c[I->fg_members[m0 + j]];
    if (or_tp_grid(dcaps, (int)nmem, tp_rf, tp_cf)) {
        out->kind = GP_ASYM_TP_DP;
        out->n_parts = (int)nmem;
        return;
    }
    out->kind = GP_ASYM_DP;
    out->n_parts = (int)nsg;
}

/* gateway_link (src/timing.py:104-113): argmin of (p_t, u, v) */
static void gateway(const gp_instance *I, uint32_t fa, uint32_t fb, uint32_t *pu,
                    uint32_t *pv)
{
    uint32_t D = I->n_devices;
    int have = 0;
    double bp = 0;
    uint32_t bu = 0, bv = 0;
    for (uint32_t x = I->fg_member_offset[fa]; x < I->fg_member_offset[fa + 1]; ++x) {
        uint32_t u = I->fg_members[x];
        for (uint32_t y = I->fg_member_offset[fb]; y < I->fg_member_offset[fb + 1]; ++y) {
            uint32_t v = I->fg_members[y];
            double p = I->p_t[(size_t)u * D + v];
            int less;
            if (!have)
                less = 1;
            else if (p != bp)
                less = p < bp;
            else if (I->id_rank[u] != I->id_rank[bu])
                less = I->id_rank[u] < I->id_rank[bu];
            else
                less = I->id_rank[v] < I->id_rank[bv];
            if (less) {
                have = 1;
                bp = p;
                bu = u;
                bv = v;
            }
        }
    }
    *pu = bu;
    *pv = bv;
}

/*
 * _evaluate (src/planner.py:313-327) for one candidate.
 * Returns a status; *cost gets the plan cost (+inf if memory-infeasible).
 */
int or_evaluate(const gp_instance *I, uint32_t k, const uint8_t *order,
                const uint8_t *counts, uint32_t bm, double *cost,
                gp_plan_info *detail)
{
    uint32_t n = I->n_layers;
    if (k < 1 || k > GP_MAX_STAGES || bm >= I->n_batch * I->n_micro)
        return GP_ERR_INPUT;
    int64_t B = I->batch[bm / I->n_micro];
    int64_t m = I->micro[bm % I->n_micro];
    /* ParallelPlan.__post_init__ (src/plans.py:106-122) */
    uint32_t starts[GP_MAX_STAGES + 1];
    uint32_t pos = 0;
    for (uint32_t s = 0; s < k; ++s) {
        if (order[s] >= I->n_fgs)
            return GP_ERR_INPUT;
        for (uint32_t t = 0; t < s; ++t)
            if (order[t] == order[s])
                return GP_ERR_INPUT;
        if (counts[s] == 0)
            return GP_ERR_INPUT;
        starts[s] = pos;
        pos += counts[s];
    }
    starts[k] = pos;
    if (pos > n)   /* slicing past the model would shrink ranges: not a plan */
        return GP_ERR_INPUT;

    /* build_plan (src/planner.py:203-223) */
    stage_split split[GP_MAX_STAGES];
    static __thread double rf[GP_MAX_STAGES][OR_MAX_DEV], cf[GP_MAX_STAGES][OR_MAX_DEV];
    for (uint32_t s = 0; s < k; ++s)
        choose_split(I, order[s], starts[s], starts[s + 1], &split[s], rf[s], cf[s]);

    /* assigned_param_bytes + memory_feasible (src/planner.py:226-253) */
    static __thread double assigned[OR_MAX_DEV];
    static __thread uint8_t touched[OR_MAX_DEV];
    uint32_t D = I->n_devices;
    memset(touched, 0, D);
    for (uint32_t s = 0; s < k; ++s) {
        uint32_t f = order[s];
        double params = psum_range(I->param_bytes, starts[s], starts[s + 1]);
        uint32_t m0 = I->fg_member_offset[f], m1 = I->fg_member_offset[f + 1];
        if (split[s].kind == GP_ASYM_PP) {
            uint32_t s0 = I->fg_sg_offset[f];
            for (int j = 0; j < split[s].n_parts; ++j) {
                double sub = psum_range(I->param_bytes, split[s].pp_start[j], split[s].pp_end[j]);
                uint32_t g = s0 + (uint32_t)j;
                for (uint32_t x = I->sg_member_offset[g]; x < I->sg_member_offset[g + 1]; ++x) {
                    uint32_t d = I->sg_members[x];
                    assigned[d] = (touched[d] ? assigned[d] : 0.0) + sub;
                    touched[d] = 1;
                }
            }
        } else if (split[s].kind == GP_ASYM_TP_DP) {
            for (uint32_t x = m0; x < m1; ++x) {
                uint32_t d = I->fg_members[x];
                double v = (params * rf[s][x - m0]) * cf[s][x - m0];
                assigned[d] = (touched[d] ? assigned[d] : 0.0) + v;
                touched[d] = 1;
            }
        } else {
            for (uint32_t x = m0; x < m1; ++x) {
                uint32_t d = I->fg_members[x];
                assigned[d] = (touched[d] ? assigned[d] : 0.0) + params;
                touched[d] = 1;
            }
        }
    }
    int feasible = 1;
    for (uint32_t d = 0; d < D; ++d)
        if (touched[d] && assigned[d] > I->memory_bytes[d]) {
            feasible = 0;
            break;
        }
    if (detail) {
        memset(detail, 0, sizeof(*detail));
        detail->k = k;
        detail->feasible = feasible;
        for (uint32_t s = 0; s < k; ++s) {
            detail->stage[s].kind = (uint32_t)split[s].kind;
            /* len(IntraSplit.parts): SGs (PP, DP) or members (TP) */
            detail->stage[s].n_parts = (uint32_t)split[s].n_parts;
            if (split[s].kind == GP_ASYM_PP) {
                for (int j = 0; j < split[s].n_parts; ++j) {
                    detail->stage[s].pp_sg[j] = (uint32_t)j;
                    detail->stage[s].pp_start[j] = split[s].pp_start[j];
                    detail->stage[s].pp_end[j] = split[s].pp_end[j];
                }
            }
        }
    }
    if (!feasible) {
        *cost = INFINITY;
        if (detail)
            detail->plan_cost = INFINITY;
        return GP_OK;
    }

    /* build_plan_timing (src/timing.py:176-231) */
    if (pos != n)
        return GP_ERR_TOPOLOGY;
    double fwd_ps[GP_MAX_STAGES], bwd_ps[GP_MAX_STAGES], wgt_ps[GP_MAX_STAGES],
        al[GP_MAX_STAGES];
    for (uint32_t s = 0; s < k; ++s) {
        uint32_t f = order[s], a = starts[s], b = starts[s + 1];
        double cap;
        /* effective_capacity (src/timing.py:116-143) */
        if (split[s].kind == GP_ASYM_PP) {
            double total = psum_total_flops(I, a, b);
            int have = 0;
            double best = 0.0;
            uint32_t s0 = I->fg_sg_offset[f];
            for (int j = 0; j < split[s].n_parts; ++j) {
                double sub = psum_total_flops(I, split[s].pp_start[j], split[s].pp_end[j]);
                double frac = sub / total;
                double capj = I->sg_capacity[s0 + (uint32_t)j];
                if (frac > 0) {
                    double val = capj / frac;
                    if (!have || val < best)
                        best = val;
                    have = 1;
                }
            }
            if (!have)
                return GP_ERR_DEGENERATE;
            cap = best;
        } else {
            cap = I->fg_capacity[f];
            if (!(cap > 0))
                return GP_ERR_DEGENERATE;
        }
        /* collective_volume + intra_group_seconds (src/timing.py:146-173) */
        uint32_t nmem = I->fg_member_offset[f + 1] - I->fg_member_offset[f];
        double params = psum_range(I->param_bytes, a, b);
        double volume = 0.0;
        if (nmem >= 2) {
            volume = 2.0 * params;
            if (split[s].kind == GP_ASYM_TP_DP)
                volume = volume + I->activation_out_bytes[b - 1] * (double)m;
        }
        if (volume == 0.0 || !I->fg_has_min_bw[f]) {
            al[s] = 0.0;
        } else {
            if (!(I->fg_min_bw[f] > 0))
                return GP_ERR_TOPOLOGY;
            al[s] = volume / I->fg_min_bw[f];
        }
        /* sync = intra_group_seconds(params, fg): raises under the same rule */
        if (params != 0.0 && I->fg_has_min_bw[f] && !(I->fg_min_bw[f] > 0))
            return GP_ERR_TOPOLOGY;
        fwd_ps[s] = psum_range(I->fwd_flops, a, b) / cap;
        bwd_ps[s] = psum_range(I->bwd_input_flops, a, b) / cap;
        wgt_ps[s] = psum_range(I->bwd_weight_flops, a, b) / cap;
    }
    double lat[GP_MAX_STAGES], bw[GP_MAX_STAGES], act[GP_MAX_STAGES];
    for (uint32_t i = 0; i + 1 < k; ++i) {
        uint32_t u, v;
        gateway(I, order[i], order[i + 1], &u, &v);
        double w = I->bandwidth[(size_t)u * D + v];
        if (!(w > 0))
            return GP_ERR_TOPOLOGY;
        bw[i] = w;
        lat[i] = I->latency[(size_t)u * D + v];
        act[i] = I->activation_out_bytes[starts[i + 1] - 1];
    }

    /* plan_cost_from_timing / stage_cost (src/costmodel.py:56-89) */
    double md = (double)m;
    int64_t M = B / m;
    double c[GP_MAX_STAGES], x[GP_MAX_STAGES];
    for (uint32_t s = 0; s < k; ++s)
        c[s] = ((fwd_ps[s] + bwd_ps[s]) + wgt_ps[s]) * md;
    for (uint32_t i = 0; i + 1 < k; ++i)
        x[i] = lat[i] + (act[i] * md) / bw[i];
    double best = 0.0;
    for (uint32_t s = 0; s < k; ++s) {
        double fill = 0.0, res = 0.0;
        for (uint32_t i = 0; i < s; ++i) {
            fill += c[i] + x[i];
            double r = x[i] - c[i + 1];
            res += (r > 0.0) ? r : 0.0;
        }
        double run = (double)M * c[s];
        double total = ((fill + run) + res) + al[s];
        if (s == 0 || total > best)
            best = total;
        if (detail) {
            detail->stage[s].fill_seconds = fill;
            detail->stage[s].run_seconds = run;
            detail->stage[s].residual_seconds = res;
            detail->stage[s].collective_seconds = al[s];
        }
    }
    *cost = best;
    if (detail)
        detail->plan_cost = best;
    return GP_OK;
}

/* ------------------------------------------------------------------------
 * exhaustive_plan (src/planner.py:374-403) over an index range
 * ---------------------------------------------------------------------- */
static uint64_t binom(uint64_t n, uint64_t r)
{
    if (r > n)
        return 0;
    uint64_t res = 1;
    for (uint64_t i = 1; i <= r; ++i)
        res = res * (n - r + i) / i;
    return res;
}

static uint64_t fact(uint32_t k)
{
    uint64_t f = 1;
    for (uint32_t i = 2; i <= k; ++i)
        f *= i;
    return f;
}

uint64_t or_space_size(const gp_instance *I)
{
    uint32_t k = I->n_fgs;
    if (k > I->n_layers)
        return 0;
    return (uint64_t)I->n_batch * I->n_micro * fact(k) * binom(I->n_layers - 1, k - 1);
}

/* permutation of 0..k-1 with lexicographic rank r */
static void unrank_perm(uint32_t k, uint64_t r, uint8_t *perm)
{
    uint8_t pool[GP_MAX_STAGES];
    for (uint32_t i = 0; i < k; ++i)
        pool[i] = (uint8_t)i;
    uint32_t left = k;
    for (uint32_t i = 0; i < k; ++i) {
        uint64_t f = fact(k - 1 - i);
        uint32_t q = (uint32_t)(r / f);
        r %= f;
        perm[i] = pool[q];
        for (uint32_t j = q; j + 1 < left; ++j)
            pool[j] = pool[j + 1];
        --left;
    }
}

/* composition of n into k positive parts with lexicographic rank r
 * (_compositions, src/planner.py:406-413) */
static void unrank_comp(uint32_t n, uint32_t k, uint64_t r, uint8_t *counts)
{
    uint32_t rem = n;
    for (uint32_t i = 0; i + 1 < k; ++i) {
        uint32_t parts = k - i;
        for (uint32_t first = 1;; ++first) {
            uint64_t cnt = binom(rem - first - 1, parts - 2);
            if (r < cnt) {
                counts[i] = (uint8_t)first;
                rem -= first;
                break;
            }
            r -= cnt;
        }
    }
    counts[k - 1] = (uint8_t)rem;
}

void or_decode(const gp_instance *I, uint64_t idx, uint8_t *order, uint8_t *counts,
               uint32_t *bm)
{
    uint32_t k = I->n_fgs;
    uint64_t nc = binom(I->n_layers - 1, k - 1), np = fact(k);
    uint64_t comp = idx % nc;
    idx /= nc;
    uint64_t perm = idx % np;
    *bm = (uint32_t)(idx / np);
    unrank_perm(k, perm, order);
    unrank_comp(I->n_layers, k, comp, counts);
}

typedef struct {
    const gp_instance *I;
    uint64_t lo, hi;
    int status;
    int have;
    double cost;
    uint64_t idx;
    uint8_t order[GP_MAX_STAGES], counts[GP_MAX_STAGES];
} range_job;

/* key (cost, (order, cuts)) strict-< then earliest index; fg index order is
 * string order, so comparing indices compares the id strings. */
static int key_less(double c1, const uint8_t *o1, const uint8_t *n1, uint64_t i1,
                    double c2, const uint8_t *o2, const uint8_t *n2, uint64_t i2,
                    uint32_t k)
{
    if (c1 != c2)
        return c1 < c2;
    for (uint32_t s = 0; s < k; ++s)
        if (o1[s] != o2[s])
            return o1[s] < o2[s];
    for (uint32_t s = 0; s < k; ++s)
        if (n1[s] != n2[s])
            return n1[s] < n2[s];
    return i1 < i2;
}

static void *range_worker(void *arg)
{
    range_job *J = (range_job *)arg;
    const gp_instance *I = J->I;
    uint32_t k = I->n_fgs;
    J->have = 0;
    J->status = GP_OK;
    for (uint64_t idx = J->lo; idx < J->hi; ++idx) {
        uint8_t order[GP_MAX_STAGES], counts[GP_MAX_STAGES];
        uint32_t bm;
        or_decode(I, idx, order, counts, &bm);
        double cost;
        int st = or_evaluate(I, k, order, counts, bm, &cost, NULL);
        if (st != GP_OK) {
            J->status = st;
            return NULL;
        }
        if (!J->have || key_less(cost, order, counts, idx, J->cost, J->order, J->counts,
                                 J->idx, k)) {
            J->have = 1;
            J->cost = cost;
            J->idx = idx;
            memcpy(J->order, order, k);
            memcpy(J->counts, counts, k);
        }
    }
    return NULL;
}

/* Argmin over [lo, hi) on `threads` host threads. */
int or_argmin_range(const gp_instance *I, uint64_t lo, uint64_t hi, int threads,
                    gp_best *out)
{
    uint32_t k = I->n_fgs;
    if (k < 1 || k > GP_MAX_STAGES || k > I->n_layers)
        return GP_ERR_INFEASIBLE_SPLIT;
    if (threads < 1)
        threads = 1;
    if (threads > 256)
        threads = 256;
    range_job jobs[256];
    pthread_t tid[256];
    uint64_t span = hi > lo ? hi - lo : 0;
    for (int t = 0; t < threads; ++t) {
        jobs[t].I = I;
        jobs[t].lo = lo + span * (uint64_t)t / (uint64_t)threads;
        jobs[t].hi = lo + span * (uint64_t)(t + 1) / (uint64_t)threads;
        if (threads == 1)
            range_worker(&jobs[0]);
        else
            pthread_create(&tid[t], NULL, range_worker, &jobs[t]);
    }
    if (threads > 1)
        for (int t = 0; t < threads; ++t)
            pthread_join(tid[t], NULL);
    memset(out, 0, sizeof(*out));
    out->k = k;
    out->evaluated = span;
    int have = 0;
    for (int t = 0; t < threads; ++t) {
        if (jobs[t].status != GP_OK)
            return jobs[t].status;
        if (!jobs[t].have)
            continue;
        if (!have || key_less(jobs[t].cost, jobs[t].order, jobs[t].counts, jobs[t].idx,
                              out->cost, out->order, out->counts, out->index, k)) {
            have = 1;
            out->cost = jobs[t].cost;
            out->index = jobs[t].idx;
            memcpy(out->order, jobs[t].order, k);
            memcpy(out->counts, jobs[t].counts, k);
        }
    }
    if (!have)
        return GP_ERR_NO_FEASIBLE;
    uint64_t per_bm = fact(k) * binom(I->n_layers - 1, k - 1);
    uint32_t bm = (uint32_t)(out->index / per_bm);
    out->batch_index = bm / I->n_micro;
    out->micro_index = bm % I->n_micro;
    return GP_OK;
}

/* Batch of explicit candidates (same layout as gp_eval_batch), threaded. */
typedef struct {
    const gp_instance *I;
    uint32_t k;
    uint64_t lo, hi;
    const uint8_t *order, *counts, *bm;
    double *cost;
    uint8_t *status;
} batch_job;

static void *batch_worker(void *arg)
{
    batch_job *J = (batch_job *)arg;
    for (uint64_t i = J->lo; i < J->hi; ++i) {
        double c = NAN;
        int st = or_evaluate(J->I, J->k, J->order + i * J->k, J->counts + i * J->k,
                             J->bm[i], &c, NULL);
        J->cost[i] = st == GP_OK ? c : NAN;
        J->status[i] = (uint8_t)st;
    }
    return NULL;
}

int or_eval_batch(const gp_instance *I, uint32_t k, uint64_t n, const uint8_t *order,
                  const uint8_t *counts, const uint8_t *bm, double *cost,
                  uint8_t *status, int threads)
{
    if (threads < 1)
        threads = 1;
    if (threads > 256)
        threads = 256;
    batch_job jobs[256];
    pthread_t tid[256];
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (batch_job){I, k, n * (uint64_t)t / (uint64_t)threads,
                              n * (uint64_t)(t + 1) / (uint64_t)threads,
                              order, counts, bm, cost, status};
        if (threads == 1)
            batch_worker(&jobs[0]);
        else
            pthread_create(&tid[t], NULL, batch_worker, &jobs[t]);
    }
    if (threads > 1)
        for (int t = 0; t < threads; ++t)
            pthread_join(tid[t], NULL);
    return GP_OK;
}

/* Every candidate of the enumeration range [lo, hi): cost[i - lo] and
 * status[i - lo] as _evaluate gives them (NaN cost where it raises); the
 * per-candidate reference for the engine's verify sink. */
typedef struct {
    const gp_instance *I;
    uint64_t lo, hi, base;
    double *cost;
    uint8_t *status;
} erange_job;

static void *erange_worker(void *arg)
{
    erange_job *J = (erange_job *)arg;
    uint32_t k = J->I->n_fgs;
    for (uint64_t idx = J->lo; idx < J->hi; ++idx) {
        uint8_t order[GP_MAX_STAGES], counts[GP_MAX_STAGES];
        uint32_t bm;
        double c = NAN;
        or_decode(J->I, idx, order, counts, &bm);
        int st = or_evaluate(J->I, k, order, counts, bm, &c, NULL);
        J->cost[idx - J->base] = st == GP_OK ? c : NAN;
        J->status[idx - J->base] = (uint8_t)st;
    }
    return NULL;
}

int or_eval_range(const gp_instance *I, uint64_t lo, uint64_t hi, double *cost,
                  uint8_t *status, int threads)
{
    uint32_t k = I->n_fgs;
    if (k < 1 || k > GP_MAX_STAGES || k > I->n_layers)
        return GP_ERR_INFEASIBLE_SPLIT;
    if (threads < 1)
        threads = 1;
    if (threads > 256)
        threads = 256;
    erange_job jobs[256];
    pthread_t tid[256];
    uint64_t span = hi > lo ? hi - lo : 0;
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (erange_job){I, lo + span * (uint64_t)t / (uint64_t)threads,
                               lo + span * (uint64_t)(t + 1) / (uint64_t)threads, lo, cost,
                               status};
        if (threads == 1)
            erange_worker(&jobs[0]);
        else
            pthread_create(&tid[t], NULL, erange_worker, &jobs[t]);
    }
    if (threads > 1)
        for (int t = 0; t < threads; ++t)
            pthread_join(tid[t], NULL);
    return GP_OK;
}

/* Per-group constants of the TP/DP splits (they depend on the group only):
 * split_asymmetric_tp_dp on device p_c in member order and
 * split_asymmetric_dp on second-level capacities (src/planner.py:188-200). */
int or_group_detail(const gp_instance *I, uint32_t f, gp_group_info *out)
{
    if (f >= I->n_fgs)
        return GP_ERR_INPUT;
    memset(out, 0, sizeof(*out));
    uint32_t m0 = I->fg_member_offset[f], m1 = I->fg_member_offset[f + 1];
    uint32_t s0 = I->fg_sg_offset[f], s1 = I->fg_sg_offset[f + 1];
    out->n_members = m1 - m0;
    out->n_sgs = s1 - s0;
    double dcaps[OR_MAX_DEV];
    for (uint32_t j = 0; j < out->n_members; ++j)
        dcaps[j] = I->p_c[I->fg_members[m0 + j]];
    out->tp_ok = or_tp_grid(dcaps, (int)out->n_members, out->tp_row, out->tp_col);
    if (out->n_sgs >= 1)
        or_dp_fractions(I->sg_capacity + s0, (int)out->n_sgs, out->dp_fraction);
    return GP_OK;
}

/* sizeof of the ABI structs, for the ctypes layout test */
size_t or_abi_sizeof(int which)
{
    switch (which) {
    case 0: return sizeof(gp_instance);
    case 1: return sizeof(gp_best);
    case 2: return sizeof(gp_plan_info);
    case 3: return sizeof(gp_group_info);
    case 4: return sizeof(gp_stage_info);
    default: return 0;
    }
}

/* ------------------------------------------------------------------------
 * PipelineEngine.run for any Policy, any NetworkTrace on the boundary links,
 * optionally the DynamicBatchAdapter and asynchronous iterations
 * (src/engine.py:125-431, src/nettrace.py:12-76, src/adapter.py:133-224).
 * A direct restatement with the reference's data structures: per
 * (stage, iteration) pools, FIFO link queues, a (time, seq) binary heap.
 * ---------------------------------------------------------------------- */
typedef struct {
    int64_t fwd_avail, fwd_taken, fwd_done, bwd_avail, bwd_taken, bwd_done;
    int64_t wq_head, wq_tail, w_done;   /* w_queue as a FIFO of sizes */
    int64_t *wq;                        /* sizes */
    int64_t *wq_id;                     /* micro-batch ids */
    int64_t fwd_next_id, bwd_next_id;
    int sync_done, opt_done, activated, first_bwd;
} sim_pool;

typedef struct {
    double t;
    uint64_t seq;
    int kind;           /* 0 op, 1 transfer */
    int s, op, it;      /* op: stage, op kind (0 F,1 B,2 W,3 S,4 O), iteration */
    int64_t size;       /* also transfer size; for transfers s=boundary, op=dir */
    double t0;          /* op / transfer start */
    int64_t mb;         /* micro-batch id (-1: None) */
} sim_ev;

/* ---- DynamicBatchAdapter (src/adapter.py:18-224) ---------------------- */
#define AD_WINDOW 20
typedef struct {
    double samples[AD_WINDOW]; /* deque(maxlen=20): ring, oldest at head */
    int head, len;
    double baseline;
    int64_t count, since;
    int degraded, exists;
} ad_window;

typedef struct {
    int64_t configured, current[GP_MAX_STAGES];
    int phase[GP_MAX_STAGES];   /* 0 FILL, 1 RUN, 2 DRAIN */
    ad_window win[2 * GP_MAX_STAGES];
    double degrade, recover;
    uint32_t actions;           /* len(adapter.actions): _apply with a change */
    gp_action *out;             /* optional action records */
} ad_state;

/* _apply (src/adapter.py:158-165); signal 0 fill, 1 drain, 2 degraded,
 * 3 recovered */
static void ad_apply(ad_state *A, double t, int s, int64_t size, int signal)
{
    if (size != A->current[s]) {
        if (A->out) {
            gp_action *a = &A->out[A->actions];
            a->t = t;
            a->stage = s;
            a->old_size = (int32_t)A->current[s];
            a->new_size = (int32_t)size;
            a->signal = (uint32_t)signal;
        }
        A->actions++;
        A->current[s] = size;
    }
}

static void ad_record(ad_window *w, double lat, int freeze)
{
    if (w->len < AD_WINDOW) {
        w->samples[(w->head + w->len) % AD_WINDOW] = lat;
        w->len++;
    } else {
        w->samples[w->head] = lat;
        w->head = (w->head + 1) % AD_WINDOW;
    }
    w->count += 1;
    w->since += 1;
    if (!freeze) {
        if (w->count == 1)
            w->baseline = lat;
        else
            w->baseline += 0.05 * (lat - w->baseline);
    }
}

/* detect_fluctuation: 0 STABLE, 1 DEGRADED, 2 RECOVERED */
static int ad_detect(const ad_window *w, int reduced, double degrade, double recover)
{
    if (w->len != AD_WINDOW || w->baseline <= 0)
        return 0;
    double buf[AD_WINDOW];
    for (int i = 0; i < w->len; ++i)
        buf[i] = w->samples[(w->head + i) % AD_WINDOW];
    double mean = or_psum(buf, (size_t)w->len) / (double)w->len;
    if (mean > degrade * w->baseline)
        return 1;
    if (reduced && mean < recover * w->baseline)
        return 2;
    return 0;
}

static int64_t ad_adjust(int64_t current, int64_t configured, int signal, int phase)
{
    if (phase == 2)
        return current / 2 > 1 ? current / 2 : 1;
    if (signal == 1)
        return current / 2 > 1 ? current / 2 : 1;
    if (signal == 2)
        return current * 2 < configured ? current * 2 : configured;
    return current;
}

static void ad_iteration_start(ad_state *A, double t, int S, int s)
{
    A->phase[s] = 0;
    int poor = 0;
    for (int b = s - 1; b <= s; ++b)
        for (int d = 0; d < 2; ++d)
            if (b >= 0 && b < S - 1 && A->win[2 * b + d].exists && A->win[2 * b + d].degraded)
                poor = 1;
    ad_apply(A, t, s, poor ? (A->configured / 2 > 1 ? A->configured / 2 : 1) : A->configured, 0);
}

static void ad_transfer_complete(ad_state *A, double t, int boundary, int dir, double raw,
                                 int64_t size)
{
    int producer = dir == 0 ? boundary : boundary + 1;
    ad_window *w = &A->win[2 * boundary + dir];
    w->exists = 1;
    int reduced = A->current[producer] < A->configured;
    ad_record(w, raw / (double)size, reduced);
    if (w->since < AD_WINDOW)
        return;
    int sig = ad_detect(w, reduced, A->degrade, A->recover);
    if (sig == 0)
        return;
    w->degraded = sig == 1;
    int64_t ns = ad_adjust(A->current[producer], A->configured, sig, A->phase[producer]);
    if (ns != A->current[producer]) {
        w->since = 0;
        ad_apply(A, t, producer, ns, sig == 1 ? 2 : 3);
    }
}

typedef struct {
    sim_ev *h;
    int n, cap;
} sim_heap;

static int ev_less(const sim_ev *a, const sim_ev *b)
{
    return a->t < b->t || (a->t == b->t && a->seq < b->seq);
}

static void heap_push(sim_heap *H, sim_ev e)
{
    if (H->n == H->cap) {
        H->cap = H->cap ? 2 * H->cap : 64;
        H->h = (sim_ev *)realloc(H->h, sizeof(sim_ev) * (size_t)H->cap);
    }
    int i = H->n++;
    H->h[i] = e;
    while (i > 0) {
        int p = (i - 1) / 2;
        if (!ev_less(&H->h[i], &H->h[p]))
            break;
        sim_ev t = H->h[i];
        H->h[i] = H->h[p];
        H->h[p] = t;
        i = p;
    }
}

static sim_ev heap_pop(sim_heap *H)
{
    sim_ev top = H->h[0];
    H->h[0] = H->h[--H->n];
    int i = 0;
    for (;;) {
        int l = 2 * i + 1, r = l + 1, m = i;
        if (l < H->n && ev_less(&H->h[l], &H->h[m]))
            m = l;
        if (r < H->n && ev_less(&H->h[r], &H->h[m]))
            m = r;
        if (m == i)
            break;
        sim_ev t = H->h[i];
        H->h[i] = H->h[m];
        H->h[m] = t;
        i = m;
    }
    return top;
}

typedef struct {
    int64_t *q_size, *q_mb;
    int *q_it;
    int64_t head, tail;
    int busy;
} sim_link;

/* NetworkTrace.multiplier (src/nettrace.py:36-43): bisect_right - 1 */
static double trace_mult(const gp_trace *tr, int link, double t)
{
    if (!tr)
        return 1.0;
    int np = (int)tr->n_points[link];
    int idx = -1;
    for (int i = 0; i < np; ++i)
        if (tr->t[link][i] <= t)
            idx = i;
    return idx < 0 ? 1.0 : tr->mult[link][idx];
}

/* transfer_end_time (src/nettrace.py:57-76) */
static double transfer_end(double start, double bytes, double base_bw, double latency,
                           const gp_trace *tr, int link)
{
    double t = start, remaining = bytes;
    if (tr) {
        int np = (int)tr->n_points[link];
        for (int i = 0; i < np; ++i) {
            double bp_t = tr->t[link][i];
            if (!(bp_t > start))
                continue;
            double bw = base_bw * trace_mult(tr, link, t);
            double span = bp_t - t;
            if (remaining <= bw * span)
                return (t + remaining / bw) + latency;
            remaining -= bw * span;
            t = bp_t;
        }
    }
    double bw = base_bw * trace_mult(tr, link, t);
    return (t + remaining / bw) + latency;
}

int or_sim_full(const gp_timing *T, int policy, int iterations, const gp_trace *trace,
                const gp_sim_options *opts, gp_sim_report *rep, double *iter_ends,
                gp_op *ops_out, gp_transfer *xf_out, gp_action *act_out, double *makespan_out);

int or_sim(const gp_timing *T, int policy, int iterations, const gp_trace *trace,
           double *makespan_out)
{
    return or_sim_full(T, policy, iterations, trace, NULL, NULL, NULL, NULL, NULL, NULL,
                       makespan_out);
}

int or_sim_1f1b(const gp_timing *T, int iterations, double *makespan_out)
{
    return or_sim(T, GP_POLICY_1F1B, iterations, NULL, makespan_out);
}

/* PipelineEngine.run (src/engine.py:230-431) with every option: policy,
 * trace, DynamicBatchAdapter hooks (src/adapter.py:167-224) and
 * asynchronous iterations (:297-314); rep / iter_ends may be NULL. */
int or_sim_full(const gp_timing *T, int policy, int iterations, const gp_trace *trace,
                const gp_sim_options *opts, gp_sim_report *rep, double *iter_ends,
                gp_op *ops_out, gp_transfer *xf_out, gp_action *act_out, double *makespan_out)
{
    const int S = (int)T->n_stages;
    if (S < 1 || S > GP_MAX_STAGES || iterations < 1)
        return GP_ERR_TIMING;
    const int adapter = opts ? (int)opts->adapter : 0;
    const int async_it = opts ? (int)opts->async_iterations : 0;
    const int64_t B = T->batch, m = T->microbatch;
    const int64_t per_it = B + 2;  /* chunks can shrink to 1 sample with the adapter */
    ad_state A;
    memset(&A, 0, sizeof(A));
    A.configured = m;
    A.out = act_out;
    A.degrade = opts ? opts->degrade_factor : 1.2;
    A.recover = opts ? opts->recover_factor : 1.05;
    double busy_f[GP_MAX_STAGES], busy_c[GP_MAX_STAGES];
    int64_t busy_n[GP_MAX_STAGES];
    uint32_t n_ops = 0, n_xfer = 0;
    for (int s = 0; s < S; ++s) {
        busy_f[s] = busy_c[s] = 0.0;
        busy_n[s] = 0;
    }
    if (iter_ends)
        for (int i = 0; i < iterations; ++i)
            iter_ends[i] = 0.0;
    for (int s = 0; s < S; ++s)
        A.current[s] = m;
    int64_t *it_fwd_done = (int64_t *)calloc((size_t)iterations, sizeof(int64_t));
    sim_pool *pools = (sim_pool *)calloc((size_t)S * iterations, sizeof(sim_pool));
    for (int i = 0; i < S * iterations; ++i) {
        pools[i].wq = (int64_t *)calloc((size_t)per_it + 1, sizeof(int64_t));
        pools[i].wq_id = (int64_t *)calloc((size_t)per_it + 1, sizeof(int64_t));
    }
#define POOL(s, it) (&pools[(s) * iterations + (it)])
    int cur[GP_MAX_STAGES], busy[GP_MAX_STAGES], closed_cnt = 0;
    int *stages_closed = (int *)calloc((size_t)iterations, sizeof(int));
    sim_link links[2 * GP_MAX_STAGES];
    const int64_t lcap = per_it * iterations + 1;
    for (int l = 0; l < 2 * (S - 1); ++l) {
        links[l].q_size = (int64_t *)calloc((size_t)lcap, sizeof(int64_t));
        links[l].q_mb = (int64_t *)calloc((size_t)lcap, sizeof(int64_t));
        links[l].q_it = (int *)calloc((size_t)lcap, sizeof(int));
        links[l].head = links[l].tail = 0;
        links[l].busy = 0;
    }
    (void)closed_cnt;
    sim_heap H = {NULL, 0, 0};
    uint64_t seq = 0;
    double now = 0.0;
    /* activate (src/engine.py:259-267) */
#define ACTIVATE(s_, it_)                                                                  \
    do {                                                                                   \
        sim_pool *q_ = POOL((s_), (it_));                                                  \
        if (!q_->activated) {                                                              \
            q_->activated = 1;                                                             \
            if ((s_) == 0)                                                                 \
                q_->fwd_avail = B;                                                         \
            if (adapter)                                                                   \
                ad_iteration_start(&A, now, S, (s_));                                      \
        }                                                                                  \
    } while (0)
    for (int s = 0; s < S; ++s) {
        cur[s] = 0;
        busy[s] = 0;
        ACTIVATE(s, 0);
    }
    /* ops[s].append(op) at start (src/engine.py:304-330) */
#define RECORD_OP(e_)                                                                      \
    do {                                                                                   \
        if (ops_out) {                                                                     \
            gp_op *o_ = &ops_out[n_ops];                                                   \
            o_->start = (e_).t0;                                                           \
            o_->end = (e_).t;                                                              \
            o_->size = (int32_t)(e_).size;                                                 \
            o_->microbatch_id = (int32_t)(e_).mb;                                          \
            o_->iteration = (uint32_t)(e_).it;                                             \
            o_->kind = (uint8_t)(e_).op;                                                   \
            o_->stage = (uint8_t)(e_).s;                                                   \
            o_->pad = 0;                                                                   \
        }                                                                                  \
        n_ops++;                                                                           \
    } while (0)

    /* try_start_link (src/engine.py:276-289) */
#define TRY_START(tnow, bnd, dir)                                                          \
    do {                                                                                   \
        sim_link *L_ = &links[2 * (bnd) + (dir)];                                           \
        if (!L_->busy && L_->head < L_->tail) {                                            \
            int64_t sz_ = L_->q_size[L_->head];                                            \
            int64_t mb_ = L_->q_mb[L_->head];                                              \
            int it_ = L_->q_it[L_->head];                                                  \
            L_->head++;                                                                    \
            L_->busy = 1;                                                                  \
            double per_ = (dir) == 0 ? T->act[bnd] : T->grad[bnd];                         \
            double end_ = transfer_end((tnow), per_ * (double)sz_, T->bw[bnd], T->lat[bnd], \
                                       trace, (bnd));                                      \
            sim_ev e_ = {end_, seq++, 1, (bnd), (dir), it_, sz_, (tnow), mb_};             \
            heap_push(&H, e_);                                                             \
        }                                                                                  \
    } while (0)

    int first = 1;
    for (;;) {
        /* dispatch(now) (src/engine.py:335-341) */
        int progress = 1;
        while (progress) {
            progress = 0;
            for (int s = 0; s < S; ++s) {
                if (busy[s])
                    continue;
                int it = cur[s];
                if (it >= iterations)
                    continue;
                sim_pool *p = POOL(s, it);
                /* _ready_op (src/engine.py:157-215): candidates F, B, W, SYNC, OPT
                 * in this order; the lowest priority wins, the earliest on ties */
                int best_pr = 100, best_k = -1;
                int64_t best_sz = 0;
                int64_t size = adapter ? A.current[s] : m;
                int64_t fwd_rem = B - p->fwd_taken;
                if (fwd_rem > 0) {
                    int64_t chunk = size < fwd_rem ? size : fwd_rem;
                    if (p->fwd_avail - p->fwd_taken >= chunk) {
                        int pr = -1;
                        if (policy == GP_POLICY_ZB_COMPACT || policy == GP_POLICY_GPIPE) {
                            pr = policy == GP_POLICY_ZB_COMPACT ? 0 : 1;
                        } else {
                            int64_t quota = (int64_t)(S - s) * m;
                            if (p->fwd_taken < quota)
                                pr = policy == GP_POLICY_ZB_ORIGINAL ? 0 : 1;
                            else if (p->fwd_taken + chunk <= quota + p->bwd_done)
                                pr = policy == GP_POLICY_ZB_ORIGINAL ? 3 : 2;
                        }
                        if (pr >= 0 && pr < best_pr) {
                            best_pr = pr;
                            best_k = 0;
                            best_sz = chunk;
                        }
                    }
                }
                int64_t bwd_rem = B - p->bwd_taken;
                int gate = policy != GP_POLICY_GPIPE || p->fwd_done == B;
                if (bwd_rem > 0 && gate) {
                    int64_t chunk = size < bwd_rem ? size : bwd_rem;
                    int64_t av = (p->bwd_avail < p->fwd_done ? p->bwd_avail : p->fwd_done) - p->bwd_taken;
                    if (s == S - 1)
                        av = p->fwd_done - p->bwd_taken;
                    int pr = (policy == GP_POLICY_ZB_COMPACT || policy == GP_POLICY_ZB_ORIGINAL) ? 1 : 2;
                    if (av >= chunk && pr < best_pr) {
                        best_pr = pr;
                        best_k = 1;
                        best_sz = chunk;
                    }
                }
                if (p->wq_head < p->wq_tail) {
                    int pr = (policy == GP_POLICY_GPIPE || policy == GP_POLICY_1F1B) ? 0 : 2;
                    if (pr < best_pr) {
                        best_pr = pr;
                        best_k = 2;
                        best_sz = p->wq[p->wq_head];
                    }
                }
                if (p->w_done == B && p->wq_head == p->wq_tail && !p->sync_done && 8 < best_pr) {
                    best_pr = 8;
                    best_k = 3;
                    best_sz = 0;
                }
                if (p->sync_done && !p->opt_done && 9 < best_pr) {
                    best_pr = 9;
                    best_k = 4;
                    best_sz = 0;
                }
                if (best_k < 0 && async_it && p->fwd_taken == B && it + 1 < iterations) {
                    /* asynchronous iterations: the next iteration's forwards may
                     * start before this one's optimizer step (src/engine.py:297-314) */
                    ACTIVATE(s, it + 1);  /* may resize the stage (on_iteration_start) */
                    size = adapter ? A.current[s] : m;
                    sim_pool *nx = POOL(s, it + 1);
                    int64_t remaining = B - nx->fwd_taken;
                    int64_t chunk = size < remaining ? size : remaining;
                    if (remaining > 0 && nx->fwd_avail - nx->fwd_taken >= chunk) {
                        nx->fwd_taken += chunk;
                        busy[s] = 1;
                        sim_ev e = {now + T->fwd[s] * (double)chunk, seq++, 0, s, 0, it + 1, chunk,
                                    now, nx->fwd_next_id};
                        heap_push(&H, e);
                        RECORD_OP(e);
                        progress = 1;
                    }
                    continue;
                }
                if (best_k < 0)
                    continue;
                double dur;
                switch (best_k) {
                case 0: dur = T->fwd[s] * (double)best_sz; p->fwd_taken += best_sz; break;
                case 1: dur = T->bwd[s] * (double)best_sz; p->bwd_taken += best_sz; break;
                case 2: dur = T->wgt[s] * (double)best_sz; p->wq_head++; break;
                case 3: dur = T->sync[s]; break;
                default: dur = T->opt[s]; break;
                }
                busy[s] = 1;
                int64_t mb = best_k == 0 ? p->fwd_next_id : best_k == 1 ? p->bwd_next_id
                             : best_k == 2 ? p->wq_id[p->wq_head - 1] : -1;
                sim_ev e = {now + dur, seq++, 0, s, best_k, it, best_sz, now, mb};
                heap_push(&H, e);
                RECORD_OP(e);
                progress = 1;
            }
        }
        if (H.n == 0)
            break;
        (void)first;
        sim_ev e = heap_pop(&H);
        now = e.t;
        if (e.kind == 0) {
            /* finish_op (src/engine.py:343-378) */
            int s = e.s, it = e.it;
            sim_pool *p = POOL(s, it);
            busy[s] = 0;
            {   /* busy[s] = sum(op.end - op.start) in op order (CPython 3.12 sum) */
                double x = now - e.t0;
                if (busy_n[s]++ == 0) {
                    busy_f[s] = 0.0 + x;
                } else {
                    double t = busy_f[s] + x;
                    if (fabs(busy_f[s]) >= fabs(x))
                        busy_c[s] += (busy_f[s] - t) + x;
                    else
                        busy_c[s] += (x - t) + busy_f[s];
                    busy_f[s] = t;
                }
            }
            if (e.op == 0) {
                p->fwd_done += e.size;
                p->fwd_next_id++;
                if (s < S - 1) {
                    sim_link *L = &links[2 * s + 0];
                    L->q_size[L->tail] = e.size;
                    L->q_mb[L->tail] = e.mb;
                    L->q_it[L->tail] = it;
                    L->tail++;
                    TRY_START(now, s, 0);
                }
                it_fwd_done[it] += e.size;
                if (adapter && it_fwd_done[it] == (int64_t)S * B)
                    for (int q = 0; q < S; ++q) {  /* on_drain: halve every stage once */
                        A.phase[q] = 2;
                        ad_apply(&A, now, q, ad_adjust(A.current[q], A.configured, 0, 2), 1);
                    }
            } else if (e.op == 1) {
                p->bwd_done += e.size;
                p->bwd_next_id++;
                p->wq_id[p->wq_tail] = e.mb;
                p->wq[p->wq_tail++] = e.size;
                if (!p->first_bwd) {
                    p->first_bwd = 1;
                    if (adapter)
                        A.phase[s] = 1;  /* on_run_phase */
                }
                if (s > 0) {
                    sim_link *L = &links[2 * (s - 1) + 1];
                    L->q_size[L->tail] = e.size;
                    L->q_mb[L->tail] = e.mb;
                    L->q_it[L->tail] = it;
                    L->tail++;
                    TRY_START(now, s - 1, 1);
                }
            } else if (e.op == 2) {
                p->w_done += e.size;
            } else if (e.op == 3) {
                p->sync_done = 1;
            } else {
                p->opt_done = 1;
                stages_closed[it] += 1;
                if (stages_closed[it] == S && iter_ends)
                    iter_ends[it] = now;
                cur[s] = it + 1;
                if (it + 1 < iterations)
                    ACTIVATE(s, it + 1);
            }
        } else {
            /* finish_transfer (src/engine.py:380-396) */
            int bnd = e.s, dir = e.op;
            links[2 * bnd + dir].busy = 0;
            if (dir == 0)
                POOL(bnd + 1, e.it)->fwd_avail += e.size;
            else
                POOL(bnd, e.it)->bwd_avail += e.size;
            if (xf_out) {  /* transfers.append(TransferRecord(...)) */
                gp_transfer *x = &xf_out[n_xfer];
                x->start = e.t0;
                x->end = now;
                x->size = (int32_t)e.size;
                x->microbatch_id = (int32_t)e.mb;
                x->iteration = (uint32_t)e.it;
                x->boundary = (uint8_t)bnd;
                x->direction = (uint8_t)dir;
                x->pad = 0;
            }
            n_xfer++;
            if (adapter)
                ad_transfer_complete(&A, now, bnd, dir, now - e.t0, e.size);
            TRY_START(now, bnd, dir);
        }
    }
    int status = GP_OK;
    for (int s = 0; s < S; ++s)
        if (cur[s] < iterations)
            status = GP_ERR_SCHEDULING;
    *makespan_out = now;
    if (rep) {
        memset(rep, 0, sizeof(*rep));
        rep->makespan = now;
        for (int s = 0; s < S; ++s)
            rep->busy[s] = (busy_c[s] != 0.0 && isfinite(busy_c[s])) ? busy_f[s] + busy_c[s] : busy_f[s];
        rep->adapter_actions = A.actions;
        rep->n_ops = n_ops;
        rep->n_transfers = n_xfer;
    }
    for (int i = 0; i < S * iterations; ++i) {
        free(pools[i].wq);
        free(pools[i].wq_id);
    }
    free(pools);
    free(stages_closed);
    free(it_fwd_done);
    for (int l = 0; l < 2 * (S - 1); ++l) {
        free(links[l].q_size);
        free(links[l].q_mb);
        free(links[l].q_it);
    }
    free(H.h);
#undef POOL
#undef TRY_START
#undef ACTIVATE
#undef RECORD_OP
    return status;
}

int or_sim_batch(const gp_timing *T, uint64_t n, int iterations, double *makespan,
                 uint8_t *status)
{
    for (uint64_t i = 0; i < n; ++i) {
        double ms = NAN;
        int st = or_sim_1f1b(&T[i], iterations, &ms);
        makespan[i] = ms;
        status[i] = (uint8_t)st;
    }
    return GP_OK;
}

int or_sim_policy_batch(const gp_timing *T, uint64_t n, int policy, int iterations,
                        const gp_trace *traces, const uint32_t *trace_index, double *makespan,
                        uint8_t *status)
{
    for (uint64_t i = 0; i < n; ++i) {
        double ms = NAN;
        const gp_trace *tr = traces ? &traces[trace_index ? trace_index[i] : 0] : NULL;
        int st = or_sim(&T[i], policy, iterations, tr, &ms);
        makespan[i] = ms;
        status[i] = (uint8_t)st;
    }
    return GP_OK;
}

/* simulate_timing reports (src/simulator.py:71-113) for a batch of timings. */
int or_sim_report_batch(const gp_timing *T, uint64_t n, int policy, int iterations,
                        const gp_trace *traces, const uint32_t *trace_index,
                        const gp_sim_options *opts, gp_sim_report *reports, double *iter_ends,
                        uint8_t *status)
{
    for (uint64_t i = 0; i < n; ++i) {
        double ms = NAN;
        const gp_trace *tr = traces ? &traces[trace_index ? trace_index[i] : 0] : NULL;
        int st = or_sim_full(&T[i], policy, iterations, tr, opts, &reports[i],
                             iter_ends ? iter_ends + i * (uint64_t)iterations : NULL, NULL, NULL,
                             NULL, &ms);
        if (st != GP_OK)
            reports[i].makespan = NAN;
        status[i] = (uint8_t)st;
    }
    return GP_OK;
}

/* ========================================================================
 * Two-level grouping (src/grouping.py): greedy agglomerative merging.
 * Devices are identified by their rank in string-sorted id order (the
 * order of ClusterTopology.device_ids, src/profiling.py:191), so tuples of
 * sorted ids compare like arrays of ranks.
 * ====================================================================== */
typedef struct {
    int n;
    int *m;                 /* sorted member ranks */
} og_group;

typedef struct {
    double key;
    int a, b;               /* group ids */
    uint64_t cnt;
} og_entry;

typedef struct {
    int level;              /* 1: network (p_t), 2: compute (p_c) */
    int D;
    const double *pt, *pc;
} og_ctx;

static int og_tuple_cmp(const og_group *x, const og_group *y)
{
    int n = x->n < y->n ? x->n : y->n;
    for (int i = 0; i < n; ++i)
        if (x->m[i] != y->m[i])
            return x->m[i] < y->m[i] ? -1 : 1;
    return x->n < y->n ? -1 : (x->n > y->n ? 1 : 0);
}

/* group_pair_metric (src/grouping.py:54-60): mean of p_t over u in a, v in b */
static double og_pair_metric(const og_ctx *c, const og_group *a, const og_group *b)
{
    size_t n = (size_t)a->n * b->n, k = 0;
    double *v = (double *)malloc(n * sizeof(double));
    for (int i = 0; i < a->n; ++i)
        for (int j = 0; j < b->n; ++j)
            v[k++] = c->pt[(size_t)a->m[i] * c->D + b->m[j]];
    double r = or_psum(v, n) / (double)n;
    free(v);
    return r;
}

/* _mean_intra_pt (:63-67); returns 0 and leaves *out for singletons */
static int og_mean_intra(const og_ctx *c, const og_group *g, double *out)
{
    if (g->n < 2)
        return 0;
    size_t n = (size_t)g->n * (g->n - 1) / 2, k = 0;
    double *v = (double *)malloc(n * sizeof(double));
    for (int i = 0; i < g->n; ++i)
        for (int j = i + 1; j < g->n; ++j)
            v[k++] = c->pt[(size_t)g->m[i] * c->D + g->m[j]];
    *out = or_psum(v, n) / (double)n;
    free(v);
    return 1;
}

static double og_mean_pc(const og_ctx *c, const og_group *g)
{
    double *v = (double *)malloc((size_t)g->n * sizeof(double));
    for (int i = 0; i < g->n; ++i)
        v[i] = c->pc[g->m[i]];
    double r = or_psum(v, (size_t)g->n) / (double)g->n;
    free(v);
    return r;
}

/* _relative_spread (:78-82) */
static double og_spread(const double *v, int n)
{
    double top = v[0], bot = v[0];
    for (int i = 1; i < n; ++i) {
        if (v[i] > top)
            top = v[i];
        if (v[i] < bot)
            bot = v[i];
    }
    if (top == 0)
        return 0.0;
    return (top - bot) / top;
}

static double og_pair_key(const og_ctx *c, const og_group *a, const og_group *b)
{
    if (c->level == 1)
        return og_pair_metric(c, a, b);
    double v[2] = {og_mean_pc(c, a), og_mean_pc(c, b)};
    return og_spread(v, 2);
}

static int og_less(const og_entry *x, const og_entry *y, const og_group *G)
{
    if (x->key != y->key)
        return x->key < y->key;
    int c = og_tuple_cmp(&G[x->a], &G[y->a]);
    if (c)
        return c < 0;
    c = og_tuple_cmp(&G[x->b], &G[y->b]);
    if (c)
        return c < 0;
    return x->cnt < y->cnt;
}

typedef struct {
    og_entry *h;
    size_t n, cap;
} og_heap;

static void og_push(og_heap *H, og_entry e, const og_group *G)
{
    if (H->n == H->cap) {
        H->cap = H->cap ? 2 * H->cap : 1024;
        H->h = (og_entry *)realloc(H->h, H->cap * sizeof(og_entry));
    }
    size_t i = H->n++;
    while (i > 0) {
        size_t p = (i - 1) / 2;
        if (!og_less(&e, &H->h[p], G))
            break;
        H->h[i] = H->h[p];
        i = p;
    }
    H->h[i] = e;
}

static og_entry og_pop(og_heap *H, const og_group *G)
{
    og_entry top = H->h[0], last = H->h[--H->n];
    size_t i = 0;
    for (;;) {
        size_t l = 2 * i + 1, r = l + 1, s = i;
        const og_entry *best = &last;
        if (l < H->n && og_less(&H->h[l], best, G)) {
            s = l;
            best = &H->h[l];
        }
        if (r < H->n && og_less(&H->h[r], best, G))
            s = r;
        if (s == i)
            break;
        H->h[i] = H->h[s];
        i = s;
    }
    if (H->n)
        H->h[i] = last;
    return top;
}

/* _agglomerate (src/grouping.py:85-143) over the (sorted) items; writes the
 * index of each item's final group in sorted(alive) order to group_of[i]
 * and returns the number of groups. */
static int og_agglomerate(const og_ctx *c, const int *items, int n, double thr, int *group_of)
{
    int cap = 2 * n + 1, ng = 0;
    og_group *G = (og_group *)calloc((size_t)cap, sizeof(og_group));
    char *alive = (char *)calloc((size_t)cap, 1);
    double *intra = (double *)calloc((size_t)cap, sizeof(double));
    char *has_intra = (char *)calloc((size_t)cap, 1);
    int *order = (int *)malloc((size_t)cap * sizeof(int));  /* alive in insertion order */
    int n_order = 0;
    for (int i = 0; i < n; ++i) {
        G[ng].n = 1;
        G[ng].m = (int *)malloc(sizeof(int));
        G[ng].m[0] = items[i];
        alive[ng] = 1;
        order[n_order++] = ng;
        ng++;
    }
    og_heap H = {NULL, 0, 0};
    uint64_t cnt = 0;
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
            og_entry e = {og_pair_key(c, &G[i], &G[j]), i, j, cnt++};
            og_push(&H, e, G);
        }
    while (H.n) {
        og_entry e = og_pop(&H, G);
        if (!alive[e.a] || !alive[e.b])
            continue;
        const og_group *a = &G[e.a], *b = &G[e.b];
        double vals[3];
        int nv;
        if (c->level == 1) {
            double cross = og_pair_metric(c, a, b);
            double va, vb;
            if (!has_intra[e.a])
                has_intra[e.a] = (char)og_mean_intra(c, a, &intra[e.a]) | 2;
            if (!has_intra[e.b])
                has_intra[e.b] = (char)og_mean_intra(c, b, &intra[e.b]) | 2;
            va = (has_intra[e.a] & 1) ? intra[e.a] : cross;
            vb = (has_intra[e.b] & 1) ? intra[e.b] : cross;
            vals[0] = va;
            vals[1] = vb;
            vals[2] = cross;
            nv = 3;
        } else {
            vals[0] = og_mean_pc(c, a);
            vals[1] = og_mean_pc(c, b);
            nv = 2;
        }
        if (og_spread(vals, nv) >= thr)
            continue;
        alive[e.a] = alive[e.b] = 0;
        og_group *mg = &G[ng];
        mg->n = a->n + b->n;
        mg->m = (int *)malloc((size_t)mg->n * sizeof(int));
        {   /* tuple(sorted(a + b)) */
            int i = 0, j = 0, k = 0;
            while (i < a->n || j < b->n)
                mg->m[k++] = (j >= b->n || (i < a->n && a->m[i] < b->m[j])) ? a->m[i++] : b->m[j++];
        }
        int mid = ng++;
        /* push_pairs(merged) over alive groups in dict order, then insert */
        int w = 0;
        for (int q = 0; q < n_order; ++q)
            if (alive[order[q]])
                order[w++] = order[q];
        n_order = w;
        for (int q = 0; q < n_order; ++q) {
            int o = order[q];
            int x = mid, y = o;
            if (og_tuple_cmp(&G[y], &G[x]) < 0) {
                x = o;
                y = mid;
            }
            og_entry ne = {og_pair_key(c, &G[x], &G[y]), x, y, cnt++};
            og_push(&H, ne, G);
        }
        alive[mid] = 1;
        order[n_order++] = mid;
    }
    /* sorted(alive): by tuple order */
    int na = 0;
    for (int q = 0; q < ng; ++q)
        if (alive[q])
            order[na++] = q;
    for (int i = 1; i < na; ++i) {  /* insertion sort, na is small */
        int v = order[i], j = i - 1;
        while (j >= 0 && og_tuple_cmp(&G[order[j]], &G[v]) > 0) {
            order[j + 1] = order[j];
            --j;
        }
        order[j + 1] = v;
    }
    for (int gi = 0; gi < na; ++gi) {
        const og_group *g = &G[order[gi]];
        for (int t = 0; t < g->n; ++t)
            for (int i = 0; i < n; ++i)
                if (items[i] == g->m[t])
                    group_of[i] = gi;
    }
    for (int q = 0; q < ng; ++q)
        free(G[q].m);
    free(G);
    free(alive);
    free(intra);
    free(has_intra);
    free(order);
    free(H.h);
    return na;
}

/* group statistics + group_second_level for a given first-level partition
 * gof[d] in sorted-member-tuple order (shared by or_group_hierarchy and the
 * fixed-partition sweep) */
static int og_second_levels(int D, const double *pt, const double *bw, const double *pc,
                            double thr_comp, const int *gof, int nf, uint16_t *fg_of,
                            uint16_t *sg_of, uint32_t *n_sg, double *fg_intra, double *fg_cap,
                            double *fg_minbw, double *sg_cap)
{
    og_ctx c1 = {1, D, pt, pc};
    uint32_t sg_base = 0;
    int *mem = (int *)malloc((size_t)D * sizeof(int));
    int *sgo = (int *)malloc((size_t)D * sizeof(int));
    double *tmp = (double *)malloc(((size_t)D * D / 2 + D + 1) * sizeof(double));
    for (int f = 0; f < nf; ++f) {
        int nm = 0;
        for (int d = 0; d < D; ++d)
            if (gof[d] == f)
                mem[nm++] = d;
        for (int i = 0; i < nm; ++i)
            fg_of[mem[i]] = (uint16_t)f;
        og_group g = {nm, mem};
        double v;
        fg_intra[f] = og_mean_intra(&c1, &g, &v) ? v : NAN;
        for (int i = 0; i < nm; ++i)
            tmp[i] = pc[mem[i]];
        fg_cap[f] = or_psum(tmp, (size_t)nm);
        if (nm < 2) {
            fg_minbw[f] = NAN;
        } else {
            double mb = INFINITY;
            for (int i = 0; i < nm; ++i)
                for (int j = i + 1; j < nm; ++j)
                    if (bw[(size_t)mem[i] * D + mem[j]] < mb)
                        mb = bw[(size_t)mem[i] * D + mem[j]];
            fg_minbw[f] = mb;
        }
        og_ctx c2 = {2, D, pt, pc};
        int ns = og_agglomerate(&c2, mem, nm, thr_comp, sgo);
        for (int i = 0; i < nm; ++i)
            sg_of[mem[i]] = (uint16_t)sgo[i];
        for (int sgi = 0; sgi < ns; ++sgi) {
            int k = 0;
            for (int i = 0; i < nm; ++i)
                if (sgo[i] == sgi)
                    tmp[k++] = pc[mem[i]];
            sg_cap[sg_base + sgi] = or_psum(tmp, (size_t)k);
        }
        sg_base += (uint32_t)ns;
    }
    *n_sg = sg_base;
    free(mem);
    free(sgo);
    free(tmp);
    return GP_OK;
}

int or_group_fixed(int D, const double *pt, const double *bw, const double *pc, const uint16_t *fg_in,
                   int nf, double thr_comp, uint16_t *sg_of, uint32_t *n_sg, double *fg_intra,
                   double *fg_cap, double *fg_minbw, double *sg_cap)
{
    if (D < 1 || nf < 1 || !(thr_comp > 0 && thr_comp < 1))
        return GP_ERR_INPUT;
    int *gof = (int *)malloc((size_t)D * sizeof(int));
    uint16_t *fg_of = (uint16_t *)malloc((size_t)D * sizeof(uint16_t));
    for (int d = 0; d < D; ++d)
        gof[d] = fg_in[d];
    int st = og_second_levels(D, pt, bw, pc, thr_comp, gof, nf, fg_of, sg_of, n_sg, fg_intra, fg_cap,
                              fg_minbw, sg_cap);
    free(gof);
    free(fg_of);
    return st;
}

/* group_first_level + group_second_level (src/grouping.py:146-228) for one
 * topology given in rank order: fg_of[d], sg_of[d] (index within the FG),
 * per FG (index f < *n_fg): intra_metric (NaN for singletons),
 * aggregate_capacity, min_intra_bandwidth (NaN for singletons); per SG in
 * FG-major order: aggregate_capacity.  Returns GP_OK / GP_ERR_INPUT. */
int or_group_hierarchy(int D, const double *pt, const double *bw, const double *pc,
                       double thr_net, double thr_comp, uint16_t *fg_of, uint16_t *sg_of,
                       uint32_t *n_fg, uint32_t *n_sg, double *fg_intra, double *fg_cap,
                       double *fg_minbw, double *sg_cap)
{
    if (D < 1)
        return GP_ERR_INPUT;  /* EmptyClusterError */
    if (!(thr_net > 0 && thr_net < 1) || !(thr_comp > 0 && thr_comp < 1))
        return GP_ERR_INPUT;  /* ValueError */
    og_ctx c1 = {1, D, pt, pc};
    int *items = (int *)malloc((size_t)D * sizeof(int));
    int *gof = (int *)malloc((size_t)D * sizeof(int));
    for (int d = 0; d < D; ++d)
        items[d] = d;
    int nf = og_agglomerate(&c1, items, D, thr_net, gof);
    *n_fg = (uint32_t)nf;
    int st = og_second_levels(D, pt, bw, pc, thr_comp, gof, nf, fg_of, sg_of, n_sg, fg_intra,
                               fg_cap, fg_minbw, sg_cap);
    free(items);
    free(gof);
    return st;
}


/* Schedules (ops + transfers) of a batch of timings at the given offsets
 * (from or_sim_report_batch's counts). */
int or_sim_schedule_batch(const gp_timing *T, uint64_t n, int policy, int iterations,
                          const gp_trace *traces, const uint32_t *trace_index,
                          const gp_sim_options *opts, const uint64_t *op_offset, gp_op *ops,
                          const uint64_t *xf_offset, gp_transfer *xfers,
                          const uint64_t *act_offset, gp_action *acts, uint8_t *status)
{
    for (uint64_t i = 0; i < n; ++i) {
        double ms = NAN;
        gp_sim_report rep;
        const gp_trace *tr = traces ? &traces[trace_index ? trace_index[i] : 0] : NULL;
        status[i] = (uint8_t)or_sim_full(&T[i], policy, iterations, tr, opts, &rep, NULL,
                                         ops + op_offset[i], xfers ? xfers + xf_offset[i] : NULL,
                                         acts ? acts + act_offset[i] : NULL, &ms);
    }
    return GP_OK;
}

/* ========================================================================
 * validate_schedule + bubble_fraction busy sums (src/schedule.py:95-182)
 * for one schedule given as gp_op records (stage lists = records of that
 * stage in array order).  The index dict keeps the first-insertion order
 * of each key and the last op stored under it, as a Python dict does.
 * ====================================================================== */
typedef struct {
    int s, kind;
    uint32_t it;
    int32_t k;
    uint64_t op;  /* last op with this key */
} ov_key;

static void ov_emit(gp_violation *out, uint32_t max_v, uint32_t *nv, int code, int stage,
                    int kind, uint32_t it, int32_t mb, double t)
{
    if (*nv < max_v) {
        gp_violation *v = &out[*nv];
        memset(v, 0, sizeof(*v));
        v->code = (uint8_t)code;
        v->stage = (uint8_t)stage;
        v->kind = (uint8_t)kind;
        v->iteration = it;
        v->microbatch_id = mb;
        v->t = t;
    }
    (*nv)++;
}

static int64_t ov_find(const ov_key *K, uint64_t nk, int s, int kind, uint32_t it, int32_t k)
{
    for (uint64_t i = 0; i < nk; ++i)
        if (K[i].s == s && K[i].kind == kind && K[i].it == it && K[i].k == k)
            return (int64_t)K[i].op;
    return -1;
}

int or_validate_schedule(const gp_timing *T, const gp_op *ops, uint64_t n, double makespan,
                         double tol_rel, uint32_t max_v, gp_violation *out, uint32_t *n_v,
                         double *busy)
{
    const int S = (int)T->n_stages;
    const double tol = tol_rel * (makespan > 1.0 ? makespan : 1.0);
    uint32_t nv = 0;
    ov_key *K = (ov_key *)malloc((n + 1) * sizeof(ov_key));
    uint64_t nk = 0;
    uint64_t *ord = (uint64_t *)malloc((n + 1) * sizeof(uint64_t));
    /* 1. end >= start, and the index */
    for (int s = 0; s < S; ++s)
        for (uint64_t i = 0; i < n; ++i) {
            const gp_op *o = &ops[i];
            if (o->stage != s)
                continue;
            if (o->end < o->start - tol)
                ov_emit(out, max_v, &nv, 0, s, o->kind, 0, 0, 0.0);
            if (o->microbatch_id >= 0) {
                uint64_t q;
                for (q = 0; q < nk; ++q)
                    if (K[q].s == s && K[q].kind == o->kind && K[q].it == o->iteration &&
                        K[q].k == o->microbatch_id)
                        break;
                if (q == nk) {
                    K[nk].s = s;
                    K[nk].kind = o->kind;
                    K[nk].it = o->iteration;
                    K[nk].k = o->microbatch_id;
                    nk++;
                }
                K[q].op = i;
            }
        }
    /* 2. overlaps in (start, end) order, stable */
    for (int s = 0; s < S; ++s) {
        uint64_t m = 0;
        for (uint64_t i = 0; i < n; ++i)
            if (ops[i].stage == s)
                ord[m++] = i;
        for (uint64_t i = 1; i < m; ++i) {  /* stable insertion sort */
            uint64_t v = ord[i];
            int64_t j = (int64_t)i - 1;
            while (j >= 0 && (ops[ord[j]].start > ops[v].start ||
                              (ops[ord[j]].start == ops[v].start && ops[ord[j]].end > ops[v].end))) {
                ord[j + 1] = ord[j];
                --j;
            }
            ord[j + 1] = v;
        }
        int have = 0;
        double prev_end = 0.0;
        for (uint64_t i = 0; i < m; ++i) {
            const gp_op *o = &ops[ord[i]];
            if (have && o->start < prev_end - tol)
                ov_emit(out, max_v, &nv, 1, s, 0, 0, 0, o->start);
            /* prev_end = max(prev_end or op.end, op.end): 0.0 is falsy */
            double base = (have && prev_end != 0.0) ? prev_end : o->end;
            prev_end = o->end > base ? o->end : base;
            have = 1;
        }
    }
    /* 3. dependencies, in index (first-insertion) order */
    for (uint64_t q = 0; q < nk; ++q) {
        const int s = K[q].s, kind = K[q].kind;
        const uint32_t it = K[q].it;
        const int32_t k = K[q].k;
        const gp_op *o = &ops[K[q].op];
        if (kind == 0 && s > 0) {
            int64_t u = ov_find(K, nk, s - 1, 0, it, k);
            if (u >= 0) {
                double arrival = ops[u].end + (T->lat[s - 1] + (T->act[s - 1] * (double)o->size) / T->bw[s - 1]);
                if (o->start < arrival - tol)
                    ov_emit(out, max_v, &nv, 2, s, 0, it, k, 0.0);
            }
        }
        if (kind == 1) {
            int64_t f = ov_find(K, nk, s, 0, it, k);
            if (f >= 0 && o->start < ops[f].end - tol)
                ov_emit(out, max_v, &nv, 3, s, 1, it, k, 0.0);
            if (s < S - 1) {
                int64_t d = ov_find(K, nk, s + 1, 1, it, k);
                if (d >= 0) {
                    double arrival = ops[d].end + (T->lat[s] + (T->grad[s] * (double)o->size) / T->bw[s]);
                    if (o->start < arrival - tol)
                        ov_emit(out, max_v, &nv, 4, s, 1, it, k, 0.0);
                }
            }
        }
        if (kind == 2) {
            int64_t b = ov_find(K, nk, s, 1, it, k);
            if (b >= 0 && o->start < ops[b].end - tol)
                ov_emit(out, max_v, &nv, 5, s, 2, it, k, 0.0);
        }
    }
    /* 4. iteration close per stage, iterations in first-appearance order */
    uint32_t *its = (uint32_t *)malloc((n + 1) * sizeof(uint32_t));
    for (int s = 0; s < S; ++s) {
        uint64_t ni = 0;
        for (uint64_t i = 0; i < n; ++i) {
            if (ops[i].stage != s)
                continue;
            uint64_t q;
            for (q = 0; q < ni; ++q)
                if (its[q] == ops[i].iteration)
                    break;
            if (q == ni)
                its[ni++] = ops[i].iteration;
        }
        for (uint64_t q = 0; q < ni; ++q) {
            int n_sync = 0, n_opt = 0, have_w = 0;
            int64_t sync = -1, opt = -1;
            double last_w = 0.0;
            for (uint64_t i = 0; i < n; ++i) {
                const gp_op *o = &ops[i];
                if (o->stage != s || o->iteration != its[q])
                    continue;
                if (o->kind == 3) { n_sync++; sync = (int64_t)i; }
                if (o->kind == 4) { n_opt++; opt = (int64_t)i; }
                if (o->kind == 2) {
                    if (!have_w || o->end > last_w)
                        last_w = o->end;
                    have_w = 1;
                }
            }
            if (n_sync != 1 || n_opt != 1) {
                ov_emit(out, max_v, &nv, 6, s, 0, its[q], 0, 0.0);
                continue;
            }
            if (ops[sync].start < last_w - tol)
                ov_emit(out, max_v, &nv, 7, s, 0, its[q], 0, 0.0);
            if (ops[opt].start < ops[sync].end - tol)
                ov_emit(out, max_v, &nv, 8, s, 0, its[q], 0, 0.0);
        }
    }
    /* bubble_fraction busy sums */
    if (busy)
        for (int s = 0; s < GP_MAX_STAGES; ++s) {
            double f = 0.0, c = 0.0;
            int64_t cnt = 0;
            for (uint64_t i = 0; i < n && s < S; ++i) {
                if (ops[i].stage != s)
                    continue;
                double x = ops[i].end - ops[i].start;
                if (cnt++ == 0) {
                    f = 0.0 + x;
                } else {
                    double t = f + x;
                    if (fabs(f) >= fabs(x))
                        c += (f - t) + x;
                    else
                        c += (x - t) + f;
                    f = t;
                }
            }
            busy[s] = (c != 0.0 && isfinite(c)) ? f + c : f;
        }
    *n_v = nv;
    free(K);
    free(ord);
    free(its);
    return GP_OK;
}
