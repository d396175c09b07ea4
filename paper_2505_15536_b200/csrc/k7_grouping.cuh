// k7_grouping.cuh - K7: two-level device grouping (group_first_level +
// group_second_level, src/grouping.py:85-228), one CTA per topology snapshot.
#pragma once
#include "common.cuh"

// ----------------------------------------------------------------------------
// The reference merges greedily from a heap of (key, a, b, counter) entries.
// Every live pair of groups has exactly one entry, pushed when the younger of
// the two groups was created, and its key depends only on the two member
// sets, so the heap pops the live pair with the smallest (key, a, b) where
// groups compare as sorted tuples of ids.  Live groups are disjoint, so the
// tuple order is the order of their smallest member; each group therefore
// lives in the slot of its smallest member (device rank, or local index for
// the second level), and the pop is an arg-min over (key, slot a, slot b).
//
// Instead of a heap the CTA keeps, per slot a, the best live pair (a, b > a)
// of its row (row minima in shared memory); a pop is a CTA arg-min over the
// row minima.  After a merge of b into a, only rows that pointed at a or b
// are rescanned; the others compare against their new pair (c, a).
// A pair that fails the merge predicate is dropped for good, as the
// reference's discarded heap entry is.
//
// Keys and merge values are the reference's sums (CPython 3.12 sum, i.e.
// Neumaier) over the reference's operand order, computed by one thread each:
// group_pair_metric runs u over the first group's sorted members and v over
// the second's (:54-60); _mean_intra_pt runs over combinations of the sorted
// members (:63-67); mean_pc over the members (:203-204).
// ----------------------------------------------------------------------------
#define K7_THREADS 256

// pair tables: keys, members, merge buffer, live flags (16-B aligned)
__host__ __device__ __forceinline__ size_t k7_scratch_bytes(int D) {
    size_t b = (size_t)D * D * 8 + (size_t)D * D * 2 + (size_t)D * 2 + (size_t)D * D;
    return (b + 15) & ~(size_t)15;
}

// per-slot arrays at the head of dynamic shared memory
__host__ __device__ __forceinline__ size_t k7_smem_head(int D) {
    return ((size_t)D * 8 * 2 + (size_t)D * 2 * 5 + (size_t)D * 2 + 16 + 15) & ~(size_t)15;
}

struct K7Shared {
    double* rowkey;     // [n] best live key of row a
    double* intra;      // [n] level 1: _mean_intra_pt cache; level 2: mean_pc
    int16_t* rowarg;    // [n] its partner b (-1: row empty)
    int16_t* cnt;       // [n] members of the group in slot a (0: dead slot)
    uint8_t* has;       // [n] intra cache valid (bit0) / singleton (bit1)
    uint8_t* need;      // [n] row minimum must be rescanned
};

struct K7Global {
    double* key;        // [n*n] pair keys, row a < column b
    uint8_t* live;      // [n*n] pair still in the heap
    uint16_t* mem;      // [n*n] members (device ranks) of slot a at mem[a*n ..]
    uint16_t* tmp;      // [n]   merge buffer
};

__device__ __forceinline__ bool k7_less(double k1, int a1, int b1, double k2, int a2, int b2) {
    if (k1 != k2) return k1 < k2;
    if (a1 != a2) return a1 < a2;
    return b1 < b2;
}

// pair key of slots x < y (level 1: group_pair_metric; level 2:
// _relative_spread of the two mean p_c)
__device__ double k7_pair_key(int level, const K7Global& g, const K7Shared& sh, int n,
                              const double* __restrict__ pt, int D, int x, int y) {
    if (level == 2) {
        const double va = sh.intra[x], vb = sh.intra[y];
        const double top = va >= vb ? va : vb, bot = va <= vb ? va : vb;
        if (top == 0) return 0.0;
        return (top - bot) / top;
    }
    const uint16_t* mx = g.mem + (size_t)x * n;
    const uint16_t* my = g.mem + (size_t)y * n;
    const int nx = sh.cnt[x], ny = sh.cnt[y];
    NeumaierSum s;
    bool first = true;
    for (int i = 0; i < nx; ++i) {
        const double* row = pt + (size_t)mx[i] * D;
        for (int j = 0; j < ny; ++j) {
            const double v = row[my[j]];
            if (first) { s.start(v); first = false; } else s.add(v);
        }
    }
    return s.value() / (double)((long long)nx * ny);
}

// _mean_intra_pt of slot a (level 1) or mean p_c (level 2), one thread
__device__ void k7_group_value(int level, const K7Global& g, const K7Shared& sh, int n,
                               const double* __restrict__ pt, const double* __restrict__ pc, int D,
                               int a) {
    const uint16_t* m = g.mem + (size_t)a * n;
    const int c = sh.cnt[a];
    if (level == 2) {
        NeumaierSum s;
        s.start(pc[m[0]]);
        for (int i = 1; i < c; ++i) s.add(pc[m[i]]);
        sh.intra[a] = s.value() / (double)c;
        sh.has[a] = 1;
        return;
    }
    if (c < 2) { sh.has[a] = 2; return; }
    NeumaierSum s;
    bool first = true;
    for (int i = 0; i < c; ++i)
        for (int j = i + 1; j < c; ++j) {
            const double v = pt[(size_t)m[i] * D + m[j]];
            if (first) { s.start(v); first = false; } else s.add(v);
        }
    sh.intra[a] = s.value() / (double)((long long)c * (c - 1) / 2);
    sh.has[a] = 1;
}

// full rescan of row a by one thread
__device__ __forceinline__ void k7_scan_row(const K7Global& g, const K7Shared& sh, int n, int a) {
    double bk = 0.0;
    int bb = -1;
    const double* kr = g.key + (size_t)a * n;
    const uint8_t* lr = g.live + (size_t)a * n;
    for (int b = a + 1; b < n; ++b)
        if (lr[b] && sh.cnt[b] && (bb < 0 || kr[b] < bk)) { bk = kr[b]; bb = b; }
    sh.rowkey[a] = bk;
    sh.rowarg[a] = (int16_t)bb;
}

// the same rescan by one warp: lanes take every 32nd column, then a warp
// arg-min on (key, column) - the first minimal column, as the serial scan
__device__ __forceinline__ void k7_scan_row_warp(const K7Global& g, const K7Shared& sh, int n,
                                                 int a, int lane) {
    double bk = 0.0;
    int bb = -1;
    const double* kr = g.key + (size_t)a * n;
    const uint8_t* lr = g.live + (size_t)a * n;
    for (int b = a + 1 + lane; b < n; b += 32)
        if (lr[b] && sh.cnt[b] && (bb < 0 || kr[b] < bk)) { bk = kr[b]; bb = b; }
    for (int o = 16; o; o >>= 1) {
        const double k2 = __shfl_down_sync(0xffffffffu, bk, o);
        const int b2 = __shfl_down_sync(0xffffffffu, bb, o);
        if (b2 >= 0 && (bb < 0 || k2 < bk || (k2 == bk && b2 < bb))) { bk = k2; bb = b2; }
    }
    if (lane == 0) {
        sh.rowkey[a] = bk;
        sh.rowarg[a] = (int16_t)bb;
    }
}

// rows flagged in sh.need, one warp per row (WARP: the calling warp alone)
template <bool WARP>
__device__ __forceinline__ void k7_rescan_flagged(const K7Global& g, const K7Shared& sh, int n) {
    const int lane = threadIdx.x & 31, wid = WARP ? 0 : threadIdx.x >> 5,
              nw = WARP ? 1 : blockDim.x >> 5;
    for (int r = wid; r < n; r += nw)
        if (sh.need[r]) k7_scan_row_warp(g, sh, n, r, lane);
}

// CTA arg-min over the row minima: returns (a, b) in s_ab, or a = -1
// (WARP: the calling warp alone, warp-synchronous)
template <bool WARP>
__device__ void k7_pop(const K7Shared& sh, int n, int* s_ab, double* s_red, int* s_ia) {
    if (!WARP && n <= 128) {  // warp 0 alone (<= 4 rows per lane), one barrier
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            double bk = 0.0;
            int ba = -1, bb = -1;
            for (int a = lane; a < n; a += 32) {
                const int b = sh.rowarg[a];
                if (sh.cnt[a] == 0 || b < 0) continue;
                const double k = sh.rowkey[a];
                if (ba < 0 || k7_less(k, a, b, bk, ba, bb)) { bk = k; ba = a; bb = b; }
            }
            for (int o = 16; o; o >>= 1) {
                const double k2 = __shfl_down_sync(0xffffffffu, bk, o);
                const int a2 = __shfl_down_sync(0xffffffffu, ba, o);
                const int b2 = __shfl_down_sync(0xffffffffu, bb, o);
                if (a2 >= 0 && (ba < 0 || k7_less(k2, a2, b2, bk, ba, bb))) { bk = k2; ba = a2; bb = b2; }
            }
            if (lane == 0) { s_ab[0] = ba; s_ab[1] = bb; }
        }
        __syncthreads();
        return;
    }
    const int tid = WARP ? (threadIdx.x & 31) : threadIdx.x, lane = threadIdx.x & 31,
              wid = threadIdx.x >> 5;
    const int nt = WARP ? 32 : blockDim.x;
    double bk = 0.0;
    int ba = -1, bb = -1;
    for (int a = tid; a < n; a += nt) {
        const int b = sh.rowarg[a];
        if (sh.cnt[a] == 0 || b < 0) continue;
        const double k = sh.rowkey[a];
        if (ba < 0 || k7_less(k, a, b, bk, ba, bb)) { bk = k; ba = a; bb = b; }
    }
    for (int o = 16; o; o >>= 1) {
        const double k2 = __shfl_down_sync(0xffffffffu, bk, o);
        const int a2 = __shfl_down_sync(0xffffffffu, ba, o);
        const int b2 = __shfl_down_sync(0xffffffffu, bb, o);
        if (a2 >= 0 && (ba < 0 || k7_less(k2, a2, b2, bk, ba, bb))) { bk = k2; ba = a2; bb = b2; }
    }
    if (WARP) {
        if (lane == 0) { s_ab[0] = ba; s_ab[1] = bb; }
        __syncwarp();
        return;
    }
    if (lane == 0) { s_red[wid] = bk; s_ia[2 * wid] = ba; s_ia[2 * wid + 1] = bb; }
    __syncthreads();
    if (tid == 0) {
        double k = 0.0;
        int a = -1, b = -1;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            const int a2 = s_ia[2 * w], b2 = s_ia[2 * w + 1];
            if (a2 >= 0 && (a < 0 || k7_less(s_red[w], a2, b2, k, a, b))) { k = s_red[w]; a = a2; b = b2; }
        }
        s_ab[0] = a;
        s_ab[1] = b;
    }
    __syncthreads();
}

// _agglomerate over n items (device ranks items[i], sorted): on return
// group_of[i] = index of the item's group in sorted(alive) order; returns
// the number of groups.  All threads of the CTA call it.
template <bool WARP>
__device__ int k7_agglomerate(int level, int n, const uint16_t* items, const double* __restrict__ pt,
                              const double* __restrict__ pc, int D, double thr, const K7Global& g,
                              const K7Shared& sh, uint16_t* group_of, int* s_ab, double* s_red,
                              int* s_ia) {
    // WARP: one warp runs the whole merge chain with warp barriers (small
    // groups: the chain is barrier-latency bound)
    const int tid = WARP ? (threadIdx.x & 31) : threadIdx.x, nt = WARP ? 32 : blockDim.x;
    auto sync = [] { if (WARP) __syncwarp(); else __syncthreads(); };
    for (int a = tid; a < n; a += nt) {
        sh.cnt[a] = 1;
        g.mem[(size_t)a * n] = items[a];
        sh.has[a] = 0;
    }
    sync();
    if (level == 2)
        for (int a = tid; a < n; a += nt) k7_group_value(2, g, sh, n, pt, pc, D, a);
    sync();
    for (long long p = tid; p < (long long)n * n; p += nt) {
        const int a = (int)(p / n), b = (int)(p % n);
        if (b > a) {
            g.key[p] = k7_pair_key(level, g, sh, n, pt, D, a, b);
            g.live[p] = 1;
        }
    }
    for (int a = tid; a < n; a += nt) sh.need[a] = 1;
    sync();
    k7_rescan_flagged<WARP>(g, sh, n);
    sync();
#if defined(K7_PROFILE)
    long long c_pop = 0, c_pred = 0, c_keys = 0, c_rows = 0, c0, c1;
    int npops = 0;
#endif
    for (;;) {
#if defined(K7_PROFILE)
        c0 = clock64();
#endif
        k7_pop<WARP>(sh, n, s_ab, s_red, s_ia);
        const int a = s_ab[0], b = s_ab[1];
#if defined(K7_PROFILE)
        c1 = clock64(); c_pop += c1 - c0; c0 = c1; ++npops;
#endif
        if (a < 0) break;
        // merge predicate (merge_values + _relative_spread, :154-180, :203-210)
        if (tid == 0) {
            double v0, v1, v2 = 0.0;
            int nv;
            if (level == 1) {
                const double cross = g.key[(size_t)a * n + b];
                if (!sh.has[a]) k7_group_value(1, g, sh, n, pt, pc, D, a);
                if (!sh.has[b]) k7_group_value(1, g, sh, n, pt, pc, D, b);
                v0 = (sh.has[a] & 1) ? sh.intra[a] : cross;
                v1 = (sh.has[b] & 1) ? sh.intra[b] : cross;
                v2 = cross;
                nv = 3;
            } else {
                v0 = sh.intra[a];
                v1 = sh.intra[b];
                nv = 2;
            }
            double top = v0, bot = v0;
            if (v1 > top) top = v1;
            if (v1 < bot) bot = v1;
            if (nv == 3) { if (v2 > top) top = v2; if (v2 < bot) bot = v2; }
            const double spread = top == 0 ? 0.0 : (top - bot) / top;
            if (spread >= thr) {
                g.live[(size_t)a * n + b] = 0;  // discarded permanently
                s_ab[2] = 0;
            } else {
                s_ab[2] = 1;
            }
        }
        sync();
        if (s_ab[2]) {
            // merged = tuple(sorted(a + b)) into slot a: member lists are
            // sorted and disjoint, so an element's place is its index plus
            // the number of the other list's members below it (binary search)
            const uint16_t* ma = g.mem + (size_t)a * n;
            const uint16_t* mb = g.mem + (size_t)b * n;
            const int na = sh.cnt[a], nb = sh.cnt[b];
            uint16_t v = 0;
            int pos = -1;
            for (int t = tid; t < na + nb; t += nt) {  // na + nb <= n <= nt in practice
                const bool in_a = t < na;
                v = in_a ? ma[t] : mb[t - na];
                const uint16_t* other = in_a ? mb : ma;
                int lo = 0, hi = in_a ? nb : na;  // first index with other[idx] > v
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (other[mid] < v) lo = mid + 1; else hi = mid;
                }
                pos = (in_a ? t : t - na) + lo;
                g.tmp[pos] = v;
            }
            sync();
            for (int t = tid; t < na + nb; t += nt) g.mem[(size_t)a * n + t] = g.tmp[t];
            if (tid == 0) {
                sh.cnt[a] = (int16_t)(na + nb);
                sh.cnt[b] = 0;
                g.live[(size_t)a * n + b] = 0;
                sh.has[a] = 0;
            }
            sync();
            (void)pos;
        }
#if defined(K7_PROFILE)
        c1 = clock64(); c_pred += c1 - c0; c0 = c1;
#endif
        if (!s_ab[2]) {  // discarded: row a loses its minimum
            if (tid < 32) k7_scan_row_warp(g, sh, n, a, tid & 31);
            sync();
            continue;
        }
        if (level == 2 && tid == 0) k7_group_value(2, g, sh, n, pt, pc, D, a);
        sync();
        // pairs of the merged group with every other live group; drop b's
        for (int c = tid; c < n; c += nt) {
            if (c == a || sh.cnt[c] == 0) continue;
            const int x = c < a ? c : a, y = c < a ? a : c;
            g.key[(size_t)x * n + y] = k7_pair_key(level, g, sh, n, pt, D, x, y);
            g.live[(size_t)x * n + y] = 1;
            if (c < b) g.live[(size_t)c * n + b] = 0;
        }
        // the merged group's _mean_intra_pt, on an otherwise idle thread
#if !defined(K7_LAZY_INTRA)
        if (level == 1 && n < nt && tid == nt - 1) k7_group_value(1, g, sh, n, pt, pc, D, a);
#endif
        sync();
#if defined(K7_PROFILE)
        c1 = clock64(); c_keys += c1 - c0; c0 = c1;
#endif
        // row minima: rows that pointed at a or b rescan; rows c < a compare
        // against their new pair (c, a); row a rescans
        for (int c = tid; c < n; c += nt) {
            sh.need[c] = 0;
            if (sh.cnt[c] == 0) continue;
            const int r = sh.rowarg[c];
            if (c == a || r == a || r == b) {
                sh.need[c] = 1;
            } else if (c < a) {
                const double k = g.key[(size_t)c * n + a];
                if (r < 0 || k7_less(k, c, a, sh.rowkey[c], c, r)) {
                    sh.rowkey[c] = k;
                    sh.rowarg[c] = (int16_t)a;
                }
            }
        }
        sync();
        k7_rescan_flagged<WARP>(g, sh, n);
        sync();
#if defined(K7_PROFILE)
        c1 = clock64(); c_rows += c1 - c0;
#endif
    }
#if defined(K7_PROFILE)
    if (tid == 0 && blockIdx.x == 0)
        printf("  level %d n %d pops %d: pop %lld pred %lld keys %lld rows %lld cycles\n", level, n, npops,
               c_pop, c_pred, c_keys, c_rows);
#endif
    // sorted(alive): slot order; group index = rank among live slots
    if (tid == 0) {
        int gi = 0;
        for (int a = 0; a < n; ++a) {
            if (sh.cnt[a] == 0) continue;
            const uint16_t* m = g.mem + (size_t)a * n;
            for (int q = 0; q < sh.cnt[a]; ++q) {
                // members are device ranks; map back to local item index
                int lo = 0, hi = n - 1;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (items[mid] < m[q]) lo = mid + 1; else hi = mid;
                }
                group_of[lo] = (uint16_t)gi;
            }
            ++gi;
        }
        s_ab[3] = gi;
    }
    sync();
    return s_ab[3];
}

// One CTA per snapshot.  Outputs (stride D per snapshot): fg_of, sg_of,
// fg_intra / fg_cap / fg_minbw per FG, sg_cap per SG (FG-major); n_fg, n_sg.
// SM = smem_mode as a template parameter, so that with the tables in shared
// memory every table access compiles to a shared-memory load (LDS) rather
// than a generic one
template <int SM>
__global__ void __launch_bounds__(K7_THREADS)
k7_group(int D, const double* __restrict__ pt_all, const double* __restrict__ bw_all,
         long long pt_stride, long long bw_stride, const double* __restrict__ pc, double thr_net,
         double thr_comp, uint8_t* __restrict__ scratch, size_t scratch_per, int smem_mode,
         const uint16_t* __restrict__ fixed_fg, int fixed_nf, uint16_t* fg_of_all,
         uint16_t* sg_of_all, uint32_t* n_fg, uint32_t* n_sg, double* fg_intra_all,
         double* fg_cap_all, double* fg_minbw_all, double* sg_cap_all, int phase,
         uint32_t* nsg_f_all, double* sg_stage_all) {
    // phase 0: one CTA per snapshot runs both levels (the FGs' second levels
    // one after another); phase 1: first level only (fg_of, n_fg); phase 2:
    // CTA (snapshot, f) runs FG f's statistics and second level, its SG
    // capacities staged at the FG's first member slot (k7_sg_finish packs
    // them).  Phases 1 + 2 need the pair tables in shared memory.
    extern __shared__ __align__(16) uint8_t k7_smem[];
    __shared__ int s_ab[4];
    __shared__ double s_red[K7_THREADS / 32];
    __shared__ int s_ia[2 * (K7_THREADS / 32)];
    const int snap = phase == 2 ? (int)(blockIdx.x / (unsigned)D) : (int)blockIdx.x, tid = threadIdx.x;
    const int f_only = phase == 2 ? (int)(blockIdx.x % (unsigned)D) : -1;
    if (phase == 2 && f_only >= (int)n_fg[snap]) return;
    const double* pt = pt_all + (size_t)snap * pt_stride;
    const double* bw = bw_all ? bw_all + (size_t)snap * bw_stride : nullptr;
    // smem_mode bit0: pair tables in shared memory (small D); bit1: p_t too
    (void)smem_mode;
    uint8_t* base = (SM & 1) ? k7_smem + k7_smem_head(D) : scratch + (size_t)snap * scratch_per;
    if constexpr ((SM & 2) != 0) {
        double* pts = reinterpret_cast<double*>(base + k7_scratch_bytes(D));
        for (int e = tid; e < D * D; e += blockDim.x) pts[e] = pt[e];
        pt = pts;  // visible after the first __syncthreads below
    }
    K7Global g;
    g.key = reinterpret_cast<double*>(base);
    g.mem = reinterpret_cast<uint16_t*>(base + (size_t)D * D * 8);
    g.tmp = g.mem + (size_t)D * D;
    g.live = reinterpret_cast<uint8_t*>(g.tmp + D);
    K7Shared sh;
    sh.rowkey = reinterpret_cast<double*>(k7_smem);
    sh.intra = sh.rowkey + D;
    sh.rowarg = reinterpret_cast<int16_t*>(sh.intra + D);
    sh.cnt = sh.rowarg + D;
    uint16_t* items = reinterpret_cast<uint16_t*>(sh.cnt + D);
    uint16_t* gof = items + D;          // level-1 group of each device
    uint16_t* sgo = gof + D;            // level-2 group of each FG member
    sh.has = reinterpret_cast<uint8_t*>(sgo + D);
    sh.need = sh.has + D;
    uint16_t* fg_of = fg_of_all + (size_t)snap * D;
    uint16_t* sg_of = sg_of_all + (size_t)snap * D;
    double* fg_intra = fg_intra_all + (size_t)snap * D;
    double* fg_cap = fg_cap_all + (size_t)snap * D;
    double* fg_minbw = fg_minbw_all + (size_t)snap * D;
    double* sg_cap = sg_cap_all + (size_t)snap * D;

    for (int d = tid; d < D; d += blockDim.x) items[d] = (uint16_t)d;
    __syncthreads();
#if defined(K7_PROFILE)
    unsigned long long tp0, tp1, tp2;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp0));
#endif
    // first level: agglomerated, or given (a fixed partition, e.g. the C2
    // region-grouping sweep; indices already in sorted-member-tuple order)
    int nf;
    if (phase == 2) {
        for (int d = tid; d < D; d += blockDim.x) gof[d] = fg_of[d];
        __syncthreads();
        nf = (int)n_fg[snap];
    } else if (fixed_fg) {
        for (int d = tid; d < D; d += blockDim.x) gof[d] = fixed_fg[d];
        __syncthreads();
        nf = fixed_nf;
    } else {
        nf = k7_agglomerate<false>(1, D, items, pt, pc, D, thr_net, g, sh, gof, s_ab, s_red, s_ia);
    }
    if (phase != 2)
        for (int d = tid; d < D; d += blockDim.x) fg_of[d] = gof[d];
    __syncthreads();
    if (phase == 1) {
        if (tid == 0) n_fg[snap] = (uint32_t)nf;
        return;
    }
#if defined(K7_PROFILE)
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp1));
#endif
    int sg_base = 0;
    for (int f = f_only < 0 ? 0 : f_only; f < (f_only < 0 ? nf : f_only + 1); ++f) {
        // members of FG f in rank order
        if (tid == 0) {
            int k = 0, before = 0;
            for (int d = 0; d < D; ++d) {
                if (gof[d] == f) items[k++] = (uint16_t)d;
                before += gof[d] < f;
            }
            s_ab[0] = k;
            if (f_only >= 0) sg_base = before;  // staging slot: FG f's first member
        }
        __syncthreads();
        const int nm = s_ab[0];
        __syncthreads();
        // FG statistics (group_first_level, :176-188): the sums on one thread
        // (operand order), min_intra_bandwidth as a CTA min (order-free)
        if (tid == 0) {
            NeumaierSum s;
            s.start(pc[items[0]]);
            for (int i = 1; i < nm; ++i) s.add(pc[items[i]]);
            fg_cap[f] = s.value();
            if (nm < 2) {
                fg_intra[f] = NAN;
            } else {
                NeumaierSum t;
                bool first = true;
                for (int i = 0; i < nm; ++i)
                    for (int j = i + 1; j < nm; ++j) {
                        const double v = pt[(size_t)items[i] * D + items[j]];
                        if (first) { t.start(v); first = false; } else t.add(v);
                    }
                fg_intra[f] = t.value() / (double)((long long)nm * (nm - 1) / 2);
            }
        }
        {
            double mb = INFINITY;
            if (bw)
                for (int q = tid; q < nm * nm; q += blockDim.x) {
                    const int i = q / nm, j = q % nm;
                    if (j > i) {
                        const double v = bw[(size_t)items[i] * D + items[j]];
                        mb = v < mb ? v : mb;
                    }
                }
            for (int o = 16; o; o >>= 1) {
                const double v = __shfl_down_sync(0xffffffffu, mb, o);
                mb = v < mb ? v : mb;
            }
            if ((tid & 31) == 0) s_red[tid >> 5] = mb;
            __syncthreads();
            if (tid == 0) {
                double r = s_red[0];
                for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = s_red[w] < r ? s_red[w] : r;
                fg_minbw[f] = (nm < 2 || !bw) ? NAN : r;
            }
            __syncthreads();
        }
        // second level over the FG's members (local slots 0..nm-1)
        // (a one-warp variant, k7_agglomerate<true>, measured slower here: the
        // chain is bound by dependent shared-memory steps, not by barriers)
        const int ns = k7_agglomerate<false>(2, nm, items, pt, pc, D, thr_comp, g, sh, sgo, s_ab,
                                             s_red, s_ia);
        for (int i = tid; i < nm; i += blockDim.x) sg_of[items[i]] = sgo[i];
        __syncthreads();
        if (tid == 0) {
            for (int q = 0; q < ns; ++q) {
                NeumaierSum s;
                bool first = true;
                for (int i = 0; i < nm; ++i)
                    if (sgo[i] == q) {
                        const double v = pc[items[i]];
                        if (first) { s.start(v); first = false; } else s.add(v);
                    }
                if (f_only >= 0) sg_stage_all[(size_t)snap * D + sg_base + q] = s.value();
                else sg_cap[sg_base + q] = s.value();
            }
            if (f_only >= 0) nsg_f_all[(size_t)snap * D + f] = (uint32_t)ns;
        }
        sg_base += ns;
        __syncthreads();
    }
    if (f_only >= 0) return;
    if (tid == 0) {
        n_fg[snap] = (uint32_t)nf;
        n_sg[snap] = (uint32_t)sg_base;
    }
#if defined(K7_PROFILE)
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp2));
    if (tid == 0 && snap == 0) printf("K7 level1 %llu ns, level2+stats %llu ns\n", tp1 - tp0, tp2 - tp1);
#endif
}

// After phase 2: per snapshot, SG capacities in FG order (sg_base = running
// count of SGs) and n_sg.  One thread per snapshot (<= D FGs).
__global__ void k7_sg_finish(int D, int n_snap, const uint32_t* __restrict__ n_fg,
                             const uint16_t* __restrict__ fg_of_all,
                             const uint32_t* __restrict__ nsg_f_all,
                             const double* __restrict__ sg_stage_all, double* sg_cap_all,
                             uint32_t* n_sg) {
    const int snap = blockIdx.x * blockDim.x + threadIdx.x;
    if (snap >= n_snap) return;
    const uint16_t* fg_of = fg_of_all + (size_t)snap * D;
    const uint32_t* nsg = nsg_f_all + (size_t)snap * D;
    const double* st = sg_stage_all + (size_t)snap * D;
    double* out = sg_cap_all + (size_t)snap * D;
    const int nf = (int)n_fg[snap];
    int base = 0, first = 0;  // first: member slots of the FGs before f
    for (int f = 0; f < nf; ++f) {
        int cnt = 0;
        for (int d = 0; d < D; ++d) cnt += fg_of[d] == f;
        for (int q = 0; q < (int)nsg[f]; ++q) out[base + q] = st[first + q];
        base += (int)nsg[f];
        first += cnt;
    }
    n_sg[snap] = (uint32_t)base;
}
