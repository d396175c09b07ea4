// engine.cu - B200 (sm_100a) plan-evaluation engine behind the C-ABI of
// include/geopipe_b200.h: the context (device buffers, streams, CUDA graph)
// and every extern "C" entry point.  Kernels live in the headers:
//   common.cuh        DevInst, arg-min keys/reductions, TMA + mbarrier helpers
//   k1_tables.cuh     K1 table build          k2_eval.cuh   K2 explicit batches
//   k3_argmin.cuh     K3 exhaustive arg-min   detail.cuh    winner plan detail
//   k4_bnb.cuh        K4 branch-and-bound     k5_sim.cuh    K5 1F1B simulation
//   k6_snapshots.cuh  K6 bandwidth snapshots
//
// Data path:
//   gp_ctx_load    H2D of the packed instance, then K1:
//                    k1_intervals  Neumaier interval sums S[col][a][b]
//                    k1_groups     per-group TP tiles, DP fractions, memory minima
//                    k1_stages     per (group, a, b): split choice, memory
//                                  feasibility, capacity, C1 = (F+Bi)+W, and per m
//                                  the table {C1*m | +inf, AL}
//                    k1_boundary   gateway pair per ordered group pair and
//                                  x = lat + (act*m)/bw per boundary layer
//   gp_eval_batch  K2: one thread per explicit candidate
//   gp_argmin_range K3: one CTA per (b,m, order, comp-chunk); the varying last
//                  cut sweeps a shared-memory triangle of the stage table;
//                  warp-shuffle + CTA + last-block argmin on the reference key
//
// Every floating-point operation mirrors the reference operation order
// (src/costmodel.py:56-89, src/timing.py:116-231, src/planner.py:157-253);
// the file is compiled with -fmad=false.  There is no CPU fallback.
#include <mutex>
#include <atomic>
#include <chrono>

#include "common.cuh"
#include "k1_tables.cuh"
#include "k2_eval.cuh"
#include "k3_argmin.cuh"
#include "k3_sweep_rec.cuh"
#include "detail.cuh"
#include "k4_bnb.cuh"
#include "k6_snapshots.cuh"
#include "k5_sim.cuh"
#include "k7_grouping.cuh"
#include "k8_validate.cuh"
#include "verify.h"

// ----------------------------------------------------------------------------
// context
// ----------------------------------------------------------------------------
// bumped on every device (re)allocation: a captured CUDA graph is only
// replayed while the buffers it was captured with are still in place
static unsigned long long g_alloc_gen = 0;

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t count) {
        if (count <= cap && p) return cudaSuccess;
        __atomic_add_fetch(&g_alloc_gen, 1ull, __ATOMIC_RELAXED);
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t c = count ? count : 1;
        cudaError_t e = cudaMalloc(&p, c * sizeof(T));
        if (e == cudaSuccess) cap = c;
        return e;
    }
    void release() { if (p) cudaFree(p); p = nullptr; cap = 0; }
};

template <typename T>
struct ArenaPtr {
    T* p = nullptr;
    void release() { p = nullptr; }
};

struct gp_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool loaded = false;
    uint32_t flags = 0;
    int n = 0, F = 0, D = 0, nb = 0, nm = 0, nsg = 0;
    std::vector<long long> h_batch, h_micro;
    // raw instance arrays live in the arena (one allocation, one H2D copy)
    ArenaPtr<double> fwd, bwd_in, bwd_w, act, param, p_c, mem, p_t, lat, bw, fg_cap, sg_cap,
        fg_minbw, fg_minbw_in;
    ArenaPtr<long long> batch, micro;
    ArenaPtr<uint32_t> id_rank, fg_off, fg_mem, fg_sg_off, sg_off, sg_mem;
    ArenaPtr<uint8_t> fg_has;
    // derived tables
    DBuf<double> S, g_rf, g_cf, g_dp, g_minmem, sg_minmem, C1, xt;
    DBuf<double4> fbws;
    DBuf<double> vtab;
    DBuf<double> mtab;           // micro-batch counts M per (b, m) index
    DBuf<double2> tpk, tcol;
    DBuf<uint32_t> flagsbuf;
    DBuf<uint8_t> g_tp_ok, scode, skind;
    DBuf<K1Grp> kgrp;
    DBuf<uint8_t> sshare0, gwbad;
    DBuf<double2> stg;
    DBuf<int> gw;
    // K3 scratch
    DBuf<Key> blk, result;
    DBuf<unsigned int> counter;
    DBuf<Key> bam_blk;              // gp_argmin_batch_device: per-CTA keys
    DBuf<unsigned int> bam_ctr;     //   and its CTA counter (re-armed by the last CTA)
    DBuf<unsigned long long> err_idx;
    DBuf<int> err_dummy;
    // K2 staging
    DBuf<uint8_t> b_order, b_counts, b_bm, b_status;
    DBuf<double> b_cost;
    DBuf<gp_plan_info> info;
    DBuf<gp_group_info> ginfo;
    DBuf<int> dstatus;
    DBuf<SolveOut> dsolve;
    DBuf<unsigned long long> gbest;  // K4 shared incumbent
    DBuf<gp_timing> s_tim;       // K5 staging
    DBuf<gp_trace> s_traces;
    DBuf<uint32_t> s_tidx;
    // K6 snapshot batch buffers
    DBuf<double> z_bw, z_mbw, z_xt;
    DBuf<uint32_t> z_flags;
    DBuf<double2> z_tpk, z_tcol;
    DBuf<Key> z_res;
    DBuf<unsigned int> z_cnt;
    DBuf<double> s_ms;
    DBuf<uint8_t> s_st;
    DBuf<gp_sim_report> s_rep;  // K5 full reports
    DBuf<double> s_ends;
    DBuf<uint32_t> s_wq;         // K5 full queue scratch
    DBuf<uint8_t> g_buf;         // K7 inputs, outputs and scratch
    uint8_t* h_stage = nullptr;  // pinned host staging (K7: one H2D, one D2H per batch)
    size_t h_stage_cap = 0;
    DBuf<unsigned long long> s_lq;
    SolveOut* h_solve = nullptr;  // pinned, mapped (the gp_replan graph's detail kernel writes it)
    SolveOut* d_hsolve = nullptr; // device alias of h_solve
    DBuf<unsigned long long> d_seq;        // completed gp_replan graphs (device count)
    unsigned long long solve_seq = 0;      // launched gp_replan graphs (host count)
    RangeGeom last_geom{};
    bool last_generic = false;
    unsigned long long last_lo = 0, last_hi = 0;
    int smem_max = 0;
    int n_sms = 148;
    uint32_t* h_flags = nullptr;      // pinned
    cudaEvent_t flags_ev = nullptr;
    cudaEvent_t arena_ev = nullptr;
    bool flags_known = false;
    // raw instance arena: one pinned staging buffer -> one H2D copy
    unsigned char* h_arena = nullptr;   // pinned, mapped
    const unsigned char* d_harena = nullptr;  // device alias (k_arena_pull reads it)
    size_t h_arena_cap = 0;
    DBuf<unsigned char> arena;
    int cache_n = -1, cache_k = -1;   // (n, k) of the enumeration helpers
    // gp_replan: CUDA graph of H2D + K1 + K3 + detail + D2H for one shape
    cudaGraphExec_t graph_exec = nullptr;
    unsigned long long graph_key[11] = {0};
    // shape key of the instance the context tables currently hold (set by
    // gp_ctx_load and gp_replan): the graph replays only while it equals
    // graph_key, i.e. no load of another shape came in between
    unsigned long long loaded_key[11] = {0};
    unsigned long long graph_gen = 0;
    RangeGeom graph_geom{};
    unsigned long long graph_lo = 0, graph_hi = 0;
    bool capturing = false;
    bool pdl = false;  // capturing the gp_replan graph: PDL launches, no memset nodes
    bool diag_timing = false;          // gp_diag_replan_timing
    cudaEvent_t t_ev0 = nullptr, t_ev1 = nullptr;
    float last_graph_ms = -1.0f;
    double host_us[4] = {0, 0, 0, 0};  // gp_replan: arena fill, launch, wait, finish
    size_t arena_bytes = 0;
    size_t bw_off = 0;  // offset of the loaded bandwidth matrix in the arena
    int force_mode = -1;  // -1 auto; 0/1/2 fast-path variant; 3 generic kernel
    // parity tests: every K3 / K6 launch uses the VER instantiation and
    // stores each candidate's cost into vbuf (gp_diag_verify_begin / _end)
    bool verify = false;
    VerifySink vs;
    DBuf<double> vbuf;
    // gp_diag_kernel_timing: CUDA events around every exhaustive sweep launch
    bool ktime = false;
    std::vector<cudaEvent_t> kt_ev;  // pairs (start, end), reused across windows
    size_t kt_used = 0;
    // device state known from earlier launches on the stream (memsets skipped):
    // item counters [0, ctr_armed) are zero (k3_sweep re-arms the ones it
    // used); err_idx holds ~0 (no launch since its reset could have written it)
    size_t ctr_armed = 0;
    bool err_clean = false;
    std::vector<uint32_t> h_fg_sg_count;  // subgroups per group (explicit plans)
    DBuf<unsigned long long> binom;
    DBuf<unsigned int> item_ctr;
    DBuf<uint8_t> tiles;
    bool tiles_ok = false;
    DBuf<uint4> groups;       // K3 sweep run groups
    DBuf<uint8_t> prefixes;   // colex (k-3)-subsets for the sweep
    DBuf<unsigned long long> bnk;  // binomial sub-table [n+1][k+1] (TMA-staged)
    int ngroups = 0;  // uint4 slots of `groups`: the run groups, then the task table
    int ng = 0;       // run groups
    unsigned int sweep_W = 0;
    bool sweep_ok = false;
    DBuf<K3Run> recruns;      // record sweep run table (k3_sweep_rec)
    unsigned int rec_W = 0;
    bool rec_ok = false;
    DBuf<uint32_t> recrow;    // record sweep padded row starts
    DBuf<uint8_t> k2img;      // K2: shared-memory image of the current tables
    unsigned long long tables_gen = 1, k2img_gen = 0;  // table builds / image's build
    DBuf<uint32_t> k5_perm;   // K5: candidates grouped by (b, m) index
    DBuf<uint32_t> k5_hist;

    DevInst view() {
        DevInst I;
        I.n = n; I.F = F; I.D = D; I.nb = nb; I.nm = nm;
        I.fwd = fwd.p; I.bwd_in = bwd_in.p; I.bwd_w = bwd_w.p; I.act = act.p; I.param = param.p;
        I.batch = batch.p; I.micro = micro.p; I.mtab = mtab.p;
        I.p_c = p_c.p; I.mem = mem.p; I.p_t = p_t.p; I.lat = lat.p; I.bw = bw.p;
        I.id_rank = id_rank.p;
        I.fg_off = fg_off.p; I.fg_mem = fg_mem.p; I.fg_sg_off = fg_sg_off.p;
        I.sg_off = sg_off.p; I.sg_mem = sg_mem.p;
        I.fg_cap = fg_cap.p; I.sg_cap = sg_cap.p;
        I.fg_minbw = fg_minbw.p; I.fg_has_minbw = fg_has.p;
        I.bf = bf;
        I.grp = kgrp.p; I.sshare0 = sshare0.p; I.gwbad = gwbad.p;
        I.S = S.p; I.g_tp_ok = g_tp_ok.p; I.g_rf = g_rf.p; I.g_cf = g_cf.p; I.g_dp = g_dp.p;
        I.g_minmem = g_minmem.p; I.sg_minmem = sg_minmem.p;
        I.stg = stg.p; I.scode = scode.p; I.skind = skind.p; I.C1 = C1.p; I.fbws = fbws.p; I.vtab = vtab.p;
        I.gw = gw.p; I.xt = xt.p; I.flags = flagsbuf.p;
        I.nxp = (n + 1) & ~1;
        I.tpk = tpk.p; I.tcol = tcol.p;
        return I;
    }
    double bf = 1.25;
};

template <typename T>
static cudaError_t upload(cudaStream_t s, DBuf<T>& d, const T* h, size_t count) {
    cudaError_t e = d.ensure(count);
    if (e != cudaSuccess) return e;
    if (count == 0) return cudaSuccess;
    return cudaMemcpyAsync(d.p, h, count * sizeof(T), cudaMemcpyHostToDevice, s);
}

// C(n, r), saturating at UINT64_MAX (exact whenever the true value fits)
static unsigned long long h_binom(int n, int r) {
    if (r < 0 || r > n) return 0ull;
    unsigned __int128 res = 1;
    for (int i = 1; i <= r; ++i) {
        res = res * (unsigned __int128)(n - r + i) / (unsigned __int128)i;
        if (res > (unsigned __int128)~0ull) return ~0ull;
    }
    return (unsigned long long)res;
}

// Kernel launch with programmatic stream serialisation (PDL) when `pdl`:
// the kernel may be scheduled while its predecessor drains and waits in
// pdl_wait() for the predecessor's results.
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                            cudaStream_t s, bool pdl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(block, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

extern "C" {

const char* gp_version(void) { return "geopipe_b200 0.1 (sm_100a)"; }
const char* gp_last_error(void) { return g_err; }

int gp_ctx_create(int device, gp_ctx** out) {
    if (!out) return fail(GP_ERR_INPUT, "null output pointer");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(GP_ERR_CUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
    if (device < 0 || device >= count) return fail(GP_ERR_INPUT, "device %d out of range", device);
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(GP_ERR_CUDA, "device %d is sm_%d%d; this engine is built for sm_100a",
                    device, prop.major, prop.minor);
    CUDA_TRY(cudaSetDevice(device));
    gp_ctx* c = new gp_ctx();
    c->device = device;
    c->smem_max = (int)prop.sharedMemPerBlockOptin;
    c->n_sms = prop.multiProcessorCount;
    if (const char* fm = getenv("GP_K3_MODE")) c->force_mode = atoi(fm);
    if (cudaHostAlloc((void**)&c->h_flags, sizeof(uint32_t), cudaHostAllocDefault) != cudaSuccess ||
        cudaHostAlloc((void**)&c->h_solve, sizeof(SolveOut), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer((void**)&c->d_hsolve, c->h_solve, 0) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->flags_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->arena_ev, cudaEventDisableTiming) != cudaSuccess) {
        gp_ctx_destroy(c);
        return fail(GP_ERR_CUDA, "pinned flag / event allocation failed");
    }
    cudaError_t se = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (se != cudaSuccess) { delete c; return fail(GP_ERR_CUDA, "stream: %s", cudaGetErrorString(se)); }
    *out = c;
    return GP_OK;
}

void* gp_ctx_stream(gp_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

void gp_ctx_destroy(gp_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    DBuf<double>* dd[] = {&c->S, &c->g_rf, &c->g_cf, &c->g_dp, &c->g_minmem, &c->sg_minmem,
                          &c->C1, &c->xt, &c->b_cost};
    for (auto* b : dd) b->release();
    c->fbws.release();
    c->kgrp.release();
    c->sshare0.release();
    c->gwbad.release();
    c->vtab.release();
    c->mtab.release();
    c->flagsbuf.release();
    DBuf<uint8_t>* bb[] = {&c->g_tp_ok, &c->scode, &c->skind, &c->b_order, &c->b_counts,
                           &c->b_bm, &c->b_status};
    for (auto* b : bb) b->release();
    c->arena.release();
    if (c->h_stage) cudaFreeHost(c->h_stage);
    if (c->h_arena) cudaFreeHost(c->h_arena);
    c->d_harena = nullptr;
    if (c->h_flags) cudaFreeHost(c->h_flags);
    if (c->h_solve) cudaFreeHost(c->h_solve);
    c->z_bw.release(); c->z_mbw.release(); c->z_xt.release(); c->z_flags.release();
    c->z_tpk.release(); c->z_tcol.release(); c->z_res.release(); c->z_cnt.release();
    c->dsolve.release(); c->d_seq.release(); c->gbest.release(); c->s_tim.release(); c->s_traces.release(); c->s_tidx.release(); c->s_ms.release(); c->s_st.release();
    c->s_rep.release(); c->s_ends.release(); c->g_buf.release(); c->s_wq.release(); c->s_lq.release();
    if (c->flags_ev) cudaEventDestroy(c->flags_ev);
    if (c->t_ev0) cudaEventDestroy(c->t_ev0);
    if (c->t_ev1) cudaEventDestroy(c->t_ev1);
    if (c->arena_ev) cudaEventDestroy(c->arena_ev);
    if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
    for (cudaEvent_t e : c->kt_ev) cudaEventDestroy(e);
    c->binom.release(); c->item_ctr.release(); c->tiles.release(); c->groups.release(); c->prefixes.release(); c->bnk.release(); c->recruns.release(); c->recrow.release(); c->k5_perm.release(); c->k5_hist.release();
    c->tpk.release(); c->tcol.release();
    c->stg.release(); c->gw.release(); c->blk.release(); c->result.release();
    c->counter.release(); c->bam_blk.release(); c->bam_ctr.release(); c->err_idx.release(); c->err_dummy.release(); c->info.release();
    c->ginfo.release(); c->dstatus.release(); c->vbuf.release();
    cudaStreamDestroy(c->stream);
    delete c;
}

static int run_tables(gp_ctx* c, bool full) {
    ++c->tables_gen;
    DevInst I = c->view();
    cudaStream_t s = c->stream;
    CUDA_TRY(cudaMemsetAsync(c->flagsbuf.p, 0, sizeof(uint32_t), s));
    if (full) {
        // interval sums + group constants + gateways (independent) in one launch
        const int gw_blocks = (c->F * c->F + 3) / 4;
        K1Reset R = {nullptr, nullptr, 0u};
        k1_phase1<<<5 + c->F + gw_blocks, 128, 0, s>>>(I, R);
    } else {
        k1_gateways<<<(c->F * c->F * 32 + 127) / 128, 128, 0, s>>>(I);
    }
    // stage table + boundary table in one launch
    long long ns = (long long)c->F * (c->n + 1) * (c->n + 1);
    long long nx = (long long)c->nm * c->F * c->F * c->n;
    k1_phase2<<<(unsigned)((ns + nx + 127) / 128), 128, 0, s>>>(I, ns);
    CUDA_TRY(cudaGetLastError());
    // flags travel back asynchronously; kernels consult the device copy when
    // the host copy is not known yet (no synchronisation on the load path)
    CUDA_TRY(cudaMemcpyAsync(c->h_flags, c->flagsbuf.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaEventRecord(c->flags_ev, s));
    c->flags_known = false;
    return GP_OK;
}

// host-side flags when the async read-back has landed; -1 when still pending
static int known_flags(gp_ctx* c) {
    if (c->capturing) return -1;  // graph: device-side dispatch
    if (c->flags_known) return (int)c->flags;
    if (cudaEventQuery(c->flags_ev) == cudaSuccess) {
        c->flags = *c->h_flags;
        c->flags_known = true;
        return (int)c->flags;
    }
    return -1;
}

static void replan_key(const gp_ctx* c, const gp_instance* in, unsigned long long* key);

int gp_ctx_load(gp_ctx* c, const gp_instance* in) {
    if (c) { c->ctr_armed = 0; c->err_clean = false; }  // launches below skip neither reset
    if (c) memset(c->loaded_key, 0, sizeof(c->loaded_key));  // valid again once this load succeeds
    if (!c || !in) return fail(GP_ERR_INPUT, "null argument");
    if (in->n_layers < 1 || in->n_layers > GP_MAX_LAYERS)
        return fail(GP_ERR_INPUT, "n_layers %u outside [1, %d]", in->n_layers, GP_MAX_LAYERS);
    if (in->n_fgs < 1 || in->n_fgs > GP_MAX_STAGES)
        return fail(GP_ERR_INPUT, "n_fgs %u outside [1, %d]", in->n_fgs, GP_MAX_STAGES);
    if (in->n_batch < 1 || in->n_micro < 1 || in->n_batch * in->n_micro > 255)
        return fail(GP_ERR_INPUT, "bad (batch, micro) candidate counts");
    for (uint32_t i = 0; i < in->n_batch; ++i)
        for (uint32_t j = 0; j < in->n_micro; ++j)
            if (in->batch[i] <= 0 || in->micro[j] <= 0 || in->batch[i] % in->micro[j])
                return fail(GP_ERR_INPUT, "micro-batch %lld does not divide batch %lld",
                            (long long)in->micro[j], (long long)in->batch[i]);
    uint32_t nsg = in->fg_sg_offset[in->n_fgs];
    for (uint32_t f = 0; f < in->n_fgs; ++f) {
        uint32_t nm = in->fg_member_offset[f + 1] - in->fg_member_offset[f];
        uint32_t ng = in->fg_sg_offset[f + 1] - in->fg_sg_offset[f];
        if (nm < 1 || nm > GP_MAX_MEMBERS) return fail(GP_ERR_INPUT, "group %u has %u members", f, nm);
        if (ng > GP_MAX_SGS) return fail(GP_ERR_INPUT, "group %u has %u subgroups", f, ng);
    }
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    uint32_t n = in->n_layers, D = in->n_devices, F = in->n_fgs;
    c->n = (int)n; c->F = (int)F; c->D = (int)D; c->nb = (int)in->n_batch; c->nm = (int)in->n_micro;
    c->h_fg_sg_count.assign(F, 0u);
    for (uint32_t f = 0; f < F; ++f) c->h_fg_sg_count[f] = in->fg_sg_offset[f + 1] - in->fg_sg_offset[f];
    c->nsg = (int)nsg;
    c->bf = in->bottleneck_factor;
    c->h_batch.assign(in->batch, in->batch + in->n_batch);
    c->h_micro.assign(in->micro, in->micro + in->n_micro);
    size_t DD = (size_t)D * D;
    uint32_t nfm = in->fg_member_offset[F];
    uint32_t nsm = in->sg_member_offset[nsg];
    // arena layout: every array 16-byte aligned
    struct Seg { const void* src; size_t bytes; size_t off; };
    Seg seg[24];
    int ns = 0;
    size_t off = 0;
    auto add = [&](const void* src, size_t bytes) {
        seg[ns].src = src; seg[ns].bytes = bytes; seg[ns].off = off;
        off += (bytes + 15) & ~(size_t)15;
        return ns++;
    };
    const int i_fwd = add(in->fwd_flops, n * 8), i_bwd = add(in->bwd_input_flops, n * 8),
              i_wgt = add(in->bwd_weight_flops, n * 8), i_act = add(in->activation_out_bytes, n * 8),
              i_par = add(in->param_bytes, n * 8), i_b = add(in->batch, in->n_batch * 8),
              i_m = add(in->micro, in->n_micro * 8), i_pc = add(in->p_c, D * 8),
              i_mem = add(in->memory_bytes, D * 8), i_rank = add(in->id_rank, D * 4),
              i_pt = add(in->p_t, DD * 8), i_lat = add(in->latency, DD * 8),
              i_bw = add(in->bandwidth, DD * 8), i_foff = add(in->fg_member_offset, (F + 1) * 4),
              i_fmem = add(in->fg_members, nfm * 4), i_fcap = add(in->fg_capacity, F * 8),
              i_fbwi = add(in->fg_min_bw, F * 8), i_fbw = add(in->fg_min_bw, F * 8),
              i_fhas = add(in->fg_has_min_bw, F), i_fsg = add(in->fg_sg_offset, (F + 1) * 4),
              i_soff = add(in->sg_member_offset, (nsg + 1) * 4), i_smem = add(in->sg_members, nsm * 4),
              i_scap = add(in->sg_capacity, nsg * 8);
    if (c->arena_ev) CUDA_TRY(cudaEventSynchronize(c->arena_ev));  // last H2D done
    if (off > c->h_arena_cap) {
        if (c->h_arena) cudaFreeHost(c->h_arena);
        c->h_arena = nullptr;
        c->h_arena_cap = 0;
        CUDA_TRY(cudaHostAlloc((void**)&c->h_arena, off, cudaHostAllocMapped));
        c->h_arena_cap = off;
        void* dp = nullptr;
        CUDA_TRY(cudaHostGetDevicePointer(&dp, c->h_arena, 0));
        c->d_harena = (const unsigned char*)dp;
    }
    for (int i = 0; i < ns; ++i)
        if (seg[i].bytes) memcpy(c->h_arena + seg[i].off, seg[i].src, seg[i].bytes);
    CUDA_TRY(c->arena.ensure(off));
    CUDA_TRY(cudaMemcpyAsync(c->arena.p, c->h_arena, off, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaEventRecord(c->arena_ev, s));
    unsigned char* A = c->arena.p;
    c->fwd.p = (double*)(A + seg[i_fwd].off);
    c->bwd_in.p = (double*)(A + seg[i_bwd].off);
    c->bwd_w.p = (double*)(A + seg[i_wgt].off);
    c->act.p = (double*)(A + seg[i_act].off);
    c->param.p = (double*)(A + seg[i_par].off);
    c->batch.p = (long long*)(A + seg[i_b].off);
    c->micro.p = (long long*)(A + seg[i_m].off);
    c->p_c.p = (double*)(A + seg[i_pc].off);
    c->mem.p = (double*)(A + seg[i_mem].off);
    c->id_rank.p = (uint32_t*)(A + seg[i_rank].off);
    c->p_t.p = (double*)(A + seg[i_pt].off);
    c->lat.p = (double*)(A + seg[i_lat].off);
    c->bw.p = (double*)(A + seg[i_bw].off);
    c->fg_off.p = (uint32_t*)(A + seg[i_foff].off);
    c->fg_mem.p = (uint32_t*)(A + seg[i_fmem].off);
    c->fg_cap.p = (double*)(A + seg[i_fcap].off);
    c->fg_minbw_in.p = (double*)(A + seg[i_fbwi].off);
    c->fg_minbw.p = (double*)(A + seg[i_fbw].off);
    c->fg_has.p = (uint8_t*)(A + seg[i_fhas].off);
    c->fg_sg_off.p = (uint32_t*)(A + seg[i_fsg].off);
    c->sg_off.p = (uint32_t*)(A + seg[i_soff].off);
    c->sg_mem.p = (uint32_t*)(A + seg[i_smem].off);
    c->sg_cap.p = (double*)(A + seg[i_scap].off);
    c->arena_bytes = off;
    size_t N2 = (size_t)(n + 1) * (n + 1);
    CUDA_TRY(c->S.ensure(5 * N2));
    CUDA_TRY(c->g_tp_ok.ensure(F));
    CUDA_TRY(c->kgrp.ensure(F));
    CUDA_TRY(c->sshare0.ensure((size_t)F * N2));
    CUDA_TRY(c->gwbad.ensure((size_t)F * F));
    CUDA_TRY(c->g_rf.ensure(nfm));
    CUDA_TRY(c->g_cf.ensure(nfm));
    CUDA_TRY(c->g_dp.ensure(nsg ? nsg : 1));
    CUDA_TRY(c->g_minmem.ensure(F));
    CUDA_TRY(c->sg_minmem.ensure(nsg ? nsg : 1));
    CUDA_TRY(c->stg.ensure((size_t)c->nm * F * N2));
    CUDA_TRY(c->scode.ensure((size_t)F * N2));
    CUDA_TRY(c->skind.ensure((size_t)F * N2));
    CUDA_TRY(c->C1.ensure((size_t)F * N2));
    CUDA_TRY(c->fbws.ensure((size_t)F * N2));
    CUDA_TRY(c->vtab.ensure((size_t)c->nm * F * ((size_t)n * (n + 1) / 2)));
    CUDA_TRY(c->mtab.ensure(256));
    CUDA_TRY(c->gw.ensure((size_t)F * F));
    CUDA_TRY(c->xt.ensure((size_t)c->nm * F * F * ((n + 1) & ~1u)));
    CUDA_TRY(c->tpk.ensure((size_t)c->nm * F * ((size_t)n * (n + 1) / 2)));
    CUDA_TRY(c->tcol.ensure((size_t)c->nm * F * (n + 1)));
    CUDA_TRY(c->flagsbuf.ensure(1));
    CUDA_TRY(c->counter.ensure(3));  // slots: a split range's sweep + 2 edge pieces
    CUDA_TRY(c->result.ensure(3));
    CUDA_TRY(c->err_idx.ensure(1));
    CUDA_TRY(c->blk.ensure(4096));  // >= the generic fix-up grid (no realloc mid-stream)
    CUDA_TRY(cudaMemsetAsync(c->counter.p, 0, c->counter.cap * sizeof(unsigned int), s));
    if (!c->binom.p) {
        // C(nn, r) for nn < 257, r <= GP_MAX_STAGES (composition unranking)
        std::vector<unsigned long long> tab((size_t)BINOM_ROWS * (GP_MAX_STAGES + 1), 0ull);
        for (int nn = 0; nn < BINOM_ROWS; ++nn)
            for (int r = 0; r <= GP_MAX_STAGES; ++r) tab[(size_t)nn * (GP_MAX_STAGES + 1) + r] = h_binom(nn, r);
        CUDA_TRY(upload(s, c->binom, tab.data(), tab.size()));
    }
    int st = run_tables(c, true);
    if (st != GP_OK) return st;
    c->bw_off = seg[i_bw].off;
    // enumeration helpers depend on (n, k) only: rebuild when those change
    if (c->cache_n == (int)n && c->cache_k == (int)F) {
        c->loaded = true;
        replan_key(c, in, c->loaded_key);
        return GP_OK;
    }
    c->cache_n = (int)n;
    c->cache_k = (int)F;
    c->tiles_ok = false;  // K3 tile table: built lazily by the sub-range path
    // K3 sweep run groups (see k3_sweep): full K3_SEG runs by a, then partial
    // runs grouped by length, longest first
    c->sweep_ok = false;
    if ((int)F >= 3 && (int)F <= (int)n) {
        int k = (int)F, nn = (int)n;
        std::vector<uint4> g;
        unsigned long long start = 0;
        for (int a = k - 2; a <= nn - 2; ++a) {
            unsigned long long rows = h_binom(a - 1, k - 3);
            int L = nn - 1 - a, nf = L / K3_SEG;
            if (rows && nf) {
                g.push_back(make_uint4((unsigned)start, (unsigned)a | ((unsigned)K3_SEG << 16),
                                       (unsigned)rows, (unsigned)nf));
                start += rows * nf;
            }
        }
        for (int len = K3_SEG - 1; len >= 1; --len)
            for (int a = k - 2; a <= nn - 2; ++a) {
                int L = nn - 1 - a;
                if (L % K3_SEG != len) continue;
                unsigned long long rows = h_binom(a - 1, k - 3);
                if (!rows) continue;
                g.push_back(make_uint4((unsigned)start, (unsigned)a | ((unsigned)len << 16),
                                       (unsigned)rows, 0u));
                start += rows;
            }
        // colex list of (k-3)-subsets of [1, n-3]: the subsets of [1, a-1]
        // are exactly its first C(a-1, k-3) entries
        std::vector<uint8_t> pre;
        unsigned long long npre = (k > 3) ? h_binom(nn - 3, k - 3) : 1;
        bool pre_ok = npre <= (1ull << 22);
        if (pre_ok && k > 3) {
            int m = k - 3;
            std::vector<int> cmb(m);
            for (int i = 0; i < m; ++i) cmb[i] = i + 1;
            pre.assign((size_t)npre * 16, 0);
            for (unsigned long long r = 0; r < npre; ++r) {
                for (int i = 0; i < m; ++i) pre[r * 16 + i] = (uint8_t)cmb[i];
                // colex successor: smallest i with cmb[i] + 1 < cmb[i+1] (or last)
                int i = 0;
                while (i < m - 1 && cmb[i] + 1 == cmb[i + 1]) ++i;
                ++cmb[i];
                for (int j = 0; j < i; ++j) cmb[j] = j + 1;
            }
        }
        if (pre_ok && start < (1ull << 31) && !g.empty()) {
            if (k > 3) CUDA_TRY(upload(s, c->prefixes, pre.data(), pre.size()));
            std::vector<unsigned long long> bk((size_t)(nn + 1) * (k + 1) + 2, 0ull);
            for (int a = 0; a <= nn; ++a)
                for (int r = 0; r <= k; ++r) bk[(size_t)a * (k + 1) + r] = h_binom(a, r);
            CUDA_TRY(upload(s, c->bnk, bk.data(), bk.size()));
            // task t (runs 32t .. 32t+31) -> group of its first run, u16,
            // appended after the groups (one staged block)
            const int ng = (int)g.size();
            const unsigned long long ntask = (start + 31) / 32;
            std::vector<uint16_t> tg((size_t)ntask + 8, 0);
            for (unsigned long long t = 0, gi = 0; t < ntask; ++t) {
                while (gi + 1 < g.size() && g[gi + 1].x <= t * 32) ++gi;
                tg[t] = (uint16_t)gi;
            }
            const size_t tslots = ((size_t)ntask * 2 + 15) / 16;
            g.resize(g.size() + tslots);
            memcpy(&g[ng], tg.data(), tslots * 16 <= tg.size() * 2 ? tslots * 16 : tg.size() * 2);
            CUDA_TRY(upload(s, c->groups, g.data(), g.size()));
            c->ngroups = (int)g.size();
            c->ng = ng;
            c->sweep_W = (unsigned)start;
            c->sweep_ok = true;
        }
        // record sweep: one run per (prefix, a), a ascending (runs longest
        // first), prefixes in colex order; rpre = composition rank of
        // (prefix, a, q = a + 1)
        c->rec_ok = false;
        if (k <= 6 && (k == 3 || pre_ok)) {
            std::vector<K3Run> runs;
            runs.reserve((size_t)h_binom(nn - 2, k - 2));
            for (int a = k - 2; a <= nn - 2; ++a) {
                const unsigned long long rows = h_binom(a - 1, k - 3);
                for (unsigned long long r = 0; r < rows; ++r) {
                    K3Run x = {};
                    int p[8] = {0};
                    for (int j = 1; j <= k - 3; ++j) p[j] = pre[(size_t)r * 16 + (j - 1)];
                    p[k - 2] = a;
                    for (int j = 0; j < k - 3; ++j) x.p[j] = (uint8_t)p[j + 1];
                    x.a = (uint8_t)a;
                    x.len = (uint8_t)(nn - 1 - a);
                    unsigned long long rp = 0;
                    for (int j = 1; j <= k - 2; ++j)
                        rp += h_binom(nn - p[j - 1] - 1, k - j) - h_binom(nn - p[j], k - j);
                    x.rpre = rp;
                    runs.push_back(x);
                }
            }
            for (size_t t0 = 0; t0 < runs.size(); t0 += 32) {
                int mx = 0;
                for (size_t u = t0; u < runs.size() && u < t0 + 32; ++u) mx = std::max(mx, k3r_lenp(nn, runs[u].a));
                for (size_t u = t0; u < runs.size() && u < t0 + 32; ++u) runs[u].tmax = (uint8_t)mx;
            }
            std::vector<uint32_t> rs((size_t)nn + 4, 0u);
            for (int a = k - 2, acc = 0; a <= nn - 2; ++a) { rs[a] = (uint32_t)acc; acc += k3r_lenp(nn, a); }
            if (!runs.empty() && runs.size() < (1ull << 31)) {
                CUDA_TRY(upload(s, c->recrow, rs.data(), rs.size()));
                CUDA_TRY(upload(s, c->recruns, runs.data(), runs.size()));
                c->rec_W = (unsigned)runs.size();
                c->rec_ok = true;
            }
        }
    }
    c->loaded = true;
    replan_key(c, in, c->loaded_key);
    return GP_OK;
}

static int ensure_tiles(gp_ctx* c) {
    if (c->tiles_ok) return GP_OK;
    int n = c->n, F = c->F;
    if (F >= 3 && F <= n) {
        unsigned long long NC = h_binom(n - 1, F - 1);
        unsigned long long ntiles = (NC + K3_TILE - 1) / K3_TILE;
        if (ntiles <= (1ull << 22)) {
            CUDA_TRY(c->tiles.ensure(ntiles * 16));
            k_tiles<<<(unsigned)((ntiles + 127) / 128), 128, 0, c->stream>>>(n, F, ntiles, c->tiles.p);
            CUDA_TRY(cudaGetLastError());
            c->tiles_ok = true;
        }
    }
    return GP_OK;
}

int gp_set_bandwidth(gp_ctx* c, const double* bandwidth) {
    if (!c || !c->loaded || !bandwidth) return fail(GP_ERR_INPUT, "context not loaded");
    CUDA_TRY(cudaSetDevice(c->device));
    size_t DD = (size_t)c->D * c->D;
    CUDA_TRY(cudaMemcpyAsync(c->bw.p, bandwidth, DD * sizeof(double), cudaMemcpyHostToDevice,
                             c->stream));
    DevInst I = c->view();
    k1_minbw<<<(c->F + 31) / 32, 32, 0, c->stream>>>(I, c->fg_minbw.p);
    CUDA_TRY(cudaGetLastError());
    return run_tables(c, false);
}

// Restore the loaded instance's bandwidth matrix and its GroupIndex
// min_intra_bandwidth values (not re-derived from the matrix: a hierarchy
// read from file may carry other values), then the boundary/AL tables.
int gp_reset_bandwidth(gp_ctx* c) {
    if (!c || !c->loaded) return fail(GP_ERR_INPUT, "context not loaded");
    CUDA_TRY(cudaSetDevice(c->device));
    if (c->arena_ev) CUDA_TRY(cudaEventSynchronize(c->arena_ev));  // pinned arena = loaded instance
    const size_t DD = (size_t)c->D * c->D;
    CUDA_TRY(cudaMemcpyAsync(c->bw.p, c->h_arena + c->bw_off, DD * sizeof(double),
                             cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->fg_minbw.p, c->fg_minbw_in.p, (size_t)c->F * sizeof(double),
                             cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(cudaEventRecord(c->arena_ev, c->stream));
    return run_tables(c, false);
}

static int kernel_slots(gp_ctx* c, const void* kern, int threads, size_t smem, int* per_sm);

int gp_argmin_batch_device(gp_ctx* c, uint64_t n, const double* d_cost, const uint8_t* d_status,
                           const uint64_t* d_keys, uint64_t* d_out) {
    if (!c || (n && (!d_cost || !d_status)) || !d_out) return fail(GP_ERR_INPUT, "bad arguments");
    CUDA_TRY(cudaSetDevice(c->device));
    const unsigned long long gmax = 2ull * (unsigned long long)c->n_sms;
    if (!c->bam_ctr.p) {
        CUDA_TRY(c->bam_ctr.ensure(1));
        CUDA_TRY(c->bam_blk.ensure(gmax));  // fixed capacity: never reallocated under a launch
        CUDA_TRY(cudaMemsetAsync(c->bam_ctr.p, 0, sizeof(unsigned int), c->stream));
    }
    unsigned long long grid = (n + 1023) / 1024;
    if (grid > gmax) grid = gmax;
    if (grid < 1) grid = 1;
    ArgminScratch S;
    S.blk = c->bam_blk.p;
    S.counter = c->bam_ctr.p;
    S.result = reinterpret_cast<Key*>(d_out);
    S.err = nullptr;
    S.err_idx = nullptr;
    k2_batch_argmin<<<(unsigned)grid, 256, 0, c->stream>>>((unsigned long long)n, d_cost, d_status,
                                                          reinterpret_cast<const unsigned long long*>(d_keys), S);
    CUDA_TRY(cudaGetLastError());
    return GP_OK;
}

int gp_eval_batch_device(gp_ctx* c, uint32_t k, uint64_t n, const uint8_t* d_order,
                         const uint8_t* d_counts, const uint8_t* d_bm, double* d_cost,
                         uint8_t* d_status) {
    if (!c || !c->loaded) return fail(GP_ERR_INPUT, "context not loaded");
    if (k < 1 || k > GP_MAX_STAGES) return fail(GP_ERR_INPUT, "k=%u outside [1,%d]", k, GP_MAX_STAGES);
    if (n == 0) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    DevInst I = c->view();
    // large batches: persistent kernel with the stage codes in shared memory
    // (GP_K2_SC=0 disables); small ones (search_plan beams): one thread each
    const size_t sc_bytes = (((size_t)c->F * (c->n + 1) * (c->n + 1)) + 15) & ~(size_t)15;
    bool sc = n >= (1u << 16) && k >= 2 && k <= 6 && sc_bytes <= (96u << 10) &&
              ((k != 4) || (((uintptr_t)d_order | (uintptr_t)d_counts) & 3u) == 0);
    if (const char* e = getenv("GP_K2_SC")) sc = sc && atoi(e) != 0;
    if (sc) {
        typedef void (*K2Fn)(DevInst, long long, const uint8_t*, const uint8_t*, const uint8_t*,
                             double*, uint8_t*);
        static const K2Fn tab[5] = {k2_eval_batch_sc<2>, k2_eval_batch_sc<3>, k2_eval_batch_sc<4>,
                                    k2_eval_batch_sc<5>, k2_eval_batch_sc<6>};
        // k = 4 (and < 2^32 candidates): the warp-compacted variant
        bool q4 = k == 4 && n < (1ull << 32);
        if (const char* e = getenv("GP_K2_Q4")) q4 = q4 && atoi(e) != 0;
        // k = 4 with 16-byte aligned arrays: the TMA-fed chunk kernel
        // (GP_K2_TMA=0 disables)
        bool t4 = q4 && ((((uintptr_t)d_order | (uintptr_t)d_counts | (uintptr_t)d_bm) & 15u) == 0) &&
                  k2t_smem(sc_bytes) <= (size_t)c->smem_max;
        if (const char* e = getenv("GP_K2_TMA")) t4 = t4 && atoi(e) != 0;
        // vector-lane variant: 32-byte aligned costs, 4-byte aligned status
        // (GP_K2_V4=0 disables)
        bool v4 = t4 && ((((uintptr_t)d_cost) & 31u) == 0) && ((((uintptr_t)d_status) & 3u) == 0) &&
                  c->n + 1 <= 128 && k2v_smem(c->F, c->n, c->nm, I.nxp, 8, false) <= (size_t)c->smem_max;
        if (const char* e = getenv("GP_K2_V4")) v4 = v4 && atoi(e) != 0;
        if (v4) {
            // 16 warps with the first/last-stage and boundary tables in shared
            // memory when they fit (GP_K2_SMT=0 disables), else 8 warps
            bool smt = k2v_smem(c->F, c->n, c->nm, I.nxp, K2V_NW, true) <= (size_t)c->smem_max;
            if (const char* e = getenv("GP_K2_SMT")) smt = smt && atoi(e) != 0;
            const int nw = smt ? K2V_NW : 8;
            const void* kfn = smt ? (const void*)k2_eval_batch_v4<K2V_NW, true> : (const void*)k2_eval_batch_v4<8, false>;
            const size_t smem_v = k2v_smem(c->F, c->n, c->nm, I.nxp, nw, smt);
            int per_sm = 0;
            { int st_ = kernel_slots(c, kfn, nw * 32, smem_v, &per_sm);
              if (st_ != GP_OK) return st_; }
            unsigned long long grid = (unsigned long long)(per_sm > 0 ? per_sm : 1) * c->n_sms;
            const unsigned long long chunks = (n + (unsigned long long)K2V_WCHUNK * nw - 1) /
                                              ((unsigned long long)K2V_WCHUNK * nw);
            if (grid > chunks) grid = chunks;
            const uint8_t* img = nullptr;
            if (smt) {  // the shared-memory image of this table generation
                const size_t ib = k2v_bits_bytes(c->F, c->n) + k2v_tab_bytes(c->F, c->n, c->nm, I.nxp);
                if (c->k2img_gen != c->tables_gen || !c->k2img.p) {
                    CUDA_TRY(c->k2img.ensure(ib));
                    k2_image_build<<<c->n_sms, 256, 0, c->stream>>>(I, c->k2img.p);
                    CUDA_TRY(cudaGetLastError());
                    c->k2img_gen = c->tables_gen;
                }
                img = c->k2img.p;
            }
            if (smt)
                k2_eval_batch_v4<K2V_NW, true><<<(unsigned)grid, K2V_NW * 32, smem_v, c->stream>>>(
                    I, (long long)n, d_order, d_counts, d_bm, d_cost, d_status, img);
            else
                k2_eval_batch_v4<8, false><<<(unsigned)grid, 256, smem_v, c->stream>>>(
                    I, (long long)n, d_order, d_counts, d_bm, d_cost, d_status, nullptr);
            CUDA_TRY(cudaGetLastError());
            return GP_OK;
        }
        if (t4) {
            const size_t smem_t = k2t_smem(sc_bytes);
            int per_sm = 0;
            { int st_ = kernel_slots(c, (const void*)k2_eval_batch_t4, K2T_THREADS, smem_t, &per_sm);
              if (st_ != GP_OK) return st_; }
            unsigned long long grid = (unsigned long long)(per_sm > 0 ? per_sm : 1) * c->n_sms;
            const unsigned long long chunks = (n + (unsigned long long)K2T_WCHUNK * K2T_WARPS - 1) /
                                              ((unsigned long long)K2T_WCHUNK * K2T_WARPS);
            if (grid > chunks) grid = chunks;
            k2_eval_batch_t4<<<(unsigned)grid, K2T_THREADS, smem_t, c->stream>>>(
                I, (long long)n, d_order, d_counts, d_bm, d_cost, d_status, (unsigned)sc_bytes);
            CUDA_TRY(cudaGetLastError());
            return GP_OK;
        }
        const K2Fn kern = q4 ? k2_eval_batch_q4 : tab[k - 2];
        const size_t smem_k2 = sc_bytes + (q4 ? (K2Q_THREADS / 32) * 64 * sizeof(uint4) : 0);
        int per_sm = 0;
        { int st_ = kernel_slots(c, (const void*)kern, 256, smem_k2, &per_sm);
          if (st_ != GP_OK) return st_; }
        unsigned long long grid = (unsigned long long)(per_sm > 0 ? per_sm : 1) * c->n_sms;
        const unsigned long long need = (n + 255) / 256;
        if (grid > need) grid = need;
        kern<<<(unsigned)grid, 256, smem_k2, c->stream>>>(I, (long long)n, d_order, d_counts, d_bm,
                                                          d_cost, d_status);
        CUDA_TRY(cudaGetLastError());
        return GP_OK;
    }
    unsigned blocks = (unsigned)((n + 255) / 256);
    k2_eval_batch<<<blocks, 256, 0, c->stream>>>(I, (int)k, (long long)n, d_order, d_counts, d_bm,
                                                 d_cost, d_status);
    CUDA_TRY(cudaGetLastError());
    return GP_OK;
}

int gp_eval_batch(gp_ctx* c, uint32_t k, uint64_t n, const uint8_t* order, const uint8_t* counts,
                  const uint8_t* bm, double* cost, uint8_t* status) {
    if (!c || !c->loaded) return fail(GP_ERR_INPUT, "context not loaded");
    if (n == 0) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    CUDA_TRY(c->b_order.ensure(n * k));
    CUDA_TRY(c->b_counts.ensure(n * k));
    CUDA_TRY(c->b_bm.ensure(n));
    CUDA_TRY(c->b_cost.ensure(n));
    CUDA_TRY(c->b_status.ensure(n));
    CUDA_TRY(cudaMemcpyAsync(c->b_order.p, order, n * k, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->b_counts.p, counts, n * k, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->b_bm.p, bm, n, cudaMemcpyHostToDevice, s));
    int st = gp_eval_batch_device(c, k, n, c->b_order.p, c->b_counts.p, c->b_bm.p, c->b_cost.p,
                                  c->b_status.p);
    if (st != GP_OK) return st;
    CUDA_TRY(cudaMemcpyAsync(cost, c->b_cost.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(status, c->b_status.p, n, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return GP_OK;
}

static unsigned long long h_fact(int k) {
    unsigned long long f = 1;
    for (int i = 2; i <= k; ++i) f *= (unsigned long long)i;
    return f;
}

int gp_space_size(gp_ctx* c, uint64_t* out) {
    if (!c || !c->loaded || !out) return fail(GP_ERR_INPUT, "context not loaded");
    int k = c->F;
    if (k > c->n) { *out = 0; return GP_OK; }
    unsigned __int128 v = (unsigned __int128)c->nb * c->nm * h_fact(k);
    const unsigned long long nc = h_binom(c->n - 1, k - 1);
    v *= nc;
    if (nc == ~0ull || v > (unsigned __int128)~0ull) {
        *out = ~0ull;
        return fail(GP_ERR_INPUT, "candidate space of %d groups x %d layers exceeds 2^64", k, c->n);
    }
    *out = (uint64_t)v;
    return GP_OK;
}

// Sweep launch over items [item_lo, item_hi) of (mi * k! + order).
// threads per block for one-thread-per-item kernels: 128, or fewer so that a
// small batch still spreads over every SM (latency-bound loops per thread)
static int item_tpb(gp_ctx* c, unsigned long long n) {
    const unsigned long long per = (unsigned long long)c->n_sms * 2;
    unsigned long long t = (n + per - 1) / per;
    t = (t + 31) / 32 * 32;
    return t < 32 ? 32 : (t > 128 ? 128 : (int)t);
}

// sweep variant: shared-memory mode x batch sizes per m x (k = 3..6 fixed at
// compile time in the all-shared-memory mode, else generic)
static SwFn pick_sweep(int mode, int nb, int k) {
    static const SwFn table[3][4] = {
        {k3_sweep<0, 1, 0>, k3_sweep<0, 2, 0>, k3_sweep<0, 3, 0>, k3_sweep<0, 4, 0>},
        {k3_sweep<1, 1, 0>, k3_sweep<1, 2, 0>, k3_sweep<1, 3, 0>, k3_sweep<1, 4, 0>},
        {k3_sweep<2, 1, 0>, k3_sweep<2, 2, 0>, k3_sweep<2, 3, 0>, k3_sweep<2, 4, 0>}};
    static const SwFn fixed[4][4] = {
        {k3_sweep<2, 1, 3>, k3_sweep<2, 1, 4>, k3_sweep<2, 1, 5>, k3_sweep<2, 1, 6>},
        {k3_sweep<2, 2, 3>, k3_sweep<2, 2, 4>, k3_sweep<2, 2, 5>, k3_sweep<2, 2, 6>},
        {k3_sweep<2, 3, 3>, k3_sweep<2, 3, 4>, k3_sweep<2, 3, 5>, k3_sweep<2, 3, 6>},
        {k3_sweep<2, 4, 3>, k3_sweep<2, 4, 4>, k3_sweep<2, 4, 5>, k3_sweep<2, 4, 6>}};
    return (mode == 2 && k >= 3 && k <= 6) ? fixed[nb - 1][k - 3] : table[mode][nb - 1];
}

// record sweep (k3_sweep_rec.cuh) for k = 3..6, when its shared memory fits
// and each CTA owns a whole item (the per-item record build is then paid
// once per item; GP_K3_REC=0 disables, force_mode 5 forces it); nullptr
// otherwise
static SwFn pick_sweep_rec(gp_ctx* c, int nb, int k, size_t* smem) {
    static const SwFn table[4][4] = {
        {k3_sweep_rec<1, 3>, k3_sweep_rec<1, 4>, k3_sweep_rec<1, 5>, k3_sweep_rec<1, 6>},
        {k3_sweep_rec<2, 3>, k3_sweep_rec<2, 4>, k3_sweep_rec<2, 5>, k3_sweep_rec<2, 6>},
        {k3_sweep_rec<3, 3>, k3_sweep_rec<3, 4>, k3_sweep_rec<3, 5>, k3_sweep_rec<3, 6>},
        {k3_sweep_rec<4, 3>, k3_sweep_rec<4, 4>, k3_sweep_rec<4, 5>, k3_sweep_rec<4, 6>}};
    static const int enabled = [] { const char* e = getenv("GP_K3_REC"); return e ? atoi(e) : 1; }();
    if (!enabled || k < 3 || k > 6 || nb < 1 || nb > 4 || !c->rec_ok) return nullptr;
    if (c->force_mode >= 0 && c->force_mode != 5) return nullptr;  // diagnostics pick a variant
    const size_t need = k3r_smem(c->n, k, nb);
    if (need > (size_t)c->smem_max) return nullptr;
    *smem = need;
    return c->verify ? pick_sweep_rec_verify(nb, k) : table[nb - 1][k - 3];
}

// Sweep launch.  With GP_K3_CLUSTER=c (2 or 4, dividing the CTAs per item)
// the CTAs of one item form a thread-block cluster and the item's tables are
// fetched once and multicast into every member (TMA .multicast::cluster).
// Measured on C4 (profiles/README.md): cluster 2 = no change (36.9 us),
// cluster 4 = 51 us (72 clusters of 4 x 113 KB do not co-schedule in one wave
// across the GPCs), so the default is a plain launch.
static cudaError_t launch_sweep_kernel(SwFn kern, unsigned grid, size_t smem, cudaStream_t s,
                                       SweepGeom& G, const DevInst& I, const ArgminScratch& S,
                                       const unsigned long long* binom, const uint32_t* flags,
                                       bool pdl = false) {
    int cs = 1;
    if (const char* e = getenv("GP_K3_CLUSTER")) cs = atoi(e) > 0 ? atoi(e) : 1;
    if (cs > 1 && (G.cpi % cs != 0)) cs = 1;
    G.csize = cs;
    G.interleave = 1;
    if (const char* e = getenv("GP_K3_BLOCKMAP")) G.interleave = atoi(e) != 0;
    if (cs == 1) return launch_k(kern, grid, K3S_THREADS, smem, s, pdl, I, G, S, binom, flags);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(K3S_THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, I, G, S, binom, flags);
    if (e != cudaSuccess) {  // cluster not schedulable here: plain launch, no multicast
        (void)cudaGetLastError();
        G.csize = 1;
        kern<<<grid, K3S_THREADS, smem, s>>>(I, G, S, binom, flags);
        e = cudaGetLastError();
    }
    return e;
}

// cudaFuncSetAttribute + occupancy query, once per (device, kernel, dynamic
// smem).  The attribute is process-wide per kernel and device, so the cache
// is too, and the attribute only ever grows (every cached size stays
// launchable whichever context configured a larger one).
struct SlotEntry { int device; const void* kern; size_t smem; int threads, per_sm; };
static std::vector<SlotEntry> g_slot_cache;
static std::mutex g_slot_mu;

static int kernel_slots(gp_ctx* c, const void* kern, int threads, size_t smem, int* per_sm) {
    std::lock_guard<std::mutex> lock(g_slot_mu);
    for (const auto& e : g_slot_cache)
        if (e.device == c->device && e.kern == kern && e.smem == smem && e.threads == threads) {
            *per_sm = e.per_sm;
            return GP_OK;
        }
    size_t top = smem;
    for (const auto& e : g_slot_cache)
        if (e.device == c->device && e.kern == kern && e.smem > top) top = e.smem;
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)top));
    int ps = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kern, threads, smem));
    g_slot_cache.push_back({c->device, kern, smem, threads, ps});
    *per_sm = ps;
    return GP_OK;
}

// event pair around one sweep launch while gp_diag_kernel_timing is on
static cudaError_t kt_mark(gp_ctx* c, bool end) {
    if (!c->ktime || c->capturing) return cudaSuccess;
    const size_t i = c->kt_used + (end ? 1 : 0);
    while (c->kt_ev.size() <= i) {
        cudaEvent_t e;
        cudaError_t err = cudaEventCreate(&e);
        if (err != cudaSuccess) return err;
        c->kt_ev.push_back(e);
    }
    cudaError_t err = cudaEventRecord(c->kt_ev[i], c->stream);
    if (end && err == cudaSuccess) c->kt_used += 2;
    return err;
}

// record sweep (persistent grid): run table, units and the per-CTA run-record
// scratch; `units` = (snapshot, item, chunk) CTA tasks, returns the grid
static int setup_rec(gp_ctx* c, SweepGeom& G) {
    G.runs = c->recruns.p;
    G.W = c->rec_W;
    G.rowstart = c->recrow.p;
    G.nrecp = k3r_nrecp(c->n, c->F);
    return GP_OK;
}

static int launch_sweep(gp_ctx* c, const RangeGeom& R, unsigned long long item_lo,
                        unsigned long long item_hi, int mode, const uint32_t* dflags,
                        int nb_sel = 0, int b0 = 0, int slot = 0) {
    cudaStream_t s = c->stream;
    const int k = R.k, n = c->n;
    size_t ntri = (size_t)n * (n + 1) / 2;
    size_t nxp = (size_t)((n + 1) & ~1);
    size_t smem0 = 16 + (((size_t)(n + 1) * (k + 1) * 8 + 15) & ~(size_t)15) + (size_t)c->ngroups * 16;
    size_t smem1 = smem0 + ntri * 16 + (n + 1) * 16 + 3 * nxp * 8 + (size_t)n * 16;
    size_t smem2 = smem1 + ntri * 16;
    if (mode == 2 && smem2 > (size_t)c->smem_max) mode = 1;
    if (mode == 1 && smem1 > (size_t)c->smem_max) mode = 0;
    size_t smem = mode == 2 ? smem2 : (mode == 1 ? smem1 : smem0);
    SwFn kern = c->verify ? pick_sweep_verify(mode, nb_sel > 0 ? nb_sel : c->nb, k)
                          : pick_sweep(mode, nb_sel > 0 ? nb_sel : c->nb, k);
    bool rec = false;
    if (c->force_mode == 5)  // whole items per CTA only in large batches (K6)
        if (SwFn r = pick_sweep_rec(c, nb_sel > 0 ? nb_sel : c->nb, k, &smem)) { kern = r; rec = true; }
    int per_sm = 0;
    { int st_ = kernel_slots(c, (const void*)kern, K3S_THREADS, smem, &per_sm);
      if (st_ != GP_OK) return st_; }
    unsigned long long resident = (unsigned long long)(per_sm > 0 ? per_sm : 1) * c->n_sms;
    unsigned long long items = item_hi - item_lo;
    unsigned long long tasks = (c->sweep_W + 31) / 32;
    unsigned long long cpi = items >= resident ? 1 : resident / items;
    unsigned long long cap = (tasks + (K3S_THREADS / 32) - 1) / (K3S_THREADS / 32);
    if (cpi > cap) cpi = cap;
    if (cpi < 1) cpi = 1;
    if (const char* e = getenv("GP_K3_CPI")) if (atoi(e) > 0) cpi = (unsigned long long)atoi(e);  // diagnostic
    unsigned long long grid = items * cpi;
    if (grid > 0x7fffffffull) return fail(GP_ERR_INPUT, "item range too large for one launch");
    const unsigned long long units = grid;
    SweepGeom G;
    if (rec) setup_rec(c, G);
    G.k = k;
    G.b0 = b0;
    G.nbm = R.nbm;
    G.NC = R.NC;
    G.NP = R.NP;
    G.item0 = item_lo;
    G.cpi = cpi;
    if (!rec) G.W = c->sweep_W;
    G.ngroups = c->ngroups;
    G.ng = c->ng;
    G.groups = c->groups.p;
    G.prefixes = c->prefixes.p;
    G.bnk = c->bnk.p;
    G.items = (unsigned int)items;
    G.tpk = c->tpk.p;
    G.tcol = c->tcol.p;
    G.xt = c->xt.p;
    G.s_tpk = G.s_tcol = G.s_xt = 0;
    G.gsteps = 1;
    while (G.gsteps * 2 <= c->ngroups) G.gsteps *= 2;
    if (c->verify) G.vs = c->vs;
    if (c->item_ctr.cap < items || !c->item_ctr.p) c->ctr_armed = 0;  // (re)allocation
    CUDA_TRY(c->item_ctr.ensure(items));
    // (the gp_replan graph resets the counters in K1 phase 1; the sweep
    // itself re-arms them at exit)
    if (!c->pdl && items > c->ctr_armed) {
        CUDA_TRY(cudaMemsetAsync(c->item_ctr.p, 0, items * sizeof(unsigned int), s));
        c->ctr_armed = items;
    }
    G.item_ctr = c->item_ctr.p;
    CUDA_TRY(c->blk.ensure(units));
    ArgminScratch S;
    S.blk = c->blk.p;
    S.counter = c->counter.p + slot;
    S.result = c->result.p + slot;
    S.err = nullptr;
    S.err_idx = c->err_idx.p;
    c->last_geom = R;
    DevInst I = c->view();
    CUDA_TRY(kt_mark(c, false));
    CUDA_TRY(launch_sweep_kernel(kern, (unsigned)grid, smem, s, G, I, S, c->binom.p, dflags,
                                 c->pdl));
    CUDA_TRY(kt_mark(c, true));
    return GP_OK;
}

// Generic status-tracking pass that runs only when the device flags are set.
static int launch_fixup(gp_ctx* c, const RangeGeom& G) {
    // grid-stride over the range; small grid because the kernel usually only
    // reads the (clear) flag and exits
    unsigned long long grid = (G.hi - G.lo + 255) / 256;
    unsigned long long gmax = (unsigned long long)c->n_sms * 2;
    if (grid > gmax) grid = gmax;
    if (grid < 1) grid = 1;
    CUDA_TRY(c->blk.ensure(grid));
    ArgminScratch S;
    S.blk = c->blk.p;
    S.counter = c->counter.p;
    S.result = c->result.p;
    S.err = nullptr;
    S.err_idx = c->err_idx.p;
    DevInst I = c->view();
    CUDA_TRY(launch_k(k3_argmin_generic, (unsigned)grid, 256, 0, c->stream, c->pdl, I, G, S,
                      (const uint32_t*)c->flagsbuf.p));
    return GP_OK;
}

static int range_async(gp_ctx* c, uint64_t lo, uint64_t hi, int slot);

int gp_argmin_range_async(gp_ctx* c, uint64_t lo, uint64_t hi) {
    return range_async(c, lo, hi, -1);
}

// slot < 0: a caller's range (resets, and the split below); slot >= 0: an
// edge piece of a split range, its key into result slot `slot`
static int range_async(gp_ctx* c, uint64_t lo, uint64_t hi, int slot) {
    if (!c || !c->loaded) return fail(GP_ERR_INPUT, "context not loaded");
    const bool top = slot < 0;
    if (top) slot = 0;
    int k = c->F;
    uint64_t total;
    { int st_ = gp_space_size(c, &total); if (st_ != GP_OK) return st_; }
    if (hi > total) hi = total;
    if (lo > hi) lo = hi;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    RangeGeom G;
    G.k = k;
    G.nbm = c->nb * c->nm;
    G.NC = h_binom(c->n - 1, k - 1);
    G.NP = h_fact(k);
    G.lo = lo;
    G.hi = hi;
    G.items_mode = 0;
    G.it_lo = 0;
    G.it_span = 1;
    G.nm = c->nm;
    G.item_ctr = nullptr;
    G.tiles = nullptr;
    if (top) {
        c->last_lo = lo;
        c->last_hi = hi;
        if (!c->pdl && !c->err_clean)  // (the gp_replan graph resets it in K1 phase 1)
            CUDA_TRY(cudaMemsetAsync(c->err_idx.p, 0xFF, sizeof(unsigned long long), s));  // = ~0
    }
    ArgminScratch S;
    c->err_clean = false;  // every branch below but the plain sweep may write it
    DevInst I = c->view();
    // table flags (error entries, overflow) force the status-tracking kernel;
    // while the async read-back is pending, launch the fast kernel with a
    // device-side check plus a generic fix-up that runs only if flagged
    const int fl = known_flags(c);
    bool generic = fl > 0 || k < 3 || c->force_mode == 3 || c->nb > 4;
    const bool pending = fl < 0 && !generic;
    const uint32_t* dflags = pending ? c->flagsbuf.p : nullptr;
    unsigned long long grid;
    // fast-path kernel variant by shared-memory fit (see k3_argmin)
    size_t ntri = (size_t)c->n * (c->n + 1) / 2;
    size_t nxp = (size_t)((c->n + 1) & ~1);
    size_t smem0 = 16 + (((size_t)(c->n + 1) * (k + 1) * 8 + 15) & ~(size_t)15);
    size_t smem1 = smem0 + ntri * 16 + (c->n + 1) * 16 + 3 * nxp * 8 + (size_t)c->n * 16;
    size_t smem2 = smem1 + ntri * 16;
    int mode = smem2 <= (size_t)c->smem_max ? 2 : (smem1 <= (size_t)c->smem_max ? 1 : 0);
    if (c->force_mode >= 0 && c->force_mode < mode) mode = c->force_mode;
    size_t smem = mode == 2 ? smem2 : (mode == 1 ? smem1 : smem0);
    static const K3Fn table[3][4] = {
        {k3_argmin<0, 1>, k3_argmin<0, 2>, k3_argmin<0, 3>, k3_argmin<0, 4>},
        {k3_argmin<1, 1>, k3_argmin<1, 2>, k3_argmin<1, 3>, k3_argmin<1, 4>},
        {k3_argmin<2, 1>, k3_argmin<2, 2>, k3_argmin<2, 3>, k3_argmin<2, 4>}};
    K3Fn kern = generic ? nullptr
                        : (c->verify ? pick_argmin_verify(mode, c->nb) : table[mode][c->nb - 1]);
    if (c->verify) G.vs = c->vs;
    if (!generic && lo == 0 && hi == total && hi > 0 && c->sweep_ok && c->force_mode != 4) {
        c->last_generic = false;
        CUDA_TRY(c->blk.ensure(1));
        int st = launch_sweep(c, G, 0, (unsigned long long)c->nm * G.NP, mode, dflags);
        if (st != GP_OK) return st;
        if (!pending) {
            c->err_clean = !c->pdl;  // the sweep never writes err_idx
            return st;
        }
        return launch_fixup(c, G);
    }
    // a range inside one batch block holding >= 2 whole (micro, order) blocks:
    // those through the sweep (that batch index only), the edge pieces through
    // the tile kernel, each key into its own slot, then one combine
    // (GP_K3_SPLIT=0 disables)
    bool split = top && !generic && !pending && c->sweep_ok && c->force_mode < 0 && !c->pdl &&
                 hi > lo;
    if (split) if (const char* e = getenv("GP_K3_SPLIT")) split = atoi(e) != 0;
    if (split) {
        const unsigned long long per_b = (unsigned long long)c->nm * G.NP;
        const unsigned long long bblk = per_b * G.NC;
        const unsigned long long b = lo / bblk;
        const unsigned long long f0 = (lo + G.NC - 1) / G.NC, f1 = hi / G.NC;  // whole blocks
        if ((hi - 1) / bblk == b && f1 >= f0 + 2) {
            c->last_generic = false;
            CUDA_TRY(c->blk.ensure(1));
            int st = launch_sweep(c, G, f0 - b * per_b, f1 - b * per_b, mode, nullptr, 1, (int)b, 0);
            if (st != GP_OK) return st;
            int nslot = 1;
            if (lo < f0 * G.NC) {
                st = range_async(c, lo, f0 * G.NC, nslot++);
                if (st != GP_OK) return st;
            }
            if (f1 * G.NC < hi) {
                st = range_async(c, f1 * G.NC, hi, nslot++);
                if (st != GP_OK) return st;
            }
            if (nslot > 1) {
                k_key_combine<<<1, 1, 0, s>>>(reinterpret_cast<Key*>(c->result.p), nslot);
                CUDA_TRY(cudaGetLastError());
            }
            c->last_geom = G;
            c->last_generic = false;
            c->err_clean = !c->pdl;  // neither kernel writes err_idx
            return GP_OK;
        }
    }
    if (hi == lo) {
        generic = true;
        grid = 1;
    } else if (generic) {
        grid = (hi - lo + 255) / 256;
        unsigned long long gmax = (unsigned long long)c->n_sms * 16;  // grid-stride
        if (grid > gmax) grid = gmax;
    } else {
        int per_sm = 0;
        { int st_ = kernel_slots(c, (const void*)kern, K3_THREADS, smem, &per_sm);
          if (st_ != GP_OK) return st_; }
        unsigned long long resident = (unsigned long long)(per_sm > 0 ? per_sm : 1) * c->n_sms;
        // items = (micro index, order); a range inside one batch block touches
        // a contiguous run of them, a wider range all of them
        unsigned long long per_b = (unsigned long long)c->nm * G.NP;
        unsigned long long blk_lo = lo / G.NC, blk_hi = (hi - 1) / G.NC;  // (bm, perm) blocks
        unsigned long long item_first, items;
        if (blk_lo / per_b == blk_hi / per_b) {
            item_first = blk_lo % per_b;
            items = blk_hi % per_b - item_first + 1;
        } else {
            item_first = 0;
            items = per_b;
        }
        // CTAs per item: fill the resident slots, at most one per 8 tiles
        unsigned long long tiles_per_item = (G.NC + K3_TILE - 1) / K3_TILE;
        unsigned long long cpi = items >= resident ? 1 : resident / items;
        unsigned long long cap = (tiles_per_item + 7) / 8;
        if (cpi > cap) cpi = cap;
        if (cpi < 1) cpi = 1;
        G.item0 = item_first;
        G.chunk = 0;
        G.chunks_per_item = cpi;
        grid = items * cpi;
        if (c->item_ctr.cap < items || !c->item_ctr.p) c->ctr_armed = 0;  // (re)allocation
        CUDA_TRY(c->item_ctr.ensure(items));
        if (!c->pdl && items > c->ctr_armed) {  // (k3_argmin re-arms the ones it used)
            CUDA_TRY(cudaMemsetAsync(c->item_ctr.p, 0, items * sizeof(unsigned int), s));
            c->ctr_armed = items;
        }
        G.item_ctr = c->item_ctr.p;
        int ts = ensure_tiles(c);
        if (ts != GP_OK) return ts;
        G.tiles = c->tiles_ok ? c->tiles.p : nullptr;
    }
    c->last_generic = generic;
    if (grid > 0x7fffffffull) return fail(GP_ERR_INPUT, "range too large for one launch");
    CUDA_TRY(c->blk.ensure(grid));
    S.blk = c->blk.p;
    S.counter = c->counter.p + slot;
    S.result = c->result.p + slot;
    S.err = nullptr;
    S.err_idx = c->err_idx.p;
    c->last_geom = G;
    if (generic) {
        if (hi == lo) G.hi = G.lo;  // one empty CTA writes the neutral key
        k3_argmin_generic<<<(unsigned)grid, 256, 0, s>>>(I, G, S, nullptr);
    } else {
        kern<<<(unsigned)grid, K3_THREADS, smem, s>>>(I, G, S, c->binom.p, dflags);
        CUDA_TRY(cudaGetLastError());
        if (pending) return launch_fixup(c, G);
        c->err_clean = !c->pdl;  // the tile kernel never writes err_idx
    }
    CUDA_TRY(cudaGetLastError());
    return GP_OK;
}

static void h_unrank_perm(int k, unsigned long long r, uint8_t* perm) {
    uint8_t pool[GP_MAX_STAGES];
    for (int i = 0; i < k; ++i) pool[i] = (uint8_t)i;
    int left = k;
    for (int i = 0; i < k; ++i) {
        unsigned long long f = h_fact(k - 1 - i);
        unsigned long long q = r / f;
        r %= f;
        perm[i] = pool[q];
        for (int j = (int)q; j + 1 < left; ++j) pool[j] = pool[j + 1];
        --left;
    }
}

static void h_unrank_counts(int n, int k, unsigned long long r, uint8_t* counts) {
    int prev = 0;
    for (int j = 1; j < k; ++j) {
        for (int q = prev + 1;; ++q) {
            unsigned long long cnt = h_binom(n - q - 1, k - 1 - j);
            if (r < cnt) { counts[j - 1] = (uint8_t)(q - prev); prev = q; break; }
            r -= cnt;
        }
    }
    counts[k - 1] = (uint8_t)(n - prev);
}

int gp_argmin_fetch(gp_ctx* c, gp_best* out) {
    if (!c || !c->loaded || !out) return fail(GP_ERR_INPUT, "context not loaded");
    CUDA_TRY(cudaSetDevice(c->device));
    Key r;
    unsigned long long err;
    CUDA_TRY(cudaMemcpyAsync(&r, c->result.p, sizeof(Key), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaMemcpyAsync(&err, c->err_idx.p, sizeof(err), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    memset(out, 0, sizeof(*out));
    const RangeGeom& G = c->last_geom;
    out->k = (uint32_t)G.k;
    out->evaluated = c->last_hi - c->last_lo;
    if (err != ~0ull) {
        int code = (int)(err & 15ull);
        out->index = err >> 4;  // first erroring candidate (enumeration order)
        return fail(code, "candidate %llu raises status %d", err >> 4, code);
    }
    if (r.tie == ~0ull) return fail(GP_ERR_NO_FEASIBLE, "empty candidate range");
    unsigned long long bm = r.tie % (unsigned long long)G.nbm;
    unsigned long long pc = r.tie / (unsigned long long)G.nbm;
    unsigned long long comp = pc % G.NC, perm = pc / G.NC;
    out->cost = r.cost;
    out->index = (bm * G.NP + perm) * G.NC + comp;
    out->batch_index = (uint32_t)(bm / c->nm);
    out->micro_index = (uint32_t)(bm % c->nm);
    h_unrank_perm(G.k, perm, out->order);
    h_unrank_counts(c->n, G.k, comp, out->counts);
    return GP_OK;
}

int gp_argmin_range(gp_ctx* c, uint64_t lo, uint64_t hi, gp_best* out) {
    int st = gp_argmin_range_async(c, lo, hi);
    if (st != GP_OK) return st;
    return gp_argmin_fetch(c, out);
}

int gp_argmin_bnb_async(gp_ctx* c) {
    if (c) { c->ctr_armed = 0; c->err_clean = false; }  // launches below skip neither reset
    if (!c || !c->loaded) return fail(GP_ERR_INPUT, "context not loaded");
    const int k = c->F, n = c->n;
    uint64_t total;
    { int st_ = gp_space_size(c, &total); if (st_ != GP_OK) return st_; }
    int fl = known_flags(c);
    if (fl < 0) {
        CUDA_TRY(cudaEventSynchronize(c->flags_ev));
        fl = known_flags(c);
    }
    if (fl != 0 || k < 2 || total == 0)  // error entries / trivial spaces: exhaustive path
        return gp_argmin_range_async(c, 0, total);
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    RangeGeom R;
    memset(&R, 0, sizeof(R));
    R.k = k; R.nbm = c->nb * c->nm; R.NC = h_binom(n - 1, k - 1); R.NP = h_fact(k);
    R.lo = 0; R.hi = total; R.nm = c->nm;
    c->last_geom = R;
    c->last_lo = 0;
    c->last_hi = total;
    const unsigned long long items = (unsigned long long)R.nbm * R.NP;
    if (items > 0x7fffffffull) return fail(GP_ERR_INPUT, "too many items for one launch");
    CUDA_TRY(c->gbest.ensure(1));
    // all-ones bits: above every finite cost as u64, a NaN bound as double
    // (prunes nothing until a finite cost is found)
    CUDA_TRY(cudaMemsetAsync(c->gbest.p, 0xFF, sizeof(unsigned long long), s));
    CUDA_TRY(cudaMemsetAsync(c->err_idx.p, 0xFF, sizeof(unsigned long long), s));
    CUDA_TRY(c->blk.ensure(items > 4096 ? items : 4096));
    ArgminScratch S;
    S.blk = c->blk.p; S.counter = c->counter.p; S.result = c->result.p; S.err = nullptr;
    S.err_idx = c->err_idx.p;
    BnbGeom G;
    G.k = k; G.nbm = R.nbm; G.NC = R.NC; G.NP = R.NP; G.gbest = c->gbest.p;
    DevInst I = c->view();
    const size_t smem = (size_t)k * (n + 1) * sizeof(double);
    k4_bnb<<<(unsigned)items, 32, smem, s>>>(I, G, S, c->binom.p);
    CUDA_TRY(cudaGetLastError());
    return GP_OK;
}

int gp_argmin_items_async(gp_ctx* c, uint64_t item_lo, uint64_t item_hi) {
    if (c) { c->ctr_armed = 0; c->err_clean = false; }  // launches below skip neither reset
    if (!c || !c->loaded) return fail(GP_ERR_INPUT, "context not loaded");
    const int k = c->F;
    uint64_t total;
    { int st_ = gp_space_size(c, &total); if (st_ != GP_OK) return st_; }
    const unsigned long long NP = h_fact(k), NC = h_binom(c->n - 1, k - 1);
    const unsigned long long n_items = total ? (unsigned long long)c->nm * NP : 0;
    if (item_hi > n_items) item_hi = n_items;
    if (item_lo > item_hi) item_lo = item_hi;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    RangeGeom G;
    memset(&G, 0, sizeof(G));
    G.k = k;
    G.nbm = c->nb * c->nm;
    G.NC = NC;
    G.NP = NP;
    G.nm = c->nm;
    G.items_mode = 1;
    G.it_lo = item_lo;
    G.it_span = item_hi > item_lo ? item_hi - item_lo : 1;
    G.lo = 0;
    G.hi = (unsigned long long)c->nb * (item_hi - item_lo) * NC;
    if (c->verify) G.vs = c->vs;
    c->last_lo = 0;
    c->last_hi = G.hi;
    c->last_geom = G;
    CUDA_TRY(cudaMemsetAsync(c->err_idx.p, 0xFF, sizeof(unsigned long long), s));
    const int fl = known_flags(c);
    const bool generic = fl > 0 || k < 3 || c->force_mode == 3 || c->force_mode == 4 ||
                         c->nb > 4 || !c->sweep_ok || G.hi == 0;
    if (!generic) {
        int mode = c->force_mode >= 0 && c->force_mode <= 2 ? c->force_mode : 2;
        const uint32_t* dflags = fl < 0 ? c->flagsbuf.p : nullptr;
        int st = launch_sweep(c, G, item_lo, item_hi, mode, dflags);
        if (st != GP_OK || fl >= 0) return st;
        return launch_fixup(c, G);
    }
    unsigned long long grid = G.hi ? (G.hi + 255) / 256 : 1;
    unsigned long long gmax = (unsigned long long)c->n_sms * 16;
    if (grid > gmax) grid = gmax;
    ArgminScratch S;
    S.blk = c->blk.p;
    S.counter = c->counter.p;
    S.result = c->result.p;
    S.err = nullptr;
    S.err_idx = c->err_idx.p;
    DevInst I = c->view();
    k3_argmin_generic<<<(unsigned)grid, 256, 0, s>>>(I, G, S, nullptr);
    CUDA_TRY(cudaGetLastError());
    return GP_OK;
}

// arg-min + on-device winner detail + D2H of the SolveOut record (no sync)
static int enqueue_solve(gp_ctx* c, uint64_t lo, uint64_t hi) {
    int st = gp_argmin_range_async(c, lo, hi);
    if (st != GP_OK) return st;
    const RangeGeom& G = c->last_geom;
    CUDA_TRY(c->dsolve.ensure(1));
    DevInst I = c->view();
    // inside the gp_replan graph the record goes straight to the mapped pinned
    // buffer (no D2H node); elsewhere to device memory + an async copy
    SolveOut* dst = c->pdl ? c->d_hsolve : c->dsolve.p;
    CUDA_TRY(launch_k(k_solve_detail, 1, 32, 0, c->stream, c->pdl, I, G.k, G.NC, G.NP, G.nbm,
                      (const Key*)c->result.p, (const unsigned long long*)c->err_idx.p,
                      (const unsigned long long*)c->binom.p, dst, c->pdl ? 1 : 0,
                      c->pdl ? c->d_seq.p : (unsigned long long*)nullptr));
    if (c->pdl) return GP_OK;
    CUDA_TRY(cudaMemcpyAsync(c->h_solve, c->dsolve.p, sizeof(SolveOut), cudaMemcpyDeviceToHost,
                             c->stream));
    return GP_OK;
}

// decode the SolveOut record that landed in pinned memory
static int finish_solve(gp_ctx* c, gp_best* best, gp_plan_info* info) {
    const RangeGeom& G = c->last_geom;
    const SolveOut& o = *c->h_solve;
    c->flags = o.flags;  // the table flags as the detail kernel saw them
    c->flags_known = true;
    memset(best, 0, sizeof(*best));
    best->k = (uint32_t)G.k;
    best->evaluated = c->last_hi - c->last_lo;
    if (o.err != ~0ull) {
        int code = (int)(o.err & 15ull);
        return fail(code, "candidate %llu raises status %d", o.err >> 4, code);
    }
    if (o.key.tie == ~0ull) return fail(GP_ERR_NO_FEASIBLE, "empty candidate range");
    unsigned long long bmv = o.key.tie % (unsigned long long)G.nbm;
    unsigned long long pc = o.key.tie / (unsigned long long)G.nbm;
    best->cost = o.key.cost;
    best->index = (bmv * G.NP + pc / G.NC) * G.NC + pc % G.NC;
    best->batch_index = (uint32_t)(bmv / c->nm);
    best->micro_index = (uint32_t)(bmv % c->nm);
    memcpy(best->order, o.order, sizeof(best->order));
    memcpy(best->counts, o.counts, sizeof(best->counts));
    if (info) *info = o.info;
    if (o.status != GP_OK) return fail(o.status, "winner raises status %d", o.status);
    return GP_OK;
}

int gp_solve(gp_ctx* c, uint64_t lo, uint64_t hi, gp_best* best, gp_plan_info* info) {
    if (!c || !c->loaded || !best) return fail(GP_ERR_INPUT, "context not loaded");
    int st = enqueue_solve(c, lo, hi);
    if (st != GP_OK) return st;
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return finish_solve(c, best, info);
}

// shape of an instance: everything the arena layout and the launch geometry
// depend on (a CUDA graph captured for one shape replays for any instance of
// the same shape)
static void instance_shape(const gp_instance* in, unsigned long long* key) {
    key[0] = in->n_layers; key[1] = in->n_devices; key[2] = in->n_fgs;
    key[3] = in->n_batch; key[4] = in->n_micro;
    key[5] = in->fg_member_offset[in->n_fgs];
    key[6] = in->fg_sg_offset[in->n_fgs];
    key[7] = in->sg_member_offset[in->fg_sg_offset[in->n_fgs]];
    unsigned long long h = 1469598103934665603ull;  // group structure (CSR offsets)
    for (uint32_t f = 0; f <= in->n_fgs; ++f) {
        h = (h ^ in->fg_member_offset[f]) * 1099511628211ull;
        h = (h ^ in->fg_sg_offset[f]) * 1099511628211ull;
    }
    for (uint32_t g = 0; g <= in->fg_sg_offset[in->n_fgs]; ++g)
        h = (h ^ in->sg_member_offset[g]) * 1099511628211ull;
    for (uint32_t i = 0; i < in->n_batch; ++i) h = (h ^ (unsigned long long)in->batch[i]) * 1099511628211ull;
    for (uint32_t i = 0; i < in->n_micro; ++i) h = (h ^ (unsigned long long)in->micro[i]) * 1099511628211ull;
    key[8] = h;
}

static void replan_key(const gp_ctx* c, const gp_instance* in, unsigned long long* key) {
    instance_shape(in, key);
    memcpy(&key[9], &in->bottleneck_factor, sizeof(double));
    key[10] = (unsigned long long)(long long)c->force_mode;
}

static inline double now_us() {
    return std::chrono::duration<double, std::micro>(
               std::chrono::steady_clock::now().time_since_epoch()).count();
}

int gp_replan(gp_ctx* c, const gp_instance* in, gp_best* best, gp_plan_info* info) {
    if (c) { c->ctr_armed = 0; c->err_clean = false; }  // launches below skip neither reset
    if (!c || !in || !best) return fail(GP_ERR_INPUT, "null argument");
    const double h0 = c->diag_timing ? now_us() : 0.0;
    unsigned long long key[11];
    replan_key(c, in, key);
    const bool same = c->graph_exec && memcmp(key, c->graph_key, sizeof(key)) == 0 &&
                      memcmp(key, c->loaded_key, sizeof(key)) == 0 &&
                      c->graph_gen == __atomic_load_n(&g_alloc_gen, __ATOMIC_RELAXED);
    cudaStream_t s = c->stream;
    if (!same) {
        // first instance of this shape: regular load (allocations, helpers),
        // then capture H2D + K1 + K3 + detail + D2H as one graph
        int st = gp_ctx_load(c, in);
        if (st != GP_OK) return st;
        CUDA_TRY(cudaStreamSynchronize(s));
        if (c->graph_exec) { cudaGraphExecDestroy(c->graph_exec); c->graph_exec = nullptr; }
        uint64_t total;
        st = gp_space_size(c, &total);
        if (st != GP_OK) return st;
        // make every buffer the graph touches exist before capturing
        CUDA_TRY(c->dsolve.ensure(1));
        CUDA_TRY(c->item_ctr.ensure((size_t)c->nm * h_fact(c->F) + 1));
        CUDA_TRY(c->d_seq.ensure(1));
        CUDA_TRY(cudaMemsetAsync(c->d_seq.p, 0, sizeof(unsigned long long), s));
        CUDA_TRY(cudaStreamSynchronize(s));
        c->solve_seq = 0;
        c->h_solve->seq = 0;
        c->capturing = true;
        CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
        // the instance arena moves host -> device by a kernel reading the mapped
        // pinned buffer (no copy-engine node; K1 phase 1 follows by PDL)
        const unsigned long long n16 = (c->arena_bytes + 15) / 16;
        const unsigned pull_blocks = (unsigned)((n16 + 255) / 256 < 148 ? (n16 + 255) / 256 : 148);
        cudaError_t ce = launch_k(k_arena_pull, pull_blocks > 0 ? pull_blocks : 1u, 256, 0, s, false,
                                  (const uint4*)c->d_harena, (uint4*)c->arena.p, n16);
        int st2 = ce == cudaSuccess ? GP_OK : fail(GP_ERR_CUDA, "capture: %s", cudaGetErrorString(ce));
        if (st2 == GP_OK) {
            // H2D -> K1 phase 1 (resets flags, err_idx, item counters) -> phase 2
            // -> sweep -> fix-up -> detail (PDL chain; the table flags return
            // inside the SolveOut record) -> D2H
            DevInst I = c->view();
            const int gw_blocks = (c->F * c->F + 3) / 4;
            K1Reset R = {c->err_idx.p, c->item_ctr.p, (unsigned)((size_t)c->nm * h_fact(c->F))};
            ce = launch_k(k1_phase1, 5 + c->F + gw_blocks, 128, 0, s, true, I, R);
            long long ns = (long long)c->F * (c->n + 1) * (c->n + 1);
            long long nx = (long long)c->nm * c->F * c->F * c->n;
            if (ce == cudaSuccess)
                ce = launch_k(k1_phase2, (unsigned)((ns + nx + 127) / 128), 128, 0, s, true, I, ns);
#if defined(GP_TIMELINE)
            if (getenv("GP_K1_TWICE") && ce == cudaSuccess)  // icache experiment
                ce = launch_k(k1_phase2, (unsigned)((ns + nx + 127) / 128), 128, 0, s, true, I, ns);
#endif
            if (ce != cudaSuccess) st2 = fail(GP_ERR_CUDA, "capture: %s", cudaGetErrorString(ce));
            c->flags_known = false;
            c->pdl = true;
            if (st2 == GP_OK) st2 = enqueue_solve(c, 0, total);
            c->pdl = false;
        }
        cudaGraph_t g = nullptr;
        cudaError_t ee = cudaStreamEndCapture(s, &g);
        c->capturing = false;
        if (st2 != GP_OK) { if (g) cudaGraphDestroy(g); return st2; }
        if (ee != cudaSuccess) return fail(GP_ERR_CUDA, "graph capture: %s", cudaGetErrorString(ee));
        ee = cudaGraphInstantiate(&c->graph_exec, g, 0);
        cudaGraphDestroy(g);
        if (ee != cudaSuccess) { c->graph_exec = nullptr; return fail(GP_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(ee)); }
        memcpy(c->graph_key, key, sizeof(key));
        c->graph_gen = __atomic_load_n(&g_alloc_gen, __ATOMIC_RELAXED);
        c->graph_geom = c->last_geom;
        c->graph_lo = c->last_lo;
        c->graph_hi = c->last_hi;
    } else {
        // same shape: refill the pinned arena in place (same offsets)
        if (c->arena_ev) CUDA_TRY(cudaEventSynchronize(c->arena_ev));
        const uint32_t n = in->n_layers, D = in->n_devices, F = in->n_fgs;
        const size_t DD = (size_t)D * D;
        const uint32_t nsg = in->fg_sg_offset[F];
        const void* src[23] = {in->fwd_flops, in->bwd_input_flops, in->bwd_weight_flops,
                               in->activation_out_bytes, in->param_bytes, in->batch, in->micro,
                               in->p_c, in->memory_bytes, in->id_rank, in->p_t, in->latency,
                               in->bandwidth, in->fg_member_offset, in->fg_members, in->fg_capacity,
                               in->fg_min_bw, in->fg_min_bw, in->fg_has_min_bw, in->fg_sg_offset,
                               in->sg_member_offset, in->sg_members, in->sg_capacity};
        const size_t bytes[23] = {n * 8ull, n * 8ull, n * 8ull, n * 8ull, n * 8ull,
                                  in->n_batch * 8ull, in->n_micro * 8ull, D * 8ull, D * 8ull,
                                  D * 4ull, DD * 8, DD * 8, DD * 8, (F + 1) * 4ull,
                                  in->fg_member_offset[F] * 4ull, F * 8ull, F * 8ull, F * 8ull,
                                  (size_t)F, (F + 1) * 4ull, (nsg + 1) * 4ull,
                                  in->sg_member_offset[nsg] * 4ull, nsg * 8ull};
        size_t off = 0;
        for (int i = 0; i < 23; ++i) {
            if (bytes[i]) memcpy(c->h_arena + off, src[i], bytes[i]);
            off += (bytes[i] + 15) & ~(size_t)15;
        }
        c->bf = in->bottleneck_factor;
        c->last_geom = c->graph_geom;
        c->last_lo = c->graph_lo;
        c->last_hi = c->graph_hi;
    }
    const double h1 = c->diag_timing ? now_us() : 0.0;
    if (c->diag_timing) CUDA_TRY(cudaEventRecord(c->t_ev0, s));
    ++c->tables_gen;  // the graph rebuilds the tables
    CUDA_TRY(cudaGraphLaunch(c->graph_exec, s));
    CUDA_TRY(cudaEventRecord(c->arena_ev, s));
    if (c->diag_timing) CUDA_TRY(cudaEventRecord(c->t_ev1, s));
    const double h2 = c->diag_timing ? now_us() : 0.0;
    const unsigned long long want = ++c->solve_seq;
    bool landed = false;
    if (!c->diag_timing) {
        // the detail kernel publishes the record with a sequence number in
        // mapped memory: poll it (the graph's last kernel may still be
        // exiting); a graph that never publishes falls through to the
        // stream synchronisation, which reports its error
        const volatile unsigned long long* seq = &c->h_solve->seq;
        const double t_end = now_us() + 20000.0;
        for (unsigned spin = 0;; ++spin) {
            if (*seq == want) { landed = true; break; }
            if ((spin & 1023u) == 1023u && now_us() > t_end) break;
        }
        std::atomic_thread_fence(std::memory_order_acquire);
    }
    if (!landed) CUDA_TRY(cudaStreamSynchronize(s));
    const double h3 = c->diag_timing ? now_us() : 0.0;
    if (c->diag_timing) CUDA_TRY(cudaEventElapsedTime(&c->last_graph_ms, c->t_ev0, c->t_ev1));
    c->flags_known = false;
    c->loaded = true;
    const int rs = finish_solve(c, best, info);
    if (c->diag_timing) {
        const double h4 = now_us();
        c->host_us[0] = h1 - h0; c->host_us[1] = h2 - h1;
        c->host_us[2] = h3 - h2; c->host_us[3] = h4 - h3;
    }
    return rs;
}

int gp_plan_detail(gp_ctx* c, uint32_t k, const uint8_t* order, const uint8_t* counts, uint32_t bm,
                   gp_plan_info* out) {
    if (!c || !c->loaded || !out) return fail(GP_ERR_INPUT, "context not loaded");
    if (k < 1 || k > GP_MAX_STAGES || bm >= (uint32_t)(c->nb * c->nm))
        return fail(GP_ERR_INPUT, "bad candidate");
    int sum = 0;
    unsigned seen = 0;
    for (uint32_t s = 0; s < k; ++s) {
        if (order[s] >= c->F || ((seen >> order[s]) & 1u) || counts[s] == 0)
            return fail(GP_ERR_INPUT, "stage order must use distinct groups and positive counts");
        seen |= 1u << order[s];
        sum += counts[s];
    }
    if (sum > c->n) return fail(GP_ERR_INPUT, "counts exceed the layer count");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    CUDA_TRY(c->b_order.ensure(GP_MAX_STAGES));
    CUDA_TRY(c->b_counts.ensure(GP_MAX_STAGES));
    CUDA_TRY(c->info.ensure(1));
    CUDA_TRY(c->dstatus.ensure(1));
    CUDA_TRY(cudaMemcpyAsync(c->b_order.p, order, k, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->b_counts.p, counts, k, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemsetAsync(c->info.p, 0, sizeof(gp_plan_info), s));
    DevInst I = c->view();
    k_plan_detail<<<1, 32, 0, s>>>(I, (int)k, c->b_order.p, c->b_counts.p, (int)bm, c->info.p,
                                   c->dstatus.p);
    CUDA_TRY(cudaGetLastError());
    int status = 0;
    CUDA_TRY(cudaMemcpyAsync(out, c->info.p, sizeof(gp_plan_info), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&status, c->dstatus.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (status != GP_OK) return fail(status, "candidate raises status %d", status);
    return GP_OK;
}

__global__ void k_group_info(DevInst I, int f, gp_group_info* out) {
    if (threadIdx.x != 0) return;
    int m0 = I.fg_off[f], m1 = I.fg_off[f + 1];
    int s0 = I.fg_sg_off[f], s1 = I.fg_sg_off[f + 1];
    out->n_members = (uint32_t)(m1 - m0);
    out->n_sgs = (uint32_t)(s1 - s0);
    out->tp_ok = I.g_tp_ok[f];
    for (int x = m0; x < m1; ++x) { out->tp_row[x - m0] = I.g_rf[x]; out->tp_col[x - m0] = I.g_cf[x]; }
    for (int g = s0; g < s1; ++g) out->dp_fraction[g - s0] = I.g_dp[g];
}

int gp_group_splits(gp_ctx* c, uint32_t f, gp_group_info* out) {
    if (!c || !c->loaded || !out || f >= (uint32_t)c->F) return fail(GP_ERR_INPUT, "bad group");
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(c->ginfo.ensure(1));
    CUDA_TRY(cudaMemsetAsync(c->ginfo.p, 0, sizeof(gp_group_info), c->stream));
    DevInst I = c->view();
    k_group_info<<<1, 32, 0, c->stream>>>(I, (int)f, c->ginfo.p);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out, c->ginfo.p, sizeof(gp_group_info), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return GP_OK;
}

// ---- diagnostics: FP64 add issue-rate microbenchmark --------------------------------
// 8 independent DADD chains per thread so the FP64 pipe, not latency, bounds it.
__global__ void k_fp64_peak(double* sink, int iters, double step) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
           a6 = a0 + 6, a7 = a0 + 7;
    for (int i = 0; i < iters; ++i) {
        a0 = a0 + step; a1 = a1 + step; a2 = a2 + step; a3 = a3 + step;
        a4 = a4 + step; a5 = a5 + step; a6 = a6 + step; a7 = a7 + step;
    }
    double r = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (r == 12345.678) sink[blockIdx.x] = r;  // never true; keeps the chains live
}

int gp_sim_1f1b_device(gp_ctx* c, const gp_timing* d_timings, uint64_t n, uint32_t iterations,
                       double* d_makespan, uint8_t* d_status) {
    if (!c) return fail(GP_ERR_INPUT, "null context");
    if (n == 0) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    const int tpb = item_tpb(c, n);
    k5_sim_1f1b<<<(unsigned)((n + tpb - 1) / tpb), tpb, 0, c->stream>>>(
        d_timings, (long long)n, GP_POLICY_1F1B, (int)iterations, nullptr, nullptr, d_makespan,
        d_status);
    CUDA_TRY(cudaGetLastError());
    return GP_OK;
}

// Timings grouped by (stage count, micro-batch count): a permutation in
// c->k5_perm (nullptr when not worth it; GP_K5_SORT=0 disables)
static int k5_sort_timings(gp_ctx* c, const gp_timing* d_T, uint64_t n, uint32_t** perm) {
    static const int sort_on = [] { const char* e = getenv("GP_K5_SORT"); return e ? atoi(e) : 1; }();
    *perm = nullptr;
    if (!sort_on || n < 1024 || n >= (1ull << 32)) return GP_OK;
    cudaStream_t s = c->stream;
    CUDA_TRY(c->k5_perm.ensure(n));
    CUDA_TRY(c->k5_hist.ensure(K5_NKEYS));
    CUDA_TRY(cudaMemsetAsync(c->k5_hist.p, 0, K5_NKEYS * sizeof(uint32_t), s));
    unsigned hb = (unsigned)((n + 255) / 256);
    if (hb > 2u * (unsigned)c->n_sms) hb = 2u * (unsigned)c->n_sms;
    k5_key_hist<<<hb, 256, 0, s>>>((long long)n, d_T, c->k5_hist.p);
    k5_key_scan<<<1, 256, 0, s>>>(c->k5_hist.p);
    k5_key_scatter<<<(unsigned)((n + 255) / 256), 256, 0, s>>>((long long)n, d_T, c->k5_hist.p, c->k5_perm.p);
    CUDA_TRY(cudaGetLastError());
    *perm = c->k5_perm.p;
    return GP_OK;
}

// Validation shared by the trace-taking simulators.
static int check_traces(const gp_trace* traces, uint32_t n_traces, const uint32_t* trace_index,
                        uint64_t n) {
    if (traces && trace_index)
        for (uint64_t i = 0; i < n; ++i)
            if (trace_index[i] >= n_traces) return fail(GP_ERR_INPUT, "trace index out of range");
    if (traces)
        for (uint32_t t = 0; t < n_traces; ++t)
            for (int b = 0; b < GP_MAX_STAGES; ++b)
                if (traces[t].n_points[b] > GP_MAX_BREAKPOINTS)
                    return fail(GP_ERR_INPUT, "trace %u link %d: too many breakpoints", t, b);
    return GP_OK;
}

int gp_simulate(gp_ctx* c, const gp_timing* timings, uint64_t n, uint32_t policy,
                uint32_t iterations, const gp_trace* traces, uint32_t n_traces,
                const uint32_t* trace_index, double* makespan, uint8_t* status) {
    if (!c) return fail(GP_ERR_INPUT, "null context");
    if (policy > GP_POLICY_ZB_COMPACT) return fail(GP_ERR_INPUT, "unknown policy %u", policy);
    if (n == 0) return GP_OK;
    if (traces && n_traces == 0) traces = nullptr;
    { int st_ = check_traces(traces, n_traces, trace_index, n); if (st_ != GP_OK) return st_; }
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    CUDA_TRY(c->s_tim.ensure(n));
    CUDA_TRY(c->s_ms.ensure(n));
    CUDA_TRY(c->s_st.ensure(n));
    CUDA_TRY(cudaMemcpyAsync(c->s_tim.p, timings, n * sizeof(gp_timing), cudaMemcpyHostToDevice, s));
    gp_trace* d_tr = nullptr;
    uint32_t* d_ti = nullptr;
    if (traces) {
        CUDA_TRY(c->s_traces.ensure(n_traces));
        CUDA_TRY(cudaMemcpyAsync(c->s_traces.p, traces, n_traces * sizeof(gp_trace),
                                 cudaMemcpyHostToDevice, s));
        d_tr = c->s_traces.p;
        if (trace_index) {
            CUDA_TRY(c->s_tidx.ensure(n));
            CUDA_TRY(cudaMemcpyAsync(c->s_tidx.p, trace_index, n * sizeof(uint32_t),
                                     cudaMemcpyHostToDevice, s));
            d_ti = c->s_tidx.p;
        }
    }
    const int tpb = item_tpb(c, n);
    uint32_t* perm = nullptr;
    { int st_ = k5_sort_timings(c, c->s_tim.p, n, &perm); if (st_ != GP_OK) return st_; }
    k5_sim_1f1b<<<(unsigned)((n + tpb - 1) / tpb), tpb, 0, s>>>(c->s_tim.p, (long long)n, (int)policy,
                                                           (int)iterations, d_tr, d_ti, c->s_ms.p,
                                                           c->s_st.p, perm);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(makespan, c->s_ms.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(status, c->s_st.p, n, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return GP_OK;
}

// Shared set-up of the full simulator (K5 full): argument checks, timings /
// traces H2D, queue-scratch sizing from the largest timing of the batch.
struct SimPlan {
    gp_sim_options opt;
    int wcap, lcap, smax;
    size_t nlinks, per;
    uint64_t chunk;
    gp_trace* d_tr;
    uint32_t* d_ti;
};

static int sim_prepare(gp_ctx* c, const gp_timing* timings, uint64_t n, uint32_t policy,
                       uint32_t iterations, const gp_trace* traces, uint32_t n_traces,
                       const uint32_t* trace_index, const gp_sim_options* opts, SimPlan& P) {
    if (policy > GP_POLICY_ZB_COMPACT) return fail(GP_ERR_INPUT, "unknown policy %u", policy);
    if (iterations < 1 || iterations > 0xffff) return fail(GP_ERR_INPUT, "iterations out of range");
    if (traces && n_traces == 0) traces = nullptr;
    { int st_ = check_traces(traces, n_traces, trace_index, n); if (st_ != GP_OK) return st_; }
    P.opt = gp_sim_options{0u, 0u, 1.2, 1.05};
    if (opts) P.opt = *opts;
    long long bmax = 1;
    P.smax = 1;
    for (uint64_t i = 0; i < n; ++i) {
        if (timings[i].batch > bmax) bmax = timings[i].batch;
        if ((int)timings[i].n_stages > P.smax && timings[i].n_stages <= GP_MAX_STAGES)
            P.smax = (int)timings[i].n_stages;
    }
    if (bmax >= (1ll << 24) - 2) return fail(GP_ERR_INPUT, "batch %lld too large", bmax);
    P.wcap = (int)bmax + 1;
    P.lcap = (int)(2 * bmax + 2);
    P.nlinks = (size_t)2 * (P.smax > 1 ? P.smax - 1 : 1);
    P.per = (size_t)P.smax * SIMF_SLOTS * P.wcap * sizeof(uint32_t) + 8 +
            P.nlinks * P.lcap * sizeof(unsigned long long) +
            (size_t)P.smax * SIMF_SLOTS * sizeof(SimFPool) + P.nlinks * sizeof(AdWindow);
    P.chunk = (uint64_t)((1ull << 30) / P.per);  // <= 1 GiB of queue scratch per launch
    if (P.chunk < 1) P.chunk = 1;
    if (P.chunk > n) P.chunk = n;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    CUDA_TRY(c->s_tim.ensure(n));
    CUDA_TRY(c->s_st.ensure(n));
    CUDA_TRY(c->s_wq.ensure(P.chunk * (P.per / sizeof(uint32_t) + 1)));  // queues, pools, windows
    CUDA_TRY(cudaMemcpyAsync(c->s_tim.p, timings, n * sizeof(gp_timing), cudaMemcpyHostToDevice, s));
    P.d_tr = nullptr;
    P.d_ti = nullptr;
    if (traces) {
        CUDA_TRY(c->s_traces.ensure(n_traces));
        CUDA_TRY(cudaMemcpyAsync(c->s_traces.p, traces, n_traces * sizeof(gp_trace),
                                 cudaMemcpyHostToDevice, s));
        P.d_tr = c->s_traces.p;
        if (trace_index) {
            CUDA_TRY(c->s_tidx.ensure(n));
            CUDA_TRY(cudaMemcpyAsync(c->s_tidx.p, trace_index, n * sizeof(uint32_t),
                                     cudaMemcpyHostToDevice, s));
            P.d_ti = c->s_tidx.p;
        }
    }
    return GP_OK;
}

static SimScratch sim_scratch(gp_ctx* c, const SimPlan& P, uint64_t nc) {
    SimScratch sc;
    sc.n = (long long)nc;
    sc.wcap = P.wcap;
    sc.lcap = P.lcap;
    sc.smax = P.smax;
    sc.wq = c->s_wq.p;
    // link FIFOs after the W queues, 8-byte aligned (wcap words per queue)
    size_t wwords = (size_t)P.smax * SIMF_SLOTS * P.wcap * nc;
    wwords = (wwords + 1) & ~(size_t)1;
    sc.lq = reinterpret_cast<unsigned long long*>(c->s_wq.p + wwords);
    sc.pools = reinterpret_cast<SimFPool*>(sc.lq + P.nlinks * P.lcap * nc);
    sc.win = reinterpret_cast<AdWindow*>(sc.pools + (size_t)P.smax * SIMF_SLOTS * nc);
    return sc;
}

int gp_simulate_report(gp_ctx* c, const gp_timing* timings, uint64_t n, uint32_t policy,
                       uint32_t iterations, const gp_trace* traces, uint32_t n_traces,
                       const uint32_t* trace_index, const gp_sim_options* opts,
                       gp_sim_report* report, double* iteration_ends, uint8_t* status) {
    if (!c || !timings || !report || !status) return fail(GP_ERR_INPUT, "bad arguments");
    if (n == 0) return GP_OK;
    SimPlan P;
    { int st_ = sim_prepare(c, timings, n, policy, iterations, traces, n_traces, trace_index, opts, P);
      if (st_ != GP_OK) return st_; }
    cudaStream_t s = c->stream;
    CUDA_TRY(c->s_rep.ensure(n));
    if (iteration_ends) {
        CUDA_TRY(c->s_ends.ensure(n * (uint64_t)iterations));
        CUDA_TRY(cudaMemsetAsync(c->s_ends.p, 0, n * (uint64_t)iterations * sizeof(double), s));
    }
    uint32_t* perm = nullptr;
    { int st_ = k5_sort_timings(c, c->s_tim.p, n, &perm); if (st_ != GP_OK) return st_; }
    for (uint64_t i0 = 0; i0 < n; i0 += P.chunk) {
        const uint64_t nc = (n - i0) < P.chunk ? (n - i0) : P.chunk;
        const int tpb = item_tpb(c, nc);
        if (perm)  // chunk = the permuted positions [i0, i0 + nc); timings by global index
            k5_sim_full<<<(unsigned)((nc + tpb - 1) / tpb), tpb, 0, s>>>(
                c->s_tim.p, (long long)nc, (int)policy, (int)iterations, P.d_tr, P.d_ti, P.opt,
                sim_scratch(c, P, nc), c->s_rep.p, iteration_ends ? c->s_ends.p : nullptr, c->s_st.p,
                perm + i0);
        else
            k5_sim_full<<<(unsigned)((nc + tpb - 1) / tpb), tpb, 0, s>>>(
                c->s_tim.p + i0, (long long)nc, (int)policy, (int)iterations, P.d_tr,
                P.d_ti ? P.d_ti + i0 : nullptr, P.opt, sim_scratch(c, P, nc), c->s_rep.p + i0,
                iteration_ends ? c->s_ends.p + i0 * iterations : nullptr, c->s_st.p + i0);
        CUDA_TRY(cudaGetLastError());
    }
    CUDA_TRY(cudaMemcpyAsync(report, c->s_rep.p, n * sizeof(gp_sim_report), cudaMemcpyDeviceToHost, s));
    if (iteration_ends)
        CUDA_TRY(cudaMemcpyAsync(iteration_ends, c->s_ends.p, n * (uint64_t)iterations * sizeof(double),
                                 cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(status, c->s_st.p, n, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return GP_OK;
}

int gp_simulate_schedule(gp_ctx* c, const gp_timing* timings, uint64_t n, uint32_t policy,
                         uint32_t iterations, const gp_trace* traces, uint32_t n_traces,
                         const uint32_t* trace_index, const gp_sim_options* opts,
                         const uint64_t* op_offset, gp_op* ops, const uint64_t* xfer_offset,
                         gp_transfer* transfers, const uint64_t* action_offset, gp_action* actions,
                         uint8_t* status) {
    if (!c || !timings || !op_offset || !ops || !status || (transfers && !xfer_offset) ||
        (actions && !action_offset))
        return fail(GP_ERR_INPUT, "bad arguments");
    if (n == 0) return GP_OK;
    SimPlan P;
    { int st_ = sim_prepare(c, timings, n, policy, iterations, traces, n_traces, trace_index, opts, P);
      if (st_ != GP_OK) return st_; }
    cudaStream_t s = c->stream;
    const uint64_t n_ops = op_offset[n] - op_offset[0];
    const uint64_t n_xf = transfers ? xfer_offset[n] - xfer_offset[0] : 0;
    const uint64_t n_ac = actions ? action_offset[n] - action_offset[0] : 0;
    // one staging buffer: offsets (3 x (n+1) u64), ops, transfers, actions
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t b_off = al(3 * (n + 1) * 8), b_ops = al(n_ops * sizeof(gp_op));
    const size_t b_xf = al(n_xf * sizeof(gp_transfer));
    CUDA_TRY(c->g_buf.ensure(b_off + b_ops + b_xf + n_ac * sizeof(gp_action) + 256));
    uint8_t* base = c->g_buf.p;
    unsigned long long* d_oo = reinterpret_cast<unsigned long long*>(base);
    unsigned long long* d_xo = d_oo + (n + 1);
    unsigned long long* d_ao = d_xo + (n + 1);
    gp_op* d_ops = reinterpret_cast<gp_op*>(base + b_off);
    gp_transfer* d_xf = reinterpret_cast<gp_transfer*>(base + b_off + b_ops);
    gp_action* d_ac = reinterpret_cast<gp_action*>(base + b_off + b_ops + b_xf);
    // offsets relative to the first timing
    std::vector<unsigned long long> h_off(3 * (n + 1));
    for (uint64_t i = 0; i <= n; ++i) {
        h_off[i] = op_offset[i] - op_offset[0];
        h_off[n + 1 + i] = transfers ? xfer_offset[i] - xfer_offset[0] : 0;
        h_off[2 * (n + 1) + i] = actions ? action_offset[i] - action_offset[0] : 0;
    }
    CUDA_TRY(cudaMemcpyAsync(d_oo, h_off.data(), 3 * (n + 1) * 8, cudaMemcpyHostToDevice, s));
    for (uint64_t i0 = 0; i0 < n; i0 += P.chunk) {
        const uint64_t nc = (n - i0) < P.chunk ? (n - i0) : P.chunk;
        const int tpb = item_tpb(c, nc);
        k5_sim_schedule<<<(unsigned)((nc + tpb - 1) / tpb), tpb, 0, s>>>(
            c->s_tim.p + i0, (long long)nc, (int)policy, (int)iterations, P.d_tr,
            P.d_ti ? P.d_ti + i0 : nullptr, P.opt, sim_scratch(c, P, nc), d_oo + i0, d_ops,
            d_xo + i0, transfers ? d_xf : nullptr, d_ao + i0, actions ? d_ac : nullptr,
            c->s_st.p + i0);
        CUDA_TRY(cudaGetLastError());
    }
    CUDA_TRY(cudaMemcpyAsync(ops + op_offset[0], d_ops, n_ops * sizeof(gp_op), cudaMemcpyDeviceToHost, s));
    if (transfers)
        CUDA_TRY(cudaMemcpyAsync(transfers + xfer_offset[0], d_xf, n_xf * sizeof(gp_transfer),
                                 cudaMemcpyDeviceToHost, s));
    if (actions)
        CUDA_TRY(cudaMemcpyAsync(actions + action_offset[0], d_ac, n_ac * sizeof(gp_action),
                                 cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(status, c->s_st.p, n, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return GP_OK;
}

int gp_validate_schedules(gp_ctx* c, const gp_timing* timings, uint64_t n,
                          const uint64_t* op_offset, const gp_op* ops, const double* makespan,
                          uint32_t iterations, double tol, uint32_t max_violations,
                          gp_violation* violations, uint32_t* n_violations, double* busy,
                          uint8_t* status) {
    if (!c || !timings || !op_offset || !ops || !makespan || !n_violations || !status ||
        (max_violations && !violations))
        return fail(GP_ERR_INPUT, "bad arguments");
    if (iterations < 1 || iterations > 0xffff) return fail(GP_ERR_INPUT, "iterations out of range");
    if (n == 0) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    const uint64_t n_ops = op_offset[n] - op_offset[0];
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t nq = (size_t)GP_MAX_STAGES * iterations * 3;
    const size_t o_tim = 0, o_off = o_tim + al(n * sizeof(gp_timing)), o_ms = o_off + al((n + 1) * 8);
    const size_t o_ops = o_ms + al(n * 8), o_v = o_ops + al(n_ops * sizeof(gp_op));
    const size_t o_nv = o_v + al(n * (size_t)max_violations * sizeof(gp_violation));
    const size_t o_busy = o_nv + al(n * 4), o_st = o_busy + al(n * GP_MAX_STAGES * 8);
    const size_t o_tab = o_st + al(n), o_idx = o_tab + al(n * nq * 2 * 4);
    const size_t o_srt = o_idx + al(n_ops * 4), o_lst = o_srt + al(n_ops * 4);
    const size_t o_its = o_lst + al(n_ops * 4);
    const size_t total = o_its + al(n * (size_t)GP_MAX_STAGES * iterations * sizeof(K8Iter));
    CUDA_TRY(c->g_buf.ensure(total));
    uint8_t* b = c->g_buf.p;
    std::vector<unsigned long long> h_off(n + 1);
    for (uint64_t i = 0; i <= n; ++i) h_off[i] = op_offset[i] - op_offset[0];
    CUDA_TRY(cudaMemcpyAsync(b + o_tim, timings, n * sizeof(gp_timing), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(b + o_off, h_off.data(), (n + 1) * 8, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(b + o_ms, makespan, n * 8, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(b + o_ops, ops + op_offset[0], n_ops * sizeof(gp_op),
                             cudaMemcpyHostToDevice, s));
    K8Scratch sc;
    sc.tab = reinterpret_cast<uint32_t*>(b + o_tab);
    sc.idx = reinterpret_cast<uint32_t*>(b + o_idx);
    sc.sorted = reinterpret_cast<uint32_t*>(b + o_srt);
    sc.lists = reinterpret_cast<uint32_t*>(b + o_lst);
    sc.its = reinterpret_cast<K8Iter*>(b + o_its);
    const int tpb = item_tpb(c, n);
    k8_validate<<<(unsigned)((n + tpb - 1) / tpb), tpb, 0, s>>>(
        reinterpret_cast<const gp_timing*>(b + o_tim), (long long)n,
        reinterpret_cast<const unsigned long long*>(b + o_off), reinterpret_cast<const gp_op*>(b + o_ops),
        reinterpret_cast<const double*>(b + o_ms), (int)iterations, tol, max_violations,
        reinterpret_cast<gp_violation*>(b + o_v), reinterpret_cast<uint32_t*>(b + o_nv),
        busy ? reinterpret_cast<double*>(b + o_busy) : nullptr, b + o_st, sc);
    CUDA_TRY(cudaGetLastError());
    if (max_violations)
        CUDA_TRY(cudaMemcpyAsync(violations, b + o_v, n * (size_t)max_violations * sizeof(gp_violation),
                                 cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(n_violations, b + o_nv, n * 4, cudaMemcpyDeviceToHost, s));
    if (busy)
        CUDA_TRY(cudaMemcpyAsync(busy, b + o_busy, n * GP_MAX_STAGES * 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(status, b + o_st, n, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return GP_OK;
}

int gp_sim_1f1b(gp_ctx* c, const gp_timing* timings, uint64_t n, uint32_t iterations,
                double* makespan, uint8_t* status) {
    if (!c) return fail(GP_ERR_INPUT, "null context");
    if (n == 0) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    CUDA_TRY(c->s_tim.ensure(n));
    CUDA_TRY(c->s_ms.ensure(n));
    CUDA_TRY(c->s_st.ensure(n));
    CUDA_TRY(cudaMemcpyAsync(c->s_tim.p, timings, n * sizeof(gp_timing), cudaMemcpyHostToDevice, s));
    int st = gp_sim_1f1b_device(c, c->s_tim.p, n, iterations, c->s_ms.p, c->s_st.p);
    if (st != GP_OK) return st;
    CUDA_TRY(cudaMemcpyAsync(makespan, c->s_ms.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(status, c->s_st.p, n, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return GP_OK;
}

// K6 for nb snapshots whose bandwidth matrices are at d_bw (device memory):
// patch the per-snapshot tables, then one sweep over (snapshot, item); the
// arg-min key of snapshot i goes to d_keys[i] and its table flags (errors
// that need the status-tracking path) to d_flags[i].  Asynchronous on the
// context stream.  `vsnap0` = global index of the first snapshot (verify sink).
static int snap_enqueue(gp_ctx* c, const double* d_bw, uint32_t nb, Key* d_keys,
                        uint32_t* d_flags, unsigned long long vsnap0) {
    cudaStream_t s = c->stream;
    const int k = c->F, n = c->n;
    uint64_t total;
    { int st_ = gp_space_size(c, &total); if (st_ != GP_OK) return st_; }
    const unsigned long long NP = h_fact(k), NC = h_binom(n - 1, k - 1);
    const unsigned long long items = (unsigned long long)c->nm * NP;
    const size_t ntri = (size_t)n * (n + 1) / 2, nxp = (size_t)((n + 1) & ~1);
    const size_t s_tpk = (size_t)c->nm * c->F * ntri, s_tcol = (size_t)c->nm * c->F * (n + 1);
    const size_t s_xt = (size_t)c->nm * c->F * c->F * nxp;
    CUDA_TRY(c->z_mbw.ensure((size_t)nb * c->F));
    CUDA_TRY(c->z_tpk.ensure((size_t)nb * s_tpk));
    CUDA_TRY(c->z_tcol.ensure((size_t)nb * s_tcol));
    CUDA_TRY(c->z_xt.ensure((size_t)nb * s_xt));
    CUDA_TRY(c->z_cnt.ensure(nb));
    CUDA_TRY(cudaMemsetAsync(d_flags, 0, nb * sizeof(uint32_t), s));
    CUDA_TRY(cudaMemsetAsync(c->z_cnt.p, 0, nb * sizeof(unsigned int), s));
    SnapGeom Z;
    Z.nsnap = (int)nb;
    Z.bw = d_bw; Z.mbw = c->z_mbw.p; Z.flags = d_flags;
    Z.tpk = c->z_tpk.p; Z.tcol = c->z_tcol.p; Z.xt = c->z_xt.p;
    Z.s_tpk = s_tpk; Z.s_tcol = s_tcol; Z.s_xt = s_xt;
    DevInst I = c->view();
    k6_minbw<<<(unsigned)((nb * c->F * 32 + 127) / 128), 128, 0, s>>>(I, Z);
    const long long work = (long long)(s_tpk + (size_t)c->nm * c->F * c->F * n);
    dim3 pg((unsigned)((work + 255) / 256), nb);
    k6_patch<<<pg, 256, 0, s>>>(I, Z);
    CUDA_TRY(cudaGetLastError());
    // sweep over (snapshot, item)
    size_t smem0 = 16 + (((size_t)(n + 1) * (k + 1) * 8 + 15) & ~(size_t)15) + (size_t)c->ngroups * 16;
    size_t smem1 = smem0 + ntri * 16 + (n + 1) * 16 + 3 * nxp * 8 + (size_t)n * 16;
    size_t smem2 = smem1 + ntri * 16;
    int mode = smem2 <= (size_t)c->smem_max ? 2 : (smem1 <= (size_t)c->smem_max ? 1 : 0);
    if (c->force_mode >= 0 && c->force_mode < mode) mode = c->force_mode;
    size_t smem = mode == 2 ? smem2 : (mode == 1 ? smem1 : smem0);
    SwFn kern = c->verify ? pick_sweep_verify(mode, c->nb, k) : pick_sweep(mode, c->nb, k);
    bool rec = false;
    if ((mode == 2 && items * nb >= 2ull * c->n_sms) || c->force_mode == 5)
        if (SwFn r = pick_sweep_rec(c, c->nb, k, &smem)) { kern = r; rec = true; }
    int per_sm = 0;
    { int st_ = kernel_slots(c, (const void*)kern, K3S_THREADS, smem, &per_sm);
      if (st_ != GP_OK) return st_; }
    unsigned long long resident = (unsigned long long)(per_sm > 0 ? per_sm : 1) * c->n_sms;
    unsigned long long cpi = (items * nb) >= resident ? 1 : resident / (items * nb);
    unsigned long long tasks = ((rec ? c->rec_W : c->sweep_W) + 31) / 32;
    unsigned long long cap = (tasks + (K3S_THREADS / 32) - 1) / (K3S_THREADS / 32);
    if (cpi > cap) cpi = cap;
    if (cpi < 1) cpi = 1;
    unsigned long long grid = (unsigned long long)nb * items * cpi;
    if (grid > 0x7fffffffull) return fail(GP_ERR_INPUT, "snapshot batch too large");
    const unsigned long long units = grid;
    SweepGeom G;
    if (rec) setup_rec(c, G);
    G.b0 = 0;
    G.k = k; G.nbm = c->nb * c->nm; G.NC = NC; G.NP = NP; G.item0 = 0; G.cpi = cpi;
    if (!rec) G.W = c->sweep_W;
    G.ngroups = c->ngroups; G.ng = c->ng; G.groups = c->groups.p;
    G.prefixes = c->prefixes.p;
    G.bnk = c->bnk.p;
    G.gsteps = 1;
    while (G.gsteps * 2 <= c->ngroups) G.gsteps *= 2;
    G.items = (unsigned int)items;
    G.tpk = c->z_tpk.p; G.tcol = c->z_tcol.p; G.xt = c->z_xt.p;
    G.s_tpk = s_tpk; G.s_tcol = s_tcol; G.s_xt = s_xt;
    if (c->verify) {  // global position = (vsnap0 + snap) * total + index
        G.vs = c->vs;
        G.vs.lo = c->vs.lo - vsnap0 * total;
    }
    // item counters, then (8-byte aligned) one u64 bound per snapshot for
    // the record sweep, all zeroed per launch
    const size_t nctr = ((size_t)nb * items + 1) & ~(size_t)1;
    if (c->item_ctr.cap < nctr + 2 * (size_t)nb || !c->item_ctr.p) c->ctr_armed = 0;
    CUDA_TRY(c->item_ctr.ensure(nctr + 2 * (size_t)nb));
    CUDA_TRY(cudaMemsetAsync(c->item_ctr.p, 0, (nctr + 2 * (size_t)nb) * sizeof(unsigned int), s));
    G.item_ctr = c->item_ctr.p;
    G.gbound = reinterpret_cast<unsigned long long*>(c->item_ctr.p + nctr);
    CUDA_TRY(c->blk.ensure(units > 4096 ? units : 4096));
    ArgminScratch S;
    S.blk = c->blk.p;
    S.counter = c->z_cnt.p;
    S.result = d_keys;
    S.err = nullptr;
    S.err_idx = c->err_idx.p;
    CUDA_TRY(kt_mark(c, false));
    CUDA_TRY(launch_sweep_kernel(kern, (unsigned)grid, smem, s, G, I, S, c->binom.p, d_flags));
    CUDA_TRY(kt_mark(c, true));
    CUDA_TRY(cudaGetLastError());
    return GP_OK;
}

// per-snapshot batch size: keep the per-snapshot tables around 256 MB
static uint32_t snap_batch(gp_ctx* c) {
    const int n = c->n;
    const size_t ntri = (size_t)n * (n + 1) / 2, nxp = (size_t)((n + 1) & ~1);
    const size_t per = ((size_t)c->nm * c->F * ntri + (size_t)c->nm * c->F * (n + 1)) * 16 +
                       (size_t)c->nm * c->F * c->F * nxp * 8 + (size_t)c->D * c->D * 8;
    uint32_t SB = (uint32_t)((256ull << 20) / (per ? per : 1));
    if (SB < 1) SB = 1;
    if (SB > 4096) SB = 4096;
    return SB;
}

// the fast (table-patch + sweep) path applies: error-free base tables, k >= 3
static int snap_fast_ok(gp_ctx* c, bool* ok) {
    uint64_t total;
    { int st_ = gp_space_size(c, &total); if (st_ != GP_OK) return st_; }
    int fl = known_flags(c);
    if (fl < 0) {
        CUDA_TRY(cudaEventSynchronize(c->flags_ev));
        fl = known_flags(c);
    }
    *ok = fl == 0 && c->F >= 3 && c->sweep_ok && c->nb <= 4 && total > 0 && c->force_mode != 3 &&
          c->force_mode != 4;
    return GP_OK;
}

int gp_replan_snapshots_async(gp_ctx* c, const double* d_bandwidth, uint32_t n_snap, void* d_keys,
                              uint32_t* d_flags) {
    if (c) { c->ctr_armed = 0; c->err_clean = false; }
    if (!c || !c->loaded || !d_bandwidth || !d_keys || !d_flags) return fail(GP_ERR_INPUT, "bad arguments");
    if (n_snap == 0) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    bool ok = false;
    { int st_ = snap_fast_ok(c, &ok); if (st_ != GP_OK) return st_; }
    if (!ok) return fail(GP_ERR_INPUT, "device snapshot path needs error-free tables and k >= 3 "
                                       "(use gp_replan_snapshots)");
    const uint32_t SB = snap_batch(c);
    const size_t DD = (size_t)c->D * c->D;
    for (uint32_t b0 = 0; b0 < n_snap; b0 += SB) {
        const uint32_t nb = (n_snap - b0) < SB ? (n_snap - b0) : SB;
        int st = snap_enqueue(c, d_bandwidth + (size_t)b0 * DD, nb, (Key*)d_keys + b0, d_flags + b0, b0);
        if (st != GP_OK) return st;
    }
    return GP_OK;
}

int gp_replan_snapshots(gp_ctx* c, const double* bandwidth, uint32_t n_snap, gp_best* out,
                        int32_t* status) {
    if (c) { c->ctr_armed = 0; c->err_clean = false; }  // launches below skip neither reset
    if (!c || !c->loaded || !bandwidth || !out || !status) return fail(GP_ERR_INPUT, "bad arguments");
    if (n_snap == 0) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    const int k = c->F, n = c->n;
    uint64_t total;
    { int st_ = gp_space_size(c, &total); if (st_ != GP_OK) return st_; }
    const unsigned long long NP = h_fact(k), NC = h_binom(n - 1, k - 1);
    const size_t DD = (size_t)c->D * c->D;
    bool fast = false;
    { int st_ = snap_fast_ok(c, &fast); if (st_ != GP_OK) return st_; }
    uint32_t SB = snap_batch(c);
    if (SB > n_snap) SB = n_snap;
    std::vector<uint32_t> h_fl(SB);
    std::vector<Key> h_res(SB);
    std::vector<uint32_t> slow;
    // matrices in pinned (mapped) host memory are read in place by the
    // patch kernels - only the member-pair and gateway entries cross PCIe
    // (about a quarter of each matrix at C4) - instead of a full H2D copy
    // (GP_SNAP_ZEROCOPY=0 disables)
    const double* zc = nullptr;
    {
        cudaPointerAttributes pa;
        const char* e = getenv("GP_SNAP_ZEROCOPY");
        if ((!e || atoi(e) != 0) && cudaPointerGetAttributes(&pa, bandwidth) == cudaSuccess &&
            pa.type == cudaMemoryTypeHost && pa.devicePointer)
            zc = static_cast<const double*>(pa.devicePointer);
        (void)cudaGetLastError();  // (pageable memory: not an error here)
    }
    for (uint32_t b0 = 0; b0 < n_snap; b0 += SB) {
        const uint32_t nb = (n_snap - b0) < SB ? (n_snap - b0) : SB;
        if (!fast) {
            for (uint32_t i = 0; i < nb; ++i) slow.push_back(b0 + i);
            continue;
        }
        CUDA_TRY(c->z_flags.ensure(SB));
        CUDA_TRY(c->z_res.ensure(SB));
        const double* d_bw = zc ? zc + (size_t)b0 * DD : nullptr;
        if (!zc) {
            CUDA_TRY(c->z_bw.ensure((size_t)SB * DD));
            CUDA_TRY(cudaMemcpyAsync(c->z_bw.p, bandwidth + (size_t)b0 * DD, (size_t)nb * DD * 8,
                                     cudaMemcpyHostToDevice, s));
            d_bw = c->z_bw.p;
        }
        int st = snap_enqueue(c, d_bw, nb, c->z_res.p, c->z_flags.p, b0);
        if (st != GP_OK) return st;
        CUDA_TRY(cudaMemcpyAsync(h_res.data(), c->z_res.p, nb * sizeof(Key), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(h_fl.data(), c->z_flags.p, nb * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        for (uint32_t i = 0; i < nb; ++i) {
            gp_best& o = out[b0 + i];
            memset(&o, 0, sizeof(o));
            o.k = (uint32_t)k;
            o.evaluated = total;
            if (h_fl[i]) { slow.push_back(b0 + i); continue; }
            const Key& r = h_res[i];
            if (r.tie == ~0ull) { status[b0 + i] = GP_ERR_NO_FEASIBLE; continue; }
            const int nbm = c->nb * c->nm;
            unsigned long long bmv = r.tie % (unsigned long long)nbm, pc = r.tie / (unsigned long long)nbm;
            o.cost = r.cost;
            o.index = (bmv * NP + pc / NC) * NC + pc % NC;
            o.batch_index = (uint32_t)(bmv / c->nm);
            o.micro_index = (uint32_t)(bmv % c->nm);
            h_unrank_perm(k, pc / NC, o.order);
            h_unrank_counts(n, k, pc % NC, o.counts);
            status[b0 + i] = GP_OK;
        }
    }
    if (!slow.empty()) {
        // exact status-tracking path, one snapshot at a time on the context
        const VerifySink vs0 = c->vs;
        for (uint32_t sn : slow) {
            int st = gp_set_bandwidth(c, bandwidth + (size_t)sn * DD);
            c->vs.lo = vs0.lo - (unsigned long long)sn * total;  // snapshot sn's slots
            if (st == GP_OK) st = gp_argmin_range(c, 0, total, &out[sn]);
            status[sn] = st;
        }
        c->vs = vs0;
        int st = gp_reset_bandwidth(c);
        if (st != GP_OK) return st;
    }
    return GP_OK;
}

int gp_sim_candidates(gp_ctx* c, uint32_t k, uint64_t n, const uint8_t* order,
                      const uint8_t* counts, const uint8_t* bm, uint32_t iterations,
                      double opt_seconds, double* makespan, uint8_t* status) {
    if (!c || !c->loaded) return fail(GP_ERR_INPUT, "context not loaded");
    if (k < 1 || k > GP_MAX_STAGES) return fail(GP_ERR_INPUT, "k=%u outside [1,%d]", k, GP_MAX_STAGES);
    if (n == 0) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    CUDA_TRY(c->b_order.ensure(n * k));
    CUDA_TRY(c->b_counts.ensure(n * k));
    CUDA_TRY(c->b_bm.ensure(n));
    CUDA_TRY(c->b_cost.ensure(n));
    CUDA_TRY(c->b_status.ensure(n));
    CUDA_TRY(cudaMemcpyAsync(c->b_order.p, order, n * k, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->b_counts.p, counts, n * k, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->b_bm.p, bm, n, cudaMemcpyHostToDevice, s));
    DevInst I = c->view();
    const int tpb = item_tpb(c, n);
    // group the candidates by (b, m) index (equal micro-batch counts per
    // warp; GP_K5_SORT=0 disables)
    uint32_t* perm = nullptr;
    static const int sort_on = [] { const char* e = getenv("GP_K5_SORT"); return e ? atoi(e) : 1; }();
    const int nbm = c->nb * c->nm;
    if (sort_on && n >= 1024 && n < (1ull << 32) && nbm <= 256) {
        CUDA_TRY(c->k5_perm.ensure(n));
        CUDA_TRY(c->k5_hist.ensure(260));
        CUDA_TRY(cudaMemsetAsync(c->k5_hist.p, 0, 260 * sizeof(uint32_t), s));
        unsigned hb = (unsigned)((n + 255) / 256);
        if (hb > 2u * (unsigned)c->n_sms) hb = 2u * (unsigned)c->n_sms;
        k5_bm_hist<<<hb, 256, 0, s>>>((long long)n, c->b_bm.p, nbm, c->k5_hist.p);
        k5_bm_scan<<<1, 1, 0, s>>>(nbm, c->k5_hist.p);
        k5_bm_scatter<<<(unsigned)((n + 255) / 256), 256, 0, s>>>((long long)n, c->b_bm.p, nbm, c->k5_hist.p,
                                                                 c->k5_perm.p);
        perm = c->k5_perm.p;
    }
    k5_sim_candidates<<<(unsigned)((n + tpb - 1) / tpb), tpb, 0, s>>>(I, (int)k, (long long)n, c->b_order.p,
                                                                 c->b_counts.p, c->b_bm.p,
                                                                 (int)iterations, opt_seconds,
                                                                 c->b_cost.p, c->b_status.p, perm);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(makespan, c->b_cost.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(status, c->b_status.p, n, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return GP_OK;
}

int gp_plan_timing(gp_ctx* c, uint32_t k, uint64_t n, const uint8_t* order, const uint8_t* counts,
                   const uint8_t* bm, double opt_seconds, gp_timing* timings, uint8_t* status) {
    if (!c || !c->loaded) return fail(GP_ERR_INPUT, "context not loaded");
    if (k < 1 || k > GP_MAX_STAGES) return fail(GP_ERR_INPUT, "k=%u outside [1,%d]", k, GP_MAX_STAGES);
    if (!order || !counts || !bm || !timings || !status) return fail(GP_ERR_INPUT, "bad arguments");
    if (n == 0) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    CUDA_TRY(c->b_order.ensure(n * k));
    CUDA_TRY(c->b_counts.ensure(n * k));
    CUDA_TRY(c->b_bm.ensure(n));
    CUDA_TRY(c->b_status.ensure(n));
    CUDA_TRY(c->s_tim.ensure(n));
    CUDA_TRY(cudaMemcpyAsync(c->b_order.p, order, n * k, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->b_counts.p, counts, n * k, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->b_bm.p, bm, n, cudaMemcpyHostToDevice, s));
    k5_plan_timing<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(c->view(), (int)k, (long long)n,
                                                              c->b_order.p, c->b_counts.p,
                                                              c->b_bm.p, opt_seconds, c->s_tim.p,
                                                              c->b_status.p);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(timings, c->s_tim.p, n * sizeof(gp_timing), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(status, c->b_status.p, n, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return GP_OK;
}

int gp_plan_cost(gp_ctx* c, uint32_t k, const gp_plan_stage* stages, int64_t batch,
                 int64_t microbatch, double opt_seconds, gp_plan_info* out, gp_timing* timing) {
    if (!c || !c->loaded) return fail(GP_ERR_INPUT, "context not loaded");
    if (!stages || !out) return fail(GP_ERR_INPUT, "bad arguments");
    if (k < 1 || k > GP_MAX_STAGES) return fail(GP_ERR_INPUT, "k=%u outside [1,%d]", k, GP_MAX_STAGES);
    if (batch <= 0 || microbatch <= 0 || batch % microbatch)
        return fail(GP_ERR_INPUT, "micro-batch %lld does not divide batch %lld",
                    (long long)microbatch, (long long)batch);
    uint32_t pos = 0, seen = 0;
    for (uint32_t s = 0; s < k; ++s) {
        const gp_plan_stage& g = stages[s];
        if (g.fg >= (uint32_t)c->F || ((seen >> g.fg) & 1u))
            return fail(GP_ERR_INPUT, "stage %u: bad or repeated group %u", s, g.fg);
        seen |= 1u << g.fg;
        if (g.layer_start != pos || g.layer_end <= g.layer_start || g.layer_end > (uint32_t)c->n)
            return fail(GP_ERR_INPUT, "stage layer ranges must tile the layer list without gaps");
        pos = g.layer_end;
        if (g.kind > GP_ASYM_TP_DP || g.n_parts > GP_MAX_SGS)
            return fail(GP_ERR_INPUT, "stage %u: bad split", s);
        const uint32_t nsg = (uint32_t)(c->h_fg_sg_count[g.fg]);
        for (uint32_t j = 0; g.kind == GP_ASYM_PP && j < g.n_parts; ++j)
            if (g.pp_sg[j] >= nsg || g.pp_start[j] > g.pp_end[j] || g.pp_end[j] > (uint32_t)c->n)
                return fail(GP_ERR_INPUT, "stage %u: bad pipeline part %u", s, j);
    }
    if (pos != (uint32_t)c->n) return fail(GP_ERR_INPUT, "plan covers %u of %d layers", pos, c->n);
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t o_st = 0, o_out = al(k * sizeof(gp_plan_stage)), o_tim = o_out + al(sizeof(gp_plan_info));
    const size_t o_stat = o_tim + al(sizeof(gp_timing));
    CUDA_TRY(c->g_buf.ensure(o_stat + 16));
    uint8_t* b = c->g_buf.p;
    CUDA_TRY(cudaMemcpyAsync(b + o_st, stages, k * sizeof(gp_plan_stage), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemsetAsync(b + o_out, 0, sizeof(gp_plan_info), s));
    CUDA_TRY(cudaMemsetAsync(b + o_tim, 0, sizeof(gp_timing), s));
    k_plan_cost<<<1, 32, 0, s>>>(c->view(), (int)k, reinterpret_cast<const gp_plan_stage*>(b + o_st),
                                 (long long)batch, (long long)microbatch, opt_seconds,
                                 reinterpret_cast<gp_plan_info*>(b + o_out),
                                 timing ? reinterpret_cast<gp_timing*>(b + o_tim) : nullptr,
                                 reinterpret_cast<int*>(b + o_stat));
    CUDA_TRY(cudaGetLastError());
    int st = GP_OK;
    CUDA_TRY(cudaMemcpyAsync(out, b + o_out, sizeof(gp_plan_info), cudaMemcpyDeviceToHost, s));
    if (timing) CUDA_TRY(cudaMemcpyAsync(timing, b + o_tim, sizeof(gp_timing), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&st, b + o_stat, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (st != GP_OK) return fail(st, "build_plan_timing raised (status %d)", st);
    return GP_OK;
}

// Parity tests: from now on every K3 / K6 launch (sweep, sub-range tile
// kernel, generic kernel, the gp_replan graph, snapshot batches) uses the
// verify instantiation and stores each evaluated candidate's cost at global
// position g = snapshot * space_size + enumeration index, for g in
// [lo, lo + n).  Unwritten slots keep an all-ones NaN pattern.
int gp_diag_verify_begin(gp_ctx* c, uint64_t lo, uint64_t n) {
    if (!c || !c->loaded || n == 0) return fail(GP_ERR_INPUT, "context not loaded / empty sink");
    CUDA_TRY(cudaSetDevice(c->device));
    uint64_t total;
    { int st_ = gp_space_size(c, &total); if (st_ != GP_OK) return st_; }
    CUDA_TRY(c->vbuf.ensure(n));
    CUDA_TRY(cudaMemsetAsync(c->vbuf.p, 0xFF, n * sizeof(double), c->stream));
    c->vs.out = c->vbuf.p;
    c->vs.lo = lo;
    c->vs.n = n;
    c->vs.stride = total;
    c->verify = true;
    if (c->graph_exec) { cudaGraphExecDestroy(c->graph_exec); c->graph_exec = nullptr; }
    return GP_OK;
}

// Ends verify mode and copies the sink (n doubles) to host memory `out`.
int gp_diag_verify_end(gp_ctx* c, double* out) {
    if (!c || !c->verify) return fail(GP_ERR_INPUT, "verify mode not active");
    CUDA_TRY(cudaSetDevice(c->device));
    const uint64_t n = c->vs.n;
    c->verify = false;
    c->vs = VerifySink();
    if (c->graph_exec) { cudaGraphExecDestroy(c->graph_exec); c->graph_exec = nullptr; }
    if (out) CUDA_TRY(cudaMemcpyAsync(out, c->vbuf.p, n * sizeof(double), cudaMemcpyDeviceToHost,
                                      c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return GP_OK;
}

// Diagnostics (bench.py roofline): enable = 1 starts a window in which every
// exhaustive sweep launch (K3 / K6) is bracketed by CUDA events on the
// context stream; enable = 0 ends it and returns the summed device time of
// those launches and their count.
int gp_diag_kernel_timing(gp_ctx* c, int enable, double* total_ms, uint64_t* launches) {
    if (!c) return fail(GP_ERR_INPUT, "null context");
    CUDA_TRY(cudaSetDevice(c->device));
    if (enable) {
        c->ktime = true;
        c->kt_used = 0;
        return GP_OK;
    }
    c->ktime = false;
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    double tot = 0.0;
    for (size_t i = 0; i + 1 < c->kt_used; i += 2) {
        float ms = 0.0f;
        CUDA_TRY(cudaEventElapsedTime(&ms, c->kt_ev[i], c->kt_ev[i + 1]));
        tot += ms;
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = c->kt_used / 2;
    c->kt_used = 0;
    return GP_OK;
}

// Checked builds (-DGP_CHECKS): first failing device check line of either
// translation unit since the last call (0 = none), then cleared.  Other
// builds report 0xFFFFFFFF (checks compiled out).
int gp_diag_checks(gp_ctx* c, uint32_t* line) {
    if (!c || !line) return fail(GP_ERR_INPUT, "null argument");
#if defined(GP_CHECKS)
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaDeviceSynchronize());
    unsigned int v = 0, z = 0;
    CUDA_TRY(cudaMemcpyFromSymbol(&v, g_chk_line, sizeof(v)));
    CUDA_TRY(cudaMemcpyToSymbol(g_chk_line, &z, sizeof(z)));
    const unsigned int w = verify_tu_checks();
    *line = v ? v : w;
#else
    *line = 0xFFFFFFFFu;
#endif
    return GP_OK;
}

int gp_ctx_set_k3_mode(gp_ctx* c, int mode) {
    if (!c || mode < -1 || mode > 5) return fail(GP_ERR_INPUT, "bad mode");
    c->force_mode = mode;
    return GP_OK;
}

int gp_diag_timeline(void* out, uint32_t cap, uint32_t* n_out) {
    if (!n_out) return fail(GP_ERR_INPUT, "null output");
    *n_out = 0;
#if defined(GP_TIMELINE)
    unsigned int n = 0;
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpyFromSymbol(&n, g_tl_n, sizeof(n)));
    if (n > GP_TL_CAP) n = GP_TL_CAP;
    if (n > cap) n = cap;
    if (out && n) CUDA_TRY(cudaMemcpyFromSymbol(out, g_tl, n * sizeof(TlRec)));
    const unsigned int zero = 0;
    CUDA_TRY(cudaMemcpyToSymbol(g_tl_n, &zero, sizeof(zero)));
    *n_out = n;
#else
    (void)out; (void)cap;
#endif
    return GP_OK;
}

int gp_diag_replan_host(gp_ctx* c, double* host_us4) {
    if (!c || !host_us4) return fail(GP_ERR_INPUT, "null argument");
    memcpy(host_us4, c->host_us, sizeof(c->host_us));
    return GP_OK;
}

int gp_diag_replan_timing(gp_ctx* c, int enable, double* last_graph_ms) {
    if (!c) return fail(GP_ERR_INPUT, "null context");
    if (enable && !c->t_ev0) {
        CUDA_TRY(cudaSetDevice(c->device));
        CUDA_TRY(cudaEventCreate(&c->t_ev0));
        CUDA_TRY(cudaEventCreate(&c->t_ev1));
    }
    c->diag_timing = enable != 0;
    if (last_graph_ms) *last_graph_ms = (double)c->last_graph_ms;
    return GP_OK;
}

int gp_diag_fp64_peak(int device, double* dadd_per_second) {
    if (!dadd_per_second) return fail(GP_ERR_INPUT, "null output");
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 1 << 14;
    double* sink = nullptr;
    CUDA_TRY(cudaMalloc(&sink, blocks * sizeof(double)));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_fp64_peak<<<blocks, threads>>>(sink, iters, 1e-9);  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_fp64_peak<<<blocks, threads>>>(sink, iters, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (err != cudaSuccess) return fail(GP_ERR_CUDA, "fp64 peak: %s", cudaGetErrorString(err));
    double ops = (double)blocks * threads * iters * 8.0;
    *dadd_per_second = ops / (best * 1e-3);
    return GP_OK;
}

}  // extern "C"

// ----------------------------------------------------------------------------
// K7: device grouping per topology snapshot
// ----------------------------------------------------------------------------
static int ensure_stage(gp_ctx* c, size_t bytes) {
    if (bytes <= c->h_stage_cap && c->h_stage) return GP_OK;
    if (c->h_stage) cudaFreeHost(c->h_stage);
    c->h_stage = nullptr;
    c->h_stage_cap = 0;
    CUDA_TRY(cudaHostAlloc((void**)&c->h_stage, bytes, cudaHostAllocDefault));
    c->h_stage_cap = bytes;
    return GP_OK;
}

static int group_launch(gp_ctx* c, uint32_t D, uint32_t n_snap, const double* p_t,
                        const double* bandwidth, const double* p_c, double threshold_net,
                        double threshold_compute, const uint16_t* fixed_fg, uint32_t fixed_nf,
                        uint16_t* fg_of, uint16_t* sg_of, uint32_t* n_fg, uint32_t* n_sg,
                        double* fg_intra, double* fg_capacity, double* fg_min_bw,
                        double* sg_capacity) {
    if (!c || !p_t || !p_c || !fg_of || !sg_of || !n_fg || !n_sg || !fg_intra || !fg_capacity ||
        !fg_min_bw || !sg_capacity)
        return fail(GP_ERR_INPUT, "bad arguments");
    if (D == 0) return fail(GP_ERR_INPUT, "topology has no devices");
    if (D > GP_MAX_MEMBERS) return fail(GP_ERR_INPUT, "%u devices exceed %d", D, GP_MAX_MEMBERS);
    if (!(threshold_net > 0 && threshold_net < 1) || !(threshold_compute > 0 && threshold_compute < 1))
        return fail(GP_ERR_INPUT, "threshold must lie in (0, 1)");
    if (n_snap == 0) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    const size_t DD = (size_t)D * D;
    const size_t per_scr = k7_scratch_bytes((int)D);
    // snapshots per launch: scratch <= 512 MiB
    uint32_t SB = (uint32_t)((512ull << 20) / per_scr);
    if (SB < 1) SB = 1;
    if (SB > n_snap) SB = n_snap;
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t o_pt = 0, o_bw = o_pt + al(SB * DD * 8), o_pc = o_bw + al(bandwidth ? SB * DD * 8 : 8);
    const size_t o_u16 = o_pc + al((size_t)D * 8), o_cnt = o_u16 + al((size_t)SB * D * 2 * 2);
    const size_t o_dbl = o_cnt + al((size_t)SB * 2 * 4), o_fix = o_dbl + al((size_t)SB * D * 4 * 8);
    const size_t o_nsf = o_fix + al((size_t)D * 2), o_stg = o_nsf + al((size_t)SB * D * 4);
    const size_t o_scr = o_stg + al((size_t)SB * D * 8);
    const size_t total = o_scr + SB * per_scr;
    CUDA_TRY(c->g_buf.ensure(total));
    uint8_t* b = c->g_buf.p;
    // small clusters keep the pair tables (and p_t) in shared memory
    const size_t head = k7_smem_head((int)D), tabs = k7_scratch_bytes((int)D);
    int smem_mode = 0;
    size_t smem = head;
    if (head + tabs + DD * 8 <= (200u << 10)) { smem_mode = 3; smem = head + tabs + DD * 8; }
    else if (head + tabs <= (200u << 10)) { smem_mode = 1; smem = head + tabs; }
    typedef decltype(&k7_group<0>) K7Fn;
    const K7Fn k7fn = smem_mode == 3 ? k7_group<3> : (smem_mode == 1 ? k7_group<1> : k7_group<0>);
    { int ps_ = 0, st_ = kernel_slots(c, (const void*)k7fn, K7_THREADS, smem, &ps_);
      if (st_ != GP_OK) return st_; }
    // inputs [o_pt, o_u16) and outputs [o_u16, o_fix) travel through one
    // pinned staging buffer: one H2D and one D2H per batch
    { int st_ = ensure_stage(c, o_scr); if (st_ != GP_OK) return st_; }
    uint8_t* hs = c->h_stage;
    memcpy(hs + o_pc, p_c, (size_t)D * 8);
    if (fixed_fg) memcpy(hs + o_fix, fixed_fg, (size_t)D * 2);
    CUDA_TRY(cudaMemcpyAsync(b + o_pc, hs + o_pc, o_u16 - o_pc, cudaMemcpyHostToDevice, s));
    if (fixed_fg) CUDA_TRY(cudaMemcpyAsync(b + o_fix, hs + o_fix, (size_t)D * 2, cudaMemcpyHostToDevice, s));
    for (uint32_t s0 = 0; s0 < n_snap; s0 += SB) {
        const uint32_t nb = (n_snap - s0) < SB ? (n_snap - s0) : SB;
        memcpy(hs + o_pt, p_t + (size_t)s0 * DD, nb * DD * 8);
        if (bandwidth) memcpy(hs + o_bw, bandwidth + (size_t)s0 * DD, nb * DD * 8);
        CUDA_TRY(cudaMemcpyAsync(b + o_pt, hs + o_pt, (bandwidth ? o_bw + nb * DD * 8 : nb * DD * 8),
                                 cudaMemcpyHostToDevice, s));
        uint16_t* d_fg = reinterpret_cast<uint16_t*>(b + o_u16);
        uint16_t* d_sg = d_fg + (size_t)SB * D;
        uint32_t* d_nf = reinterpret_cast<uint32_t*>(b + o_cnt);
        uint32_t* d_ns = d_nf + SB;
        double* d_dbl = reinterpret_cast<double*>(b + o_dbl);
        double *d_fi = d_dbl, *d_fc = d_fi + (size_t)SB * D, *d_fb = d_fc + (size_t)SB * D,
               *d_sc = d_fb + (size_t)SB * D;
        uint32_t* d_nsf = reinterpret_cast<uint32_t*>(b + o_nsf);
        double* d_stg = reinterpret_cast<double*>(b + o_stg);
        auto launch = [&](unsigned grid, int phase) {
            k7fn<<<grid, K7_THREADS, smem, s>>>(
                (int)D, reinterpret_cast<const double*>(b + o_pt),
                bandwidth ? reinterpret_cast<const double*>(b + o_bw) : nullptr, (long long)DD,
                (long long)DD, reinterpret_cast<const double*>(b + o_pc), threshold_net,
                threshold_compute, b + o_scr, per_scr, smem_mode,
                fixed_fg ? reinterpret_cast<const uint16_t*>(b + o_fix) : nullptr, (int)fixed_nf,
                d_fg, d_sg, d_nf, d_ns, d_fi, d_fc, d_fb, d_sc, phase, d_nsf, d_stg);
        };
        // pair tables in shared memory: the FGs' second levels run as
        // separate CTAs (phase 2) instead of one after another in the
        // snapshot's CTA; GP_K7_SPLIT=0 keeps the single-kernel form
        // (only while the snapshots alone leave SMs idle: a large batch fills
        // the GPU with whole-snapshot CTAs already)
        bool split = (smem_mode & 1) != 0 && nb < 2u * (uint32_t)c->n_sms;
        if (const char* e = getenv("GP_K7_SPLIT")) split = split && atoi(e) != 0;
        if (split) {
            launch(nb, 1);
            launch(nb * D, 2);
            k7_sg_finish<<<(nb + 127) / 128, 128, 0, s>>>((int)D, (int)nb, d_nf, d_fg, d_nsf, d_stg,
                                                          d_sc, d_ns);
        } else {
            launch(nb, 0);
        }
        CUDA_TRY(cudaGetLastError());
        const size_t o = (size_t)s0 * D;
        CUDA_TRY(cudaMemcpyAsync(hs + o_u16, b + o_u16, o_fix - o_u16, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));  // staging buffers are reused by the next batch
        auto hp = [&](const void* dptr) { return hs + ((const uint8_t*)dptr - b); };
        memcpy(fg_of + o, hp(d_fg), (size_t)nb * D * 2);
        memcpy(sg_of + o, hp(d_sg), (size_t)nb * D * 2);
        memcpy(n_fg + s0, hp(d_nf), (size_t)nb * 4);
        memcpy(n_sg + s0, hp(d_ns), (size_t)nb * 4);
        memcpy(fg_intra + o, hp(d_fi), (size_t)nb * D * 8);
        memcpy(fg_capacity + o, hp(d_fc), (size_t)nb * D * 8);
        memcpy(fg_min_bw + o, hp(d_fb), (size_t)nb * D * 8);
        memcpy(sg_capacity + o, hp(d_sc), (size_t)nb * D * 8);
    }
    return GP_OK;
}

extern "C" int gp_group_snapshots(gp_ctx* c, uint32_t D, uint32_t n_snap, const double* p_t,
                                  const double* bandwidth, const double* p_c, double threshold_net,
                                  double threshold_compute, uint16_t* fg_of, uint16_t* sg_of,
                                  uint32_t* n_fg, uint32_t* n_sg, double* fg_intra,
                                  double* fg_capacity, double* fg_min_bw, double* sg_capacity) {
    return group_launch(c, D, n_snap, p_t, bandwidth, p_c, threshold_net, threshold_compute,
                        nullptr, 0, fg_of, sg_of, n_fg, n_sg, fg_intra, fg_capacity, fg_min_bw,
                        sg_capacity);
}

extern "C" int gp_group_fixed(gp_ctx* c, uint32_t D, const double* p_t, const double* bandwidth,
                              const double* p_c, const uint16_t* fg_of_in, uint32_t n_fg_in,
                              double threshold_compute, uint16_t* sg_of, uint32_t* n_sg,
                              double* fg_intra, double* fg_capacity, double* fg_min_bw,
                              double* sg_capacity) {
    if (!fg_of_in || n_fg_in == 0 || n_fg_in > D) return fail(GP_ERR_INPUT, "bad first-level partition");
    std::vector<uint32_t> cnt(n_fg_in, 0);
    for (uint32_t d = 0; d < D; ++d) {
        if (fg_of_in[d] >= n_fg_in) return fail(GP_ERR_INPUT, "device %u: group index out of range", d);
        cnt[fg_of_in[d]]++;
    }
    for (uint32_t f = 0; f < n_fg_in; ++f) if (!cnt[f]) return fail(GP_ERR_INPUT, "group %u is empty", f);
    std::vector<uint16_t> fg_out(D);
    uint32_t nf = 0;
    return group_launch(c, D, 1, p_t, bandwidth, p_c, 0.5, threshold_compute, fg_of_in, n_fg_in,
                        fg_out.data(), sg_of, &nf, n_sg, fg_intra, fg_capacity, fg_min_bw,
                        sg_capacity);
}

// ----------------------------------------------------------------------------
// Peer-memory all-gather of small per-rank records over NVLink / NVSwitch:
// each rank owns one device buffer [arrival counter (256 B) | 2 x world x
// slot bytes]; the buffers are exported as CUDA IPC handles and opened by
// every other rank of the box.  A rank's gather = one kernel that stores its
// slot into every peer's buffer (P2P stores over NVLink), fences at system
// scope and bumps every peer's counter, then one kernel that waits (acquire)
// until its own counter shows all ranks of this epoch.  Epochs alternate
// between the two tables: a peer already at epoch e + 1 writes the other
// table while this rank still reads epoch e's, and it cannot reach e + 2
// before this rank's own epoch-(e + 1) store, which this rank issues after
// consuming epoch e in stream order.  Replaces the NCCL all-gather of the K6
// winners (16 B per snapshot) inside the bench step.
// ----------------------------------------------------------------------------
#define GP_PEER_MAX 16
struct PeerSet { unsigned char* base[GP_PEER_MAX]; };

static __global__ void k_peer_put(const unsigned char* __restrict__ src, unsigned long long slot_bytes,
                                  int rank, int world, int table, PeerSet P) {
    // blockIdx.x = destination rank; the slot copied 16 B per thread
    const int dst = blockIdx.x;
    unsigned char* d = P.base[dst] + 256 + ((size_t)table * world + rank) * slot_bytes;
    const unsigned long long n16 = slot_bytes / 16;
    for (unsigned long long i = threadIdx.x; i < n16; i += blockDim.x)
        reinterpret_cast<uint4*>(d)[i] = reinterpret_cast<const uint4*>(src)[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();  // the slot before the arrival
        atomicAdd_system(reinterpret_cast<unsigned long long*>(P.base[dst]), 1ull);
    }
}

// bounded: gives up after ~2 s (a peer that never arrives must not hang the
// GPU) and records the shortfall in the buffer's second word for
// gp_peer_read's caller to see
static __global__ void k_peer_wait(unsigned long long* counter, unsigned long long target) {
    if (threadIdx.x != 0) return;
    unsigned long long v, t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(counter) : "memory");
        if (v >= target) return;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 2000000000ull) { counter[1] = target - v; return; }  // timed out
        __nanosleep(100);
    }
}

extern "C" {

int gp_peer_alloc(gp_ctx* c, uint64_t bytes, void** d_ptr, void* ipc_handle) {
    if (!c || !d_ptr || !ipc_handle || bytes == 0) return fail(GP_ERR_INPUT, "bad arguments");
    CUDA_TRY(cudaSetDevice(c->device));
    void* p = nullptr;
    CUDA_TRY(cudaMalloc(&p, bytes));
    CUDA_TRY(cudaMemset(p, 0, bytes));
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) { cudaFree(p); return fail(GP_ERR_CUDA, "ipc handle: %s", cudaGetErrorString(e)); }
    memcpy(ipc_handle, &h, sizeof(h));
    *d_ptr = p;
    return GP_OK;
}

int gp_peer_open(gp_ctx* c, const void* ipc_handle, void** d_ptr) {
    if (!c || !ipc_handle || !d_ptr) return fail(GP_ERR_INPUT, "bad arguments");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof(h));
    CUDA_TRY(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return GP_OK;
}

int gp_peer_close(gp_ctx* c, void* d_ptr, int owned) {
    if (!c || !d_ptr) return GP_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    if (owned) CUDA_TRY(cudaFree(d_ptr));
    else CUDA_TRY(cudaIpcCloseMemHandle(d_ptr));
    return GP_OK;
}

int gp_peer_read(gp_ctx* c, const void* d_ptr, void* host, uint64_t bytes) {
    if (!c || !d_ptr || !host) return fail(GP_ERR_INPUT, "bad arguments");
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaMemcpyAsync(host, d_ptr, bytes, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return GP_OK;
}

int gp_peer_allgather(gp_ctx* c, const void* d_src, uint64_t slot_bytes, uint32_t rank,
                      uint32_t world, void* const* peer_bases, uint64_t epoch) {
    if (!c || !d_src || !peer_bases || world == 0 || world > GP_PEER_MAX || rank >= world ||
        slot_bytes % 16 != 0)
        return fail(GP_ERR_INPUT, "bad arguments");
    CUDA_TRY(cudaSetDevice(c->device));
    PeerSet P = {};
    for (uint32_t r = 0; r < world; ++r) P.base[r] = reinterpret_cast<unsigned char*>(peer_bases[r]);
    k_peer_put<<<world, 128, 0, c->stream>>>(reinterpret_cast<const unsigned char*>(d_src), slot_bytes,
                                             (int)rank, (int)world, (int)(epoch & 1), P);
    k_peer_wait<<<1, 32, 0, c->stream>>>(reinterpret_cast<unsigned long long*>(peer_bases[rank]),
                                         (unsigned long long)epoch * world);
    CUDA_TRY(cudaGetLastError());
    return GP_OK;
}

}  // extern "C"
