/*
 * geopipe_b200.h - C-ABI of the B200 plan-evaluation engine.
 *
 * Drop-in boundary for the reference planner's hot path
 * (/root/reference/pkg/src/geopipe/, "src/" below).  The reference is pure
 * Python with no FFI of its own; each entry point here replaces one Python
 * seam and is bound from Python with ctypes:
 *
 *   gp_ctx_create / gp_ctx_load  <- the frozen inputs of search_plan /
 *                                   exhaustive_plan: ModelSpec, ClusterTopology,
 *                                   GroupIndex, SearchConfig.bottleneck_factor
 *                                   (src/planner.py:330-335, :374-379)
 *   gp_eval_batch               <- a batch of _evaluate(candidate, b, m, ...)
 *                                   calls (src/planner.py:313-327)
 *   gp_argmin_range             <- the exhaustive_plan loop nest and its
 *                                   strict-< key (src/planner.py:389-399)
 *   gp_plan_detail              <- build_plan + plan_cost for one candidate:
 *                                   splits and CostBreakdown of the winner
 *                                   (src/planner.py:203-223, src/costmodel.py:84-100)
 *   gp_set_bandwidth            <- a bandwidth snapshot: LinkMeasurement with
 *                                   scaled bandwidth -> build_topology ->
 *                                   group_first_level (min_intra_bandwidth)
 *                                   (src/profiling.py:48-78,167-215,
 *                                    src/grouping.py:69-75)
 *   gp_sim_1f1b                 <- simulate_timing(timing, ONE_F_ONE_B,
 *                                   SimConfig(iterations=1)).makespan
 *                                   (src/simulator.py:71-113, src/engine.py:230-431)
 *
 * Conventions: plain pointers and sizes, no exceptions.  Every call returns a
 * status; GP_OK is 0 and the others map onto the reference's exceptions
 * (src/errors.py).  gp_last_error() returns the message of the last failure
 * on the calling thread.  One context per host thread; a context owns one
 * CUDA device and one stream.  There is no CPU fallback: when no sm_100
 * device is present gp_ctx_create fails with GP_ERR_CUDA.
 */
#ifndef GEOPIPE_B200_H
#define GEOPIPE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (src/errors.py) */
enum {
    GP_OK = 0,
    GP_ERR_INPUT = 1,          /* InputFileError / ValueError                 */
    GP_ERR_INFEASIBLE_SPLIT = 2,/* InfeasibleSplitError                       */
    GP_ERR_NO_FEASIBLE = 3,    /* NoFeasiblePlanError                         */
    GP_ERR_DEGENERATE = 4,     /* DegenerateGroupError (src/timing.py:138,142)*/
    GP_ERR_TOPOLOGY = 5,       /* InvalidTopologyError (src/timing.py:172,184,215) */
    GP_ERR_CUDA = 6,           /* device failure / no sm_100 device           */
    GP_ERR_TIMING = 7,         /* InvalidTimingError (src/engine.py:136-141)  */
    GP_ERR_SCHEDULING = 8      /* SchedulingBugError (src/engine.py:422)      */
};

/* split kinds, src/plans.py:60-66 */
enum { GP_UNIFORM = 0, GP_ASYM_PP = 1, GP_ASYM_DP = 2, GP_ASYM_TP_DP = 3 };

#define GP_MAX_STAGES 16   /* first-level groups per plan            */
#define GP_MAX_SGS 16      /* second-level groups per first-level one */
#define GP_MAX_LAYERS 255  /* layer counts travel as uint8            */
#define GP_MAX_MEMBERS 1024 /* devices per first-level group          */

/*
 * One planner instance, structure-of-arrays, host memory.  All values are
 * the reference's own (already derived) numbers:
 *   layers   : LayerSpec fields (src/plans.py:12-30)
 *   devices  : p_c = compute[d].p_c, memory_bytes (src/profiling.py:125-156);
 *              `id_rank` = position of the device id in sorted string order
 *              (gateway tie-break, src/timing.py:104-113)
 *   links    : dense D x D matrices of p_t, latency_seconds and
 *              bandwidth_bytes_per_s (symmetric; diagonal unused)
 *   groups   : first-level groups in *string-sorted id order* (the order of
 *              sorted(groups.fgs), src/planner.py:384); members in
 *              member_device_ids order; second-level groups of each in
 *              sgs_by_fg order (src/grouping.py:21-39, src/timing.py:28-44)
 */
typedef struct gp_instance {
    uint32_t n_layers;
    const double *fwd_flops, *bwd_input_flops, *bwd_weight_flops;
    const double *activation_out_bytes, *param_bytes;
    uint32_t n_batch;            /* global_batch_candidates */
    const int64_t *batch;
    uint32_t n_micro;            /* microbatch_candidates   */
    const int64_t *micro;

    uint32_t n_devices;
    const double *p_c;
    const double *memory_bytes;
    const uint32_t *id_rank;
    const double *p_t;           /* [n_devices * n_devices] */
    const double *latency;       /* [n_devices * n_devices] */
    const double *bandwidth;     /* [n_devices * n_devices] */

    uint32_t n_fgs;
    const uint32_t *fg_member_offset;   /* [n_fgs + 1]  -> fg_members          */
    const uint32_t *fg_members;         /* device indices                       */
    const double *fg_capacity;          /* aggregate_capacity                   */
    const double *fg_min_bw;            /* min_intra_bandwidth                  */
    const uint8_t *fg_has_min_bw;       /* 0 where min_intra_bandwidth is None  */
    const uint32_t *fg_sg_offset;       /* [n_fgs + 1]  -> second-level groups  */
    const uint32_t *sg_member_offset;   /* [n_sgs + 1]  -> sg_members           */
    const uint32_t *sg_members;         /* device indices                       */
    const double *sg_capacity;          /* aggregate_capacity                   */

    double bottleneck_factor;           /* SearchConfig.bottleneck_factor       */
} gp_instance;

/* Result of an argmin over a candidate range (exhaustive_plan's `best`). */
typedef struct gp_best {
    double cost;           /* +inf when every candidate is memory-infeasible   */
    uint64_t index;        /* enumeration index of the winner (see below)      */
    uint32_t batch_index;  /* into gp_instance.batch                           */
    uint32_t micro_index;  /* into gp_instance.micro                           */
    uint32_t k;            /* number of stages                                 */
    uint8_t order[GP_MAX_STAGES];   /* fg indices (string order)               */
    uint8_t counts[GP_MAX_STAGES];  /* layers per stage                        */
    uint64_t evaluated;    /* candidates evaluated (exhaustive_plan.evaluated) */
} gp_best;

/* Full evaluation of one candidate (plan + CostBreakdown). */
typedef struct gp_stage_info {
    uint32_t kind;                    /* GP_UNIFORM ...                         */
    uint32_t n_parts;
    /* ASYM_PP: part i = (sg index within fg, layer_start, layer_end)          */
    uint32_t pp_sg[GP_MAX_SGS];
    uint32_t pp_start[GP_MAX_SGS];
    uint32_t pp_end[GP_MAX_SGS];
    double fill_seconds, run_seconds, residual_seconds, collective_seconds;
} gp_stage_info;

typedef struct gp_plan_info {
    int32_t feasible;                 /* memory_feasible (src/planner.py:248)   */
    uint32_t k;
    double plan_cost;                 /* +inf when infeasible                   */
    gp_stage_info stage[GP_MAX_STAGES];
} gp_plan_info;

/* Group constants of the TP x DP grid and DP splits (src/planner.py:107-154):
 * they depend on the group only, not on the layer range. */
typedef struct gp_group_info {
    int32_t tp_ok;                        /* rank-1 grid exists            */
    uint32_t n_members, n_sgs;
    double tp_row[GP_MAX_MEMBERS];        /* row fraction, member order    */
    double tp_col[GP_MAX_MEMBERS];        /* column fraction               */
    double dp_fraction[GP_MAX_SGS];       /* second-level data fractions   */
} gp_group_info;

/*
 * One pipeline timing (PlanTiming, src/timing.py:47-101) for the 1F1B
 * simulator: per-stage seconds per sample and closing costs, per-boundary
 * gateway link and bytes per sample.  Boundary arrays use n_stages-1 slots.
 */
typedef struct gp_timing {
    uint32_t n_stages;                 /* S, 1..GP_MAX_STAGES            */
    uint32_t pad;
    int64_t batch, microbatch;         /* PlanTiming.batch / .microbatch */
    double fwd[GP_MAX_STAGES];         /* StageTiming.fwd_per_sample     */
    double bwd[GP_MAX_STAGES];         /* .bwd_per_sample                */
    double wgt[GP_MAX_STAGES];         /* .wgt_per_sample                */
    double sync[GP_MAX_STAGES];        /* .sync_seconds                  */
    double opt[GP_MAX_STAGES];         /* .opt_seconds                   */
    double lat[GP_MAX_STAGES];         /* BoundaryTiming.latency_seconds */
    double bw[GP_MAX_STAGES];          /* .bandwidth_bytes_per_s         */
    double act[GP_MAX_STAGES];         /* .act_bytes_per_sample          */
    double grad[GP_MAX_STAGES];        /* .grad_bytes_per_sample         */
} gp_timing;

/* schedule policies (src/engine.py:48-52) */
enum { GP_POLICY_GPIPE = 0, GP_POLICY_1F1B = 1, GP_POLICY_ZB_ORIGINAL = 2, GP_POLICY_ZB_COMPACT = 3 };

#define GP_MAX_BREAKPOINTS 256
/* NetworkTrace (src/nettrace.py:12-45) restricted to the plan's boundary
 * links "b-(b+1)": per boundary b, n_points[b] breakpoints (t, multiplier)
 * sorted by strictly increasing t; the multiplier before the first one is 1. */
typedef struct gp_trace {
    uint32_t n_points[GP_MAX_STAGES];
    double t[GP_MAX_STAGES][GP_MAX_BREAKPOINTS];
    double mult[GP_MAX_STAGES][GP_MAX_BREAKPOINTS];
} gp_trace;

/* SimConfig knobs beyond the iteration count (src/simulator.py:21-28,
 * src/adapter.py:127-130): the DynamicBatchAdapter and asynchronous
 * iterations (src/engine.py:297-314). */
typedef struct gp_sim_options {
    uint32_t adapter;             /* adapter_enabled                         */
    uint32_t async_iterations;    /* SimConfig.async_iterations              */
    double degrade_factor;        /* AdapterConfig.degrade_factor (1.2)      */
    double recover_factor;        /* AdapterConfig.recover_factor (1.05)     */
} gp_sim_options;

/* One executed operation (PipeOp, src/engine.py:55-64); kinds F, B, W,
 * SYNC, OPT = 0..4 (OpKind "F","B","W","S","O"). */
typedef struct gp_op {
    double start, end;
    int32_t size;
    int32_t microbatch_id;        /* -1 for None (sync / optimizer step)     */
    uint32_t iteration;
    uint8_t kind, stage;
    uint16_t pad;
} gp_op;

/* One finished transfer (TransferRecord, src/engine.py:67-76); link_id is
 * the plan's boundary link, direction 0 "fwd", 1 "bwd". */
typedef struct gp_transfer {
    double start, end;
    int32_t size, microbatch_id;
    uint32_t iteration;
    uint8_t boundary, direction;
    uint16_t pad;
} gp_transfer;

/* One adapter resize (AdapterAction, src/adapter.py:116-124); signal 0
 * "fill", 1 "drain", 2 "degraded", 3 "recovered". */
typedef struct gp_action {
    double t;
    int32_t stage, old_size, new_size;
    uint32_t signal;
} gp_action;

/* One validate_schedule violation (src/schedule.py:95-171); the message
 * text is formatted by the host from these fields.  Codes:
 * 0 op ends before it starts (stage, kind); 1 ops overlap (stage, t);
 * 2 F before its activation arrives; 3 B before F ends; 4 B before its
 * gradient arrives; 5 W before B ends (stage, microbatch, iteration);
 * 6 not one sync and one optimizer; 7 sync before last weight update;
 * 8 optimizer before sync ends (stage, iteration). */
typedef struct gp_violation {
    double t;
    uint32_t iteration;
    int32_t microbatch_id;
    uint8_t code, stage, kind, pad;
    uint32_t pad2;
} gp_violation;

/* Per-timing SimReport ingredients (src/simulator.py:84-113): the host
 * derives throughput, steady_throughput and bubble_fractions from these
 * exactly as simulate_timing does. */
typedef struct gp_sim_report {
    double makespan;
    double busy[GP_MAX_STAGES];   /* sum(op.end - op.start) per stage        */
    uint32_t adapter_actions;     /* len(adapter.actions)                    */
    uint32_t n_ops;               /* ops over all stages                     */
    uint32_t n_transfers;         /* len(result.transfers)                   */
    uint32_t pad;
} gp_sim_report;

typedef struct gp_ctx gp_ctx;

/* Version / capability probe (no device needed). */
const char *gp_version(void);
/* Message of the last failing call on this thread. */
const char *gp_last_error(void);

/* Create a context on CUDA device `device` (no data yet). */
int gp_ctx_create(int device, gp_ctx **out);
/* Stage an instance into HBM and build the per-(group, layer-range) tables
 * (kernel K1).  Re-callable: a new instance replaces the old one. */
int gp_ctx_load(gp_ctx *ctx, const gp_instance *inst);
void gp_ctx_destroy(gp_ctx *ctx);

/*
 * Explicit batch (kernel K2): candidate i is stage order order[i*k .. i*k+k),
 * layer counts counts[i*k .. i*k+k) and (b, m) pair
 * bm[i] = batch_index * n_micro + micro_index.  Writes cost[i] (+inf when
 * memory-infeasible, as _evaluate's INFEASIBLE) and status[i] (GP_OK or the
 * per-candidate error the reference would raise).  Host pointers.
 */
int gp_eval_batch(gp_ctx *ctx, uint32_t k, uint64_t n,
                  const uint8_t *order, const uint8_t *counts,
                  const uint8_t *bm, double *cost, uint8_t *status);
/* Same with device pointers, asynchronous on the context's stream. */
int gp_eval_batch_device(gp_ctx *ctx, uint32_t k, uint64_t n,
                         const uint8_t *d_order, const uint8_t *d_counts,
                         const uint8_t *d_bm, double *d_cost,
                         uint8_t *d_status);

/*
 * Exhaustive enumeration (kernel K3).  Index space, as exhaustive_plan walks
 * it (src/planner.py:389-392): idx = (bm * k! + perm_rank) * C(n-1, k-1)
 * + comp_rank with bm = batch_index * n_micro + micro_index, permutations of
 * all fgs in lexicographic order and compositions in lexicographic order.
 * Returns the argmin over [lo, hi) of the reference key
 * (cost, (order, cuts)) with earliest-index tie-break.
 * gp_space_size() gives the total count.
 */
/*
 * Arg-min over a batch evaluated by gp_eval_batch_device (device pointers,
 * asynchronous on the context stream): the least (cost, key) over the n
 * candidates with status 0, key = d_keys[i] (u64; e.g. the enumeration
 * index of a sampled candidate) or i when d_keys is NULL, written to d_out
 * as {cost bits, key} (2 x u64, device memory); {+inf bits, ~0} when no
 * candidate has status 0.  The min over a candidate list the reference
 * takes in _evaluate's callers (src/planner.py:313-327), keyed for a
 * deterministic tie-break across shards.
 */
int gp_argmin_batch_device(gp_ctx *ctx, uint64_t n, const double *d_cost, const uint8_t *d_status,
                           const uint64_t *d_keys, uint64_t *d_out);

int gp_space_size(gp_ctx *ctx, uint64_t *out);
int gp_argmin_range(gp_ctx *ctx, uint64_t lo, uint64_t hi, gp_best *out);
/* Same result as gp_argmin_range over the whole space, by exact
 * branch-and-bound with min-max DP bounds (kernel K4): for large stage
 * counts where enumeration explodes.  Read with gp_argmin_fetch. */
int gp_argmin_bnb_async(gp_ctx *ctx);
/* Asynchronous variant writing the per-launch result to device memory
 * (benchmarks / multi-GPU reduction); read with gp_argmin_fetch. */
int gp_argmin_range_async(gp_ctx *ctx, uint64_t lo, uint64_t hi);
/* Arg-min over the (micro-batch, stage order) items [item_lo, item_hi),
 * item = micro_index * k! + order rank, all batch sizes and cuts included:
 * the unit of multi-GPU sharding (the union over ranks of disjoint item
 * ranges is the whole exhaustive space).  Read with gp_argmin_fetch; the
 * returned index is the global enumeration index. */
int gp_argmin_items_async(gp_ctx *ctx, uint64_t item_lo, uint64_t item_hi);
/* Result of the last asynchronous arg-min.  When a candidate of the range
 * raises (its status is returned), out->index is the enumeration index of
 * the first such candidate, so that a multi-GPU caller can order the ranks'
 * errors as the reference's sequential loop would meet them. */
int gp_argmin_fetch(gp_ctx *ctx, gp_best *out);

/* One-call exact re-plan: arg-min over [lo, hi) and the winner's splits +
 * CostBreakdown, decoded on the device; a single device->host copy and one
 * synchronisation.  `info` may be NULL. */
int gp_solve(gp_ctx *ctx, uint64_t lo, uint64_t hi, gp_best *best, gp_plan_info *info);

/* Full exact re-plan of an instance in one call: H2D of the instance, table
 * build, exhaustive arg-min and winner detail, replayed as one CUDA graph for
 * every instance of the same shape (layers, devices, group structure,
 * (b, m) candidates).  Equivalent to gp_ctx_load + gp_solve(0, total). */
int gp_replan(gp_ctx *ctx, const gp_instance *inst, gp_best *best, gp_plan_info *info);

/* Splits + CostBreakdown of one candidate (the winner), on the device. */
int gp_plan_detail(gp_ctx *ctx, uint32_t k, const uint8_t *order,
                   const uint8_t *counts, uint32_t bm, gp_plan_info *out);

/* TP tiles / DP fractions of group f, computed on the device. */
int gp_group_splits(gp_ctx *ctx, uint32_t f, gp_group_info *out);

/*
 * Bandwidth snapshot: replace bandwidth_bytes_per_s of every link with
 * bandwidth[u*D+v] (p_t and latency unchanged) and recompute each group's
 * min_intra_bandwidth and the boundary tables on the device.
 */
int gp_set_bandwidth(gp_ctx *ctx, const double *bandwidth);

/*
 * 1F1B makespans (kernel K5): makespan[i] = simulate_timing(timings[i],
 * Policy.ONE_F_ONE_B, CONSTANT_TRACE, adapter_enabled=False,
 * SimConfig(iterations)).makespan; status[i] = GP_OK or GP_ERR_SCHEDULING /
 * GP_ERR_TIMING.  Host pointers; the context need not be loaded.
 */
int gp_sim_1f1b(gp_ctx *ctx, const gp_timing *timings, uint64_t n, uint32_t iterations,
                double *makespan, uint8_t *status);
/*
 * Makespans under any schedule policy and network trace:
 * simulate_timing(timings[i], policy, trace, adapter_enabled=False,
 * SimConfig(iterations)).makespan with trace = traces[trace_index[i]]
 * (constant trace when traces is NULL / n_traces == 0; trace_index NULL
 * means trace 0 for every timing).  Host pointers.
 */
int gp_simulate(gp_ctx *ctx, const gp_timing *timings, uint64_t n, uint32_t policy,
                uint32_t iterations, const gp_trace *traces, uint32_t n_traces,
                const uint32_t *trace_index, double *makespan, uint8_t *status);
/*
 * Full simulate_timing(timings[i], policy, trace, opts->adapter,
 * SimConfig(iterations, async_iterations, AdapterConfig(...))) reports:
 * report[i] as above and, when iteration_ends is not NULL,
 * iteration_ends[i*iterations + j] = result.iteration_ends[j].  Host
 * pointers.  Per-timing queues live in device scratch sized by the largest
 * batch (chunks shrink to one sample under the adapter).
 */
int gp_simulate_report(gp_ctx *ctx, const gp_timing *timings, uint64_t n, uint32_t policy,
                       uint32_t iterations, const gp_trace *traces, uint32_t n_traces,
                       const uint32_t *trace_index, const gp_sim_options *opts,
                       gp_sim_report *report, double *iteration_ends, uint8_t *status);
/*
 * Two-level device grouping per topology snapshot (kernel K7):
 * group_first_level(topology, threshold_net) and group_second_level(fg,
 * topology, threshold_compute) for every first-level group
 * (src/grouping.py:146-228).  Devices are given in string-sorted id order
 * (ClusterTopology.device_ids): p_t[s*D*D + u*D + v] is snapshot s's link
 * metric, bandwidth (may be NULL) its bytes/s for min_intra_bandwidth, p_c
 * shared.  Outputs, stride D per snapshot: fg_of[d] = index of d's group in
 * the reference's fg{i} order; sg_of[d] = index of its subgroup within the
 * group (fg{i}.sg{j}); fg_intra / fg_capacity / fg_min_bw per group
 * (intra_metric, aggregate_capacity, min_intra_bandwidth; NaN where the
 * reference has None); sg_capacity per subgroup in group-major order.
 * GP_ERR_INPUT for D == 0 (EmptyClusterError) or a threshold outside (0, 1).
 */
int gp_group_snapshots(gp_ctx *ctx, uint32_t D, uint32_t n_snap, const double *p_t,
                       const double *bandwidth, const double *p_c, double threshold_net,
                       double threshold_compute, uint16_t *fg_of, uint16_t *sg_of,
                       uint32_t *n_fg, uint32_t *n_sg, double *fg_intra, double *fg_capacity,
                       double *fg_min_bw, double *sg_capacity);

/*
 * The schedules themselves (generate_schedule / SimReport.schedule,
 * .transfers and .adapter_actions): timing i writes its ops, in per-stage
 * start order interleaved by start, to ops[op_offset[i] ..], its transfers,
 * in completion order, to transfers[xfer_offset[i] ..] and its adapter
 * actions to actions[action_offset[i] ..] (transfers / actions and their
 * offsets may be NULL).  Offsets come from gp_simulate_report's n_ops /
 * n_transfers / adapter_actions; a timing whose counts disagree reports
 * GP_ERR_INPUT.
 */
int gp_simulate_schedule(gp_ctx *ctx, const gp_timing *timings, uint64_t n, uint32_t policy,
                         uint32_t iterations, const gp_trace *traces, uint32_t n_traces,
                         const uint32_t *trace_index, const gp_sim_options *opts,
                         const uint64_t *op_offset, gp_op *ops, const uint64_t *xfer_offset,
                         gp_transfer *transfers, const uint64_t *action_offset,
                         gp_action *actions, uint8_t *status);

/*
 * validate_schedule(schedule_i, timings[i], tol) and the per-stage busy sums
 * of bubble_fraction (src/schedule.py:95-182) for a batch of schedules:
 * schedule i = ops[op_offset[i] .. op_offset[i+1]) (stage field decides the
 * stage list; order within a stage is list order), makespan[i].  Writes
 * n_violations[i] and the first max_violations records to
 * violations[i*max_violations ..]; busy[i*GP_MAX_STAGES + s] =
 * sum(op.end - op.start) over stage s (may be NULL).  Micro-batch ids must
 * be dense per (stage, iteration, kind) in list order, as the engine
 * produces them (else status GP_ERR_INPUT).
 */
int gp_validate_schedules(gp_ctx *ctx, const gp_timing *timings, uint64_t n,
                          const uint64_t *op_offset, const gp_op *ops, const double *makespan,
                          uint32_t iterations, double tol, uint32_t max_violations,
                          gp_violation *violations, uint32_t *n_violations, double *busy,
                          uint8_t *status);

/*
 * Group statistics and second level for a GIVEN first-level partition
 * (fg_of_in[d] = group index in sorted-member-tuple order, n_fg_in groups):
 * the FirstLevelGroup fields as group_first_level would build them and
 * group_second_level per group (SURVEY App. D region-grouping sweep).
 * Outputs as gp_group_snapshots for one snapshot.
 */
int gp_group_fixed(gp_ctx *ctx, uint32_t D, const double *p_t, const double *bandwidth,
                   const double *p_c, const uint16_t *fg_of_in, uint32_t n_fg_in,
                   double threshold_compute, uint16_t *sg_of, uint32_t *n_sg, double *fg_intra,
                   double *fg_capacity, double *fg_min_bw, double *sg_capacity);

/* Same with device pointers, asynchronous on the context's stream. */
int gp_sim_1f1b_device(gp_ctx *ctx, const gp_timing *d_timings, uint64_t n,
                       uint32_t iterations, double *d_makespan, uint8_t *d_status);

/*
 * 1F1B makespans of explicit candidates (same encoding as gp_eval_batch):
 * simulate(build_plan(...), ..., Policy.ONE_F_ONE_B,
 * SimConfig(iterations, opt_seconds)).makespan (src/simulator.py:116-128).
 * status GP_ERR_NO_FEASIBLE marks memory-infeasible plans.
 */
int gp_sim_candidates(gp_ctx *ctx, uint32_t k, uint64_t n, const uint8_t *order,
                      const uint8_t *counts, const uint8_t *bm, uint32_t iterations,
                      double opt_seconds, double *makespan, uint8_t *status);

/* One StageAssignment of an explicit plan (src/plans.py:84-95): group index
 * (sorted fg id order), layer range, split kind; for ASYMMETRIC_PP the parts
 * (subgroup index within the group, layer start, layer end). */
typedef struct gp_plan_stage {
    uint32_t fg, layer_start, layer_end, kind, n_parts;
    uint32_t pp_sg[GP_MAX_SGS], pp_start[GP_MAX_SGS], pp_end[GP_MAX_SGS];
} gp_plan_stage;

/*
 * plan_cost(plan, topology, model, groups, opt_seconds) (src/costmodel.py:92-100)
 * of an explicit plan with the splits it carries, and optionally its
 * build_plan_timing (src/timing.py:176-231) record.  out->stage[s] holds the
 * StageCost fields; status as build_plan_timing's exceptions.
 */
int gp_plan_cost(gp_ctx *ctx, uint32_t k, const gp_plan_stage *stages, int64_t batch,
                 int64_t microbatch, double opt_seconds, gp_plan_info *out, gp_timing *timing);

/*
 * PlanTiming of explicit candidates (build_plan_timing(build_plan(...),
 * topology, model, groups, opt_seconds), src/timing.py:176-231): timings[i]
 * for the candidate's plan as _evaluate builds it (splits chosen by
 * choose_intra_split).  status as _evaluate's errors; memory feasibility is
 * not checked (build_plan_timing does not check it).
 */
int gp_plan_timing(gp_ctx *ctx, uint32_t k, uint64_t n, const uint8_t *order,
                   const uint8_t *counts, const uint8_t *bm, double opt_seconds,
                   gp_timing *timings, uint8_t *status);

/*
 * Batched re-plan over bandwidth snapshots (kernel K6 + K3): for snapshot i,
 * bandwidth[i*D*D ..] replaces every link's bandwidth_bytes_per_s (p_t and
 * latency unchanged) and out[i] receives exhaustive_plan's arg-min on that
 * topology (min_intra_bandwidth re-derived as group_first_level would).
 * status[i] = GP_OK or the error exhaustive_plan would raise.  The loaded
 * instance is left unchanged.  When `bandwidth` lies in pinned (mapped) host
 * memory the device reads the entries it needs in place (zero-copy);
 * pageable memory is copied to the device first.  The buffer must not change
 * until the call returns (it is synchronous).
 */
int gp_replan_snapshots(gp_ctx *ctx, const double *bandwidth, uint32_t n_snap, gp_best *out,
                        int32_t *status);

/*
 * Device-pointer, asynchronous form of gp_replan_snapshots (the bench's and
 * the multi-GPU path's hot loop): d_bandwidth = n_snap D x D matrices in
 * device memory; per snapshot i, d_keys[2i] = the winner's cost (f64 bits)
 * and d_keys[2i+1] = its tie rank ((order rank * C(n-1,k-1) + cuts rank) *
 * |B||M| + (b, m) index; ~0 when empty), d_flags[i] != 0 when the snapshot's
 * tables raise (then gp_replan_snapshots gives its status).  Needs an
 * error-free loaded instance with k >= 3 (else GP_ERR_INPUT).
 */
int gp_replan_snapshots_async(gp_ctx *ctx, const double *d_bandwidth, uint32_t n_snap,
                              void *d_keys, uint32_t *d_flags);

/* Peer-memory all-gather of small per-rank records between the GPUs of one
 * box (replaces the NCCL all-gather of the per-snapshot winners of
 * gp_replan_snapshots_async).  Each rank allocates one
 * buffer of 256 + 2 * world * slot_bytes bytes (gp_peer_alloc: device
 * pointer + a 64-byte CUDA IPC handle to share), opens every other rank's
 * handle (gp_peer_open), then per gather (gp_peer_allgather, asynchronous on
 * the context stream) stores its slot_bytes (multiple of 16) from d_src into
 * slot `rank` of table (epoch & 1) of every rank's buffer over NVLink (table t
 * at byte 256 + t * world * slot_bytes), fences at system scope, bumps each
 * buffer's arrival counter (the first 8 bytes), and waits on the device until
 * its own counter reaches epoch * world (epoch = 1, 2, ...).  A rank must
 * consume epoch e's table (in stream order) before its gather of e + 1.
 * peer_bases[r] = rank r's buffer as seen from this rank. */
int gp_peer_alloc(gp_ctx *ctx, uint64_t bytes, void **d_ptr, void *ipc_handle);
int gp_peer_open(gp_ctx *ctx, const void *ipc_handle, void **d_ptr);
int gp_peer_close(gp_ctx *ctx, void *d_ptr, int owned);
int gp_peer_read(gp_ctx *ctx, const void *d_ptr, void *host, uint64_t bytes);  /* sync copy-out */
int gp_peer_allgather(gp_ctx *ctx, const void *d_src, uint64_t slot_bytes, uint32_t rank,
                      uint32_t world, void *const *peer_bases, uint64_t epoch);

/* Restore the loaded instance's link bandwidths and its GroupIndex
 * min_intra_bandwidth values after gp_set_bandwidth snapshots. */
int gp_reset_bandwidth(gp_ctx *ctx);

/* Stream the context uses (cudaStream_t), for event timing by callers. */
void *gp_ctx_stream(gp_ctx *ctx);

/* Diagnostics: measured FP64 DADD issue rate of `device` (ops/s), the
 * roofline denominator of the range kernel (bench.py). */
int gp_diag_fp64_peak(int device, double *dadd_per_second);
/* Diagnostics: when `enable`, gp_replan brackets its graph launch with CUDA
 * events; *last_graph_ms (optional) receives the device time of the last
 * timed graph (-1 before the first). */
int gp_diag_replan_timing(gp_ctx *ctx, int enable, double *last_graph_ms);
/* Diagnostics: host-side phases of the last timed gp_replan in microseconds:
 * [0] arena fill (+ shape check), [1] graph launch call, [2] wait for the
 * graph, [3] result decode. */
int gp_diag_replan_host(gp_ctx *ctx, double *host_us4);
/* Diagnostics: enable = 1 opens a window in which every exhaustive sweep
 * launch (K3 / K6) is bracketed by CUDA events on the context stream;
 * enable = 0 closes it and returns the launches' summed device time (ms)
 * and their count (the roofline's per-launch kernel duration). */
int gp_diag_kernel_timing(gp_ctx *ctx, int enable, double *total_ms, uint64_t *launches);
/* Diagnostics: drain the per-CTA kernel timeline of a -DGP_TIMELINE build
 * (records of 40 bytes: u64 entry, after-dependency-wait and exit
 * globaltimer ns; u32 kernel id, CTA, SM, pad).  Shipped builds return 0. */
int gp_diag_timeline(void *out, uint32_t cap, uint32_t *n);
/* Diagnostics: force the exhaustive kernel variant (-1 auto; 0 tables in
 * L1/L2; 1 one triangle in shared memory; 2 two triangles; 3 generic
 * status-tracking kernel).  Results are identical in every mode. */
int gp_ctx_set_k3_mode(gp_ctx *ctx, int mode);
/* Checked builds (make checked: -DGP_CHECKS, the device-side stand-in for
 * compute-sanitizer): *line = first failing device check's source line since
 * the last call (0 = none), then cleared; other builds set 0xFFFFFFFF. */
int gp_diag_checks(gp_ctx *ctx, uint32_t *line);
/* Parity tests (not a production path): until gp_diag_verify_end, every
 * exhaustive / snapshot launch (K3 sweep, sub-range and generic kernels, the
 * gp_replan graph, gp_replan_snapshots) uses its verify instantiation - the
 * same arithmetic source plus a store - and records each evaluated
 * candidate's cost at position g - lo, g = snapshot * space_size + index,
 * for g in [lo, lo + n).  Error candidates record a NaN whose low 4 bits are
 * the status code; unwritten slots hold the all-ones NaN pattern.
 * gp_diag_verify_end copies the n slots to `out` (may be NULL). */
int gp_diag_verify_begin(gp_ctx *ctx, uint64_t lo, uint64_t n);
int gp_diag_verify_end(gp_ctx *ctx, double *out);

#ifdef __cplusplus
}
#endif
#endif /* GEOPIPE_B200_H */
