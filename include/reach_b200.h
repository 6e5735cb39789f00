/*
 * reach_b200.h -- C ABI of the B200-native batched reachability primitive.
 *
 * This is the drop-in boundary for the reference's DT reachability hot path.
 * The reference (`/root/reference/proj/include/reach/`) is a header-only C++
 * template library with no FFI; its callers bind these C++ signatures:
 *
 *   dt_reach        (dt_reach.hpp:40-42)   ReachTube dt_reach(sys, x0, actions, prm)
 *   dt_reach_batch  (dt_reach.hpp:108-112) vector<ReachTube> dt_reach_batch(sys, x0s, seqs, prm)
 *   reach_with_splitting(engine = dt_reach) (refine.hpp:121-160) + split_box (refine.hpp:83-115)
 *   certify_tm_input (neural.hpp:342-394), crown_backward (neural.hpp:290-335)
 *
 * Each entry point below replaces one of those calls for a whole batch. The
 * network descriptor is the reference's `MLPNet<double>` flattened in the
 * order of `net_params` (neural.hpp:133-140): per layer the row-major weight
 * matrix (out x in) then the bias.  Per-sample failures are data (a status
 * code mapping 1:1 to the reference failure_reason strings, tube.hpp:30-34),
 * never exceptions; argument errors return REACH_E_INVALID_ARGUMENT where the
 * reference throws std::invalid_argument (dt_reach.hpp:43-47).
 *
 * No torch types appear here: plain pointers and sizes.  The same structs are
 * used by the CPU oracle (oracle/, test-only) so tests bind one layout.
 */
#ifndef REACH_B200_H
#define REACH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define REACH_B200_ABI_VERSION 1

/* Activation tags, as reach::Act (neural.hpp:18). */
enum reach_act { REACH_ACT_RELU = 0, REACH_ACT_TANH = 1, REACH_ACT_IDENTITY = 2 };

/* Call status. */
enum reach_status {
  REACH_OK = 0,
  REACH_E_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  REACH_E_CUDA = 2,             /* CUDA runtime / launch failure */
  REACH_E_UNSUPPORTED = 3,      /* shape outside the compiled kernel family */
  REACH_E_NO_DEVICE = 4,
  REACH_E_OOM = 5,
  REACH_E_NONFINITE = 6         /* reference: std::runtime_error of grad_forward / grad_fd / gradient_refine
                                   (non-finite objective or derivative) */
};

/* Per-sample tube status; reason strings via reach_tube_status_string(). */
enum reach_tube_status {
  REACH_TUBE_OK = 0,
  REACH_TUBE_NONFINITE_PREACT = 1, /* "relax_activation: non-finite preactivation" (neural.hpp:171) */
  REACH_TUBE_DIVERGED_CERT = 2,    /* "diverged certification" (dt_reach.hpp:65) */
  REACH_TUBE_DIVERGED_BOX = 3,     /* "diverged box" (dt_reach.hpp:98) */
  REACH_TUBE_CTL_FAILED = 4,       /* "controller certification failed: relax_activation: non-finite preactivation"
                                      (closed_loop.hpp:106-109) */
  REACH_TUBE_CTL_DIVERGED = 5,     /* "controller certification diverged" (closed_loop.hpp:111-114) */
  REACH_TUBE_REMAINDER = 6,        /* "remainder not contractive after max enlargements (reduce h)"
                                      (flowpipe_ct.hpp:200-210) */
  REACH_TUBE_PICARD_NONFINITE = 7, /* "poly_picard: non-finite coefficients" (flowpipe_ct.hpp:135) */
  REACH_TUBE_TME_INV = 8,          /* "tme_inv: range contains zero" (taylor_model.hpp:367-368) */
  REACH_TUBE_OTHER = 99            /* any other reference exception text */
};

/* Flags for the batch entry points. */
#define REACH_FLAG_DEVICE_PTRS 1 /* every pointer in args/out is a device pointer */
/* The reference's outward-rounding mode (g_outward_rounding, interval.hpp:19): not supported by the
 * device kernels (the reference's own worker threads ignore it too); requesting it
 * returns REACH_E_UNSUPPORTED instead of silently computing in round-to-nearest. */
#define REACH_FLAG_OUTWARD_ROUNDING 0x10
/* Precision mode (flags bits 8..11) of the DT engines (reach_dt_batch, reach_dtcl_batch,
 * reach_split_hull).  REACH_PREC_EXACT (default): the reference's arithmetic, bit for bit.
 * REACH_PREC_TC: the CROWN contractions Lambda_s . W_l (neural.hpp:326) on the int8 tensor
 * cores (tcgen05.mma kind::i8, Ozaki split into 7 slices, exact int32 accumulation); the
 * rigorous contraction-error bound widens the intercepts, so tubes stay sound and match the
 * exact mode to ~1e-9 relative.  Wide (CTA-per-sample) family only:
 * n <= 72, controller outputs <= 72, hidden widths <= 256. */
#define REACH_FLAG_PREC_MASK 0xF00
#define REACH_PREC_EXACT 0x000
#define REACH_PREC_TC 0x100
/* REACH_PREC_FUSED: the exact mode's kernels and operation order with every a*b+c contracted into
 * one fused multiply-add (DFMA, one rounding) -- about half the FP64 instructions of the CROWN
 * contractions and IBP.  Not bit-identical to the reference (which rounds twice); bounds match it
 * within the north_star's fp64 tolerance (measured ~1e-12 relative, tests/test_gpu_fused.py) and
 * enclose Monte-Carlo rollouts.  All DT engines (warp and wide families). */
#define REACH_PREC_FUSED 0x200

/* MLPNet<double> (neural.hpp:42-88), flattened. */
typedef struct reach_net_desc {
  int32_t n_layers;
  const int32_t* dims;  /* n_layers+1 entries: dims[0] = input dim, dims[l+1] = rows of layer l */
  const int32_t* acts;  /* n_layers entries (reach_act); the last must be IDENTITY (neural.hpp:54) */
  const double* params; /* per layer: W (dims[l+1] x dims[l], row-major) then b (dims[l+1]) */
} reach_net_desc;

/* dt_reach_batch arguments (dt_reach.hpp:31-36, 108-112). The DTSystem's
 * one-step map is the network over (x, u) with n + m inputs and n outputs. */
typedef struct reach_dt_args {
  int32_t batch;
  int32_t horizon;          /* H = actions.size() */
  int32_t n;                /* DTSystem::n */
  int32_t m;                /* DTSystem::m */
  int32_t window;           /* DTReachParams::window */
  int32_t rebuild_from_box; /* DTReachParams::rebuild_from_box */
  const double* x0_lo;      /* [batch][n] */
  const double* x0_hi;      /* [batch][n] */
  const double* actions;    /* [batch][H][m], or [H][m] when actions_shared */
  int32_t actions_shared;
} reach_dt_args;

/* Batch of ReachTube<double> (tube.hpp:12-35). Box k of sample b is
 * lo/hi[(b*(H+1) + k)*n + d] for k < n_boxes[b]; its time stamp is t = k.
 * Entries at k >= n_boxes[b] are left untouched. */
typedef struct reach_tube_out {
  double* lo;
  double* hi;
  int32_t* n_boxes;     /* [batch] ReachTube::steps() */
  int32_t* failed_step; /* [batch] ReachTube::failed_step (-1 if completed) */
  int32_t* status;      /* [batch] reach_tube_status */
} reach_tube_out;

/* reach_with_splitting(dt_reach engine, x0, SplitPlan) (refine.hpp:121-160). */
typedef struct reach_split_args {
  int32_t n, m, horizon, window, rebuild_from_box;
  const double* x0_lo;   /* [n] */
  const double* x0_hi;   /* [n] */
  const int32_t* counts; /* [n] SplitPlan::counts */
  const double* actions; /* [H][m], shared by every sub-box */
  int64_t part_begin;    /* shard range of sub-box indices [begin, end) */
  int64_t part_end;      /* <= 0 means "all parts" */
} reach_split_args;

/* Per-step hull over the sub-tubes of [part_begin, part_end).
 * lo/hi follow the reference reduction (box_hull in ascending index order,
 * interval.hpp:260): NaN entries of parts other than part 0 are skipped. */
typedef struct reach_hull_out {
  double* lo;            /* [H+1][n] */
  double* hi;            /* [H+1][n] */
  int32_t* box_diverged; /* [H+1] */
  int32_t* n_boxes;      /* [1] min over parts of steps() */
  int64_t* fail_key;     /* [1] (div_step << 40 | part << 8 | status), INT64_MAX if no part failed */
} reach_hull_out;

/* Reachability-aware MPC (mpc.hpp).  Constraint::Type (mpc.hpp:26-86). */
enum reach_constraint_type {
  REACH_CON_HALFSPACE_AVOID = 0, /* unsafe {y : a.y >= b} */
  REACH_CON_SPHERE_AVOID = 1,    /* unsafe open ball B(center, radius) */
  REACH_CON_BOX_STAY_IN = 2,     /* safe box [lo, hi] */
  REACH_CON_MAX_VOLUME = 3       /* width-sum budget vmax */
};

typedef struct reach_constraint {
  int32_t type;
  int32_t n_dims;        /* 0 = all state dims */
  const int32_t* dims;   /* [n_dims] */
  const double* a;       /* halfspace normal [k] */
  double b;              /* halfspace offset */
  const double* center;  /* sphere center [k] */
  double radius;
  const double* lo;      /* stay-in box [k] */
  const double* hi;
  double vmax;
} reach_constraint;

/* PlanProblem (mpc.hpp:115-142); the one-step map is the uploaded network. */
typedef struct reach_plan_problem {
  int32_t n, m, horizon, window, rebuild_from_box;
  const double* x_goal;     /* [n] */
  const double* q_weights;  /* [n] */
  const double* r_weights;  /* [m] */
  int32_t n_constraints;
  const reach_constraint* constraints;
  double penalty;           /* C */
  double diverged_margin;
  double eps;               /* planning radius around x0 */
  const double* u_lo;       /* [m] action box */
  const double* u_hi;
} reach_plan_problem;

/* SamplerConfig (mpc.hpp:220-234). */
typedef struct reach_sampler_config {
  int32_t population;
  double elite_frac;
  int32_t iterations;
  double init_std;
  double smoothing;
  int32_t refine_iters; /* reach_plan_cem: forward-dual gradient refinement; the reach_cem_* pieces: must be 0 */
  uint64_t seed;
} reach_sampler_config;

/* ----------------------------------------------------------------------- */
/* GPU product (libreach_b200.so).                                          */
typedef struct reach_ctx reach_ctx;
typedef struct reach_net reach_net;

int reach_abi_version(void);
const char* reach_tube_status_string(int32_t status);

int reach_ctx_create(int32_t device, reach_ctx** out);
int reach_ctx_destroy(reach_ctx* ctx);
/* Work is enqueued on this stream (cudaStream_t; NULL = the ctx's own). */
int reach_ctx_set_stream(reach_ctx* ctx, void* cuda_stream);

/* ---- Multi-GPU: one process (or host thread) per GPU, each with its own ctx.
 * Once a ctx has collectives, the batch entry points that the reference runs in
 * one parallel_for -- reach_split_hull, reach_cl_split_hull, reach_ct_split_hull
 * (refine.hpp:121-160) and reach_plan_cem / reach_plan_cem_ex (mpc.hpp:300-304) --
 * shard their batch over the ranks (contiguous part / candidate ranges) and
 * combine on the ctx stream: the hull with one all-reduce per buffer (min / max of
 * order-preserving keys -- exact and order independent), the CEM scores with one
 * all-gather per iteration.  Every rank passes the full problem and receives the
 * full result, bit-identical to the single-GPU call.
 *
 * Built-in NCCL (over NVLink / NVSwitch): rank 0 calls reach_nccl_unique_id, the
 * 128-byte id reaches every rank out of band, every rank calls
 * reach_ctx_init_nccl on its ctx.  NCCL is loaded at run time (dlopen of
 * libnccl.so.2), so the library has no link dependency on it.
 * User collectives: reach_ctx_set_collectives with callbacks that reduce /
 * gather device buffers ordered on the given stream (e.g. torch.distributed). */
#define REACH_DT_U64 0
#define REACH_DT_I32 1
#define REACH_DT_F64 2
#define REACH_OP_MIN 0
#define REACH_OP_MAX 1
typedef struct reach_collectives {
  int32_t rank;
  int32_t world;
  /* in-place all-reduce of `count` elements (REACH_DT_*, REACH_OP_*) at device pointer `buf` */
  int (*allreduce)(void* user, void* buf, size_t count, int32_t dtype, int32_t op, void* cuda_stream);
  /* all-gather: `count` elements per rank from `send` into `recv` ([world][count], rank order) */
  int (*allgather)(void* user, const void* send, void* recv, size_t count, int32_t dtype, void* cuda_stream);
  void* user;
} reach_collectives;
int reach_nccl_unique_id(uint8_t out_id[128]);
int reach_ctx_init_nccl(reach_ctx* ctx, const uint8_t unique_id[128], int32_t world, int32_t rank);
int reach_ctx_set_collectives(reach_ctx* ctx, const reach_collectives* coll); /* NULL: back to one GPU */
/* Blocking copy between host / device memory of this ctx's device (cudaMemcpyDefault). */
int reach_ctx_memcpy(reach_ctx* ctx, void* dst, const void* src, size_t bytes);
int reach_ctx_synchronize(reach_ctx* ctx);
const char* reach_ctx_last_error(const reach_ctx* ctx);
/* Number of kernels this ctx has launched so far. */
int64_t reach_ctx_launch_count(const reach_ctx* ctx);

/* Kernel timing: when enabled, the library brackets every main kernel
 * (the DT horizon kernel) with CUDA events on its stream; query the total
 * device time and launch count since the last query (synchronizes). */
int reach_ctx_enable_kernel_timing(reach_ctx* ctx, int32_t on);
int reach_ctx_kernel_time(reach_ctx* ctx, double* total_ms, int64_t* launches);

/* FP64 pipe ceilings of this device (TFLOP/s): DFMA (2 flops/instr) and the
 * DMUL+DADD mix the exact kernels issue (1 flop/instr).  Roofline denominators. */
int reach_measure_fp64_peak(reach_ctx* ctx, double* tflops_fma, double* tflops_muladd);

/* Profiling builds only (-DRB_PHASE_TIMING, libreach_b200_phase.so): clock64
 * cycles per DT-kernel phase summed over warps since the last call
 * (prepend, IBP, backward init, chains, GEMM, first-layer GEMM, tail, fold,
 * box, drain).  The product build returns REACH_E_UNSUPPORTED. */
int reach_debug_phase_cycles(reach_ctx* ctx, uint64_t* out, int32_t count);

// Test hook of the tensor-core contraction (not part of the reference API): one
// Ozaki int8 tcgen05 product D = A . B^T (A M x K, B N x K row-major, host
// pointers; N in 8..56, multiple of 8; K <= 256) with the per-element rigorous
// bound |A . B^T - D| <= bound.
// Test hook: cycles per tcgen05.mma.kind::i8 (M = 128, N, K = 32, SS) issued back to back by one thread.
int reach_debug_mma_rate(reach_ctx* ctx, int32_t count, int32_t N, int32_t naccum, double* cycles_per_mma);
int reach_debug_ozaki_gemm(reach_ctx* ctx, int32_t M, int32_t N, int32_t K, const double* A, const double* B,
                           double* D, double* bound);

/* Uploads an immutable network (SPEC: nets are values). */
int reach_net_upload(reach_ctx* ctx, const reach_net_desc* desc, reach_net** out);
int reach_net_free(reach_ctx* ctx, reach_net* net);

/* dt_reach_batch on the device. Host pointers (default) are copied in/out
 * inside the call; with REACH_FLAG_DEVICE_PTRS the call is stream-ordered
 * and returns without synchronizing. */
int reach_dt_batch(reach_ctx* ctx, const reach_net* net, const reach_dt_args* args,
                   const reach_tube_out* out, int32_t flags);

/* dt_interval_baseline (dt_reach.hpp:129-149): the naive per-step interval tube of the same one-step map
 * (freeze the action, interval_forward the box), the CLI's `reach-dt --baseline interval`.  Same
 * arguments and tube layout as reach_dt_batch (host pointers). */
int reach_dt_interval_baseline_batch(reach_ctx* ctx, const reach_net* net, const reach_dt_args* a,
                                     const reach_tube_out* out);


/* DT closed loop (the cl_reach stacking of closed_loop.hpp:
 * 118-153 on a discrete-time one-step network): per step u = ctl_crown(x_tm,
 * ctl) (neural.hpp:418), the symbolic state is stacked to [x; u] over the shared
 * variables (control remainder as a fresh diagonal block), the dynamics network
 * (n + l inputs -> n outputs) is certified on it, then re-seed / fold / box as
 * dt_reach.  args->m must be 0 (the control comes from the controller). */
int reach_dtcl_batch(reach_ctx* ctx, const reach_net* dyn, const reach_net* ctl, const reach_dt_args* args,
                     const reach_tube_out* out, int32_t flags);

/* reach_with_splitting(dt_reach) on the device: split, per-part horizon,
 * hull reduction, all without materializing per-part tubes.  The X0 box and
 * the counts are plan parameters and always HOST pointers; with
 * REACH_FLAG_DEVICE_PTRS the actions and every hull output are device
 * pointers and the call is stream-ordered. */
int reach_split_hull(reach_ctx* ctx, const reach_net* net, const reach_split_args* args,
                     const reach_hull_out* out, int32_t flags);

/* plan_eval (mpc.hpp:158-202) for a batch of action sequences from one x0:
 * objective[b] and diverged[b] (the tube's diverged flag) per candidate;
 * tubes (optional, may be NULL) receives the certified tubes.  Host pointers
 * unless REACH_FLAG_DEVICE_PTRS (then x0, actions, objective, diverged and
 * the tube arrays are device pointers; the problem struct stays on the host). */
int reach_plan_eval_batch(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* prob, const double* x0,
                          int32_t batch, const double* actions, double* objective, int32_t* diverged,
                          const reach_tube_out* tubes, int32_t flags);

/* plan_cem (mpc.hpp:258-368): the reference's sequential mt19937_64 /
 * Box-Muller sampling on the host, every population evaluated by
 * reach_plan_eval_batch, stable-sort elite refit on the host, then (for
 * refine_iters > 0, the reference default 5) gradient_refine of the best
 * candidate (refine.hpp:347-398) with forward-dual gradients computed on the
 * device (reach_plan_objective_grad).  best_actions [H][m], best_history
 * [iterations], best_effort flag, and the final plan's tube (batch 1,
 * optional).  A non-finite dual derivative is REACH_E_NONFINITE, where
 * the reference's grad_forward throws. */
int reach_plan_cem(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* prob,
                   const reach_sampler_config* cfg, const double* x0, double* best_actions, double* objective,
                   double* best_history, int32_t* best_effort, const reach_tube_out* final_tube);
/* As reach_plan_cem, plus PlanResult::refined (mpc.hpp:241): the refinement made progress. */
int reach_plan_cem_ex(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* prob,
                      const reach_sampler_config* cfg, const double* x0, double* best_actions, double* objective,
                      double* best_history, int32_t* best_effort, int32_t* refined, const reach_tube_out* final_tube);

/* plan_cem's refinement step alone (mpc.hpp:337-361): gradient_refine of the plan objective from
 * best_actions [H][m] (the CEM result, objective best_objective), replaced in place when the refined
 * objective is lower; refined = PlanResult::refined.  For drivers running the CEM in pieces. */
int reach_plan_refine(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* prob, const double* x0,
                      int32_t refine_iters, double best_objective, double* best_actions, int32_t* refined);

/* grad_forward (refine.hpp:186-207) of plan_objective (mpc.hpp:204-208) over
 * the flat action sequence [H][m]: one reach::Dual pass per direction, all
 * directions in one launch.  grad [H*m]; objective (optional) = the primal. */
int reach_plan_objective_grad(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* prob, const double* x0,
                              const double* actions, double* grad, double* objective);

/* grad_tube_volume (refine.hpp:263-311): the gradient of tube_volume(dt_reach(sys, box_from_center(c, r),
 * actions, prm)) (tube.hpp:40-46) with respect to GradTarget (refine.hpp:240) -- the X0 centre (radii held
 * fixed; c, r = box_center / box_radius of [x0_lo, x0_hi]), the flat action sequence [H][m], or the one-step
 * map's parameters in net_params order (neural.hpp:133-140) -- by GradMethod (refine.hpp:165):
 * forward_dual (grad_forward: one reach::Dual pass per parameter, one CTA each) or finite_difference
 * (grad_fd: central differences, h = 1e-5 * max(1, |p_j|), 2 passes per parameter), all passes in one
 * launch.  `a` describes one tube (batch 1).  grad [dim]; subgradient = Gradient::subgradient (a ReLU
 * preactivation bound sat exactly at zero, neural.hpp:180); volume = the primal tube volume.  A
 * non-finite objective or derivative is REACH_E_NONFINITE (the reference throws std::runtime_error). */
enum reach_grad_target { REACH_GRAD_X0_CENTER = 0, REACH_GRAD_ACTIONS = 1, REACH_GRAD_WEIGHTS = 2 };
enum reach_grad_method { REACH_GRAD_FORWARD_DUAL = 0, REACH_GRAD_FINITE_DIFFERENCE = 1 };
int reach_grad_tube_volume(reach_ctx* ctx, const reach_net* net, const reach_dt_args* a, int32_t target,
                           int32_t method, double* grad, int32_t* subgradient, double* volume);
/* The passes of parameters [param_begin, param_end) only (param_end = -1: to the end); grad receives that
 * slice.  Multi-GPU drivers shard the parameters over ranks and all-gather the slices (the passes are
 * independent); the subgradient flag and the volume are per call. */
int reach_grad_tube_volume_range(reach_ctx* ctx, const reach_net* net, const reach_dt_args* a, int32_t target,
                                 int32_t method, int64_t param_begin, int64_t param_end, double* grad,
                                 int32_t* subgradient, double* volume);

/* mpc_run (mpc.hpp:373-495): receding-horizon execution.  MPCConfig (mpc.hpp:373-387). */
typedef struct reach_mpc_config {
  int32_t replan_period;  /* actions executed per plan */
  int32_t total_steps;
  double dist_action;     /* uniform noise bound on executed actions */
  double dist_state;      /* uniform noise bound on the next state */
  int32_t n_goal_dims;    /* 0 = all */
  const int32_t* goal_dims;
  double goal_radius;
  uint64_t seed;
} reach_mpc_config;
/* The true simulator x_next = sim(x, u); return 0 on success. */
typedef int (*reach_sim_fn)(void* user, const double* x, const double* u, double* x_next);
/* MPCResult::log (mpc.hpp:389-396), row-major, capacity total_steps rows; any pointer may be NULL. */
typedef struct reach_mpc_log {
  int32_t* step;
  double* state;        /* [rows][n] */
  double* action;       /* [rows][m] */
  double* objective;
  double* tube_volume;
  double* g_margin;
} reach_mpc_log;
/* Plans with reach_plan_cem_ex (seed = sampler.seed ^ (0x9e3779b97f4a7c15 * (step + 1))), executes
 * replan_period actions through `sim` (NULL: the uploaded one-step model's forward on the device, as the
 * reference CLI does) with the reference's disturbance stream, replans.  Outputs MPCResult's success,
 * violated, steps_used, final_state [n] and the log (log_rows rows). */
int reach_mpc_run(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* prob,
                  const reach_sampler_config* sampler, const reach_mpc_config* cfg, reach_sim_fn sim, void* sim_user,
                  const double* x0, int32_t* success, int32_t* violated, int32_t* steps_used, double* final_state,
                  const reach_mpc_log* log, int32_t* log_rows);

/* gradient_refine (refine.hpp:354-398; RefineParams defaults: step0 1, shrink 0.5, armijo 1e-4, 30
 * backtracks, forward_dual) of tube_volume(dt_reach(box_from_center(center, radius), actions)) over the X0
 * centre (target REACH_GRAD_X0_CENTER, dim n) or the flat action sequence (REACH_GRAD_ACTIONS, dim H*m),
 * inside [lo, hi] -- the reference CLI's `refine` objective.  `a` gives n, m, H, DTReachParams and the
 * actions (x0_lo / x0_hi unused).  x [dim]: start point in, refined point out; RefineResult's fields out.
 * A non-finite initial objective or derivative is REACH_E_NONFINITE. */
int reach_refine_tube_volume(reach_ctx* ctx, const reach_net* net, const reach_dt_args* a, const double* center,
                             const double* radius, int32_t target, const double* lo, const double* hi,
                             int32_t iters, double* x, double* initial_objective, double* objective,
                             int32_t* progressed, int32_t* subgradient, int32_t* accepted_steps);

/* reach_loss (training.hpp:99-126): the certified-training reachability regularizer of a batch of
 * `episodes` episodes, (1/M) sum_m [tube diverged ? cap : log(1 + predicted_volume(dt_reach(
 * box_from_center(x0_m, eps), first H actions)))], and (grad != NULL) its gradient over the one-step
 * model's parameters in net_params order -- grad_forward's Dual passes, one CTA per (parameter, episode),
 * all in one launch.  a->x0_lo = the episode start states [M][n], a->actions [M][H][m], a->horizon = t_h
 * (x0_hi, batch unused).  diverged_count = the episodes charged the cap. */
int reach_reach_loss(reach_ctx* ctx, const reach_net* net, const reach_dt_args* a, int32_t episodes,
                     double eps, double cap, double* loss, double* grad, int32_t* diverged_count);

/* Certified training (training.hpp).  An episode set of `episodes` rollouts of one length T:
 * states [episodes][T+1][n], actions [episodes][T][m] (Episode, training.hpp:28-45). */
typedef struct reach_episode_set {
  int32_t episodes, length, n, m;
  const double* states;
  const double* actions;
  int32_t ref_dim;      /* per-step references y_ref [episodes][T][ref_dim] (controller training), */
  const double* y_ref;  /* or ref_dim = 0 / NULL: none */
} reach_episode_set;

/* pred_loss (training.hpp:60-83) of the first t_h steps of every episode of `batch` under the one-step
 * model `net` with weights [t_h], and (grad != NULL) its grad_forward over net_params (neural.hpp:133-140):
 * one Dual rollout per (parameter, episode) on the device, terms summed in the reference's order. */
int reach_pred_loss(reach_ctx* ctx, const reach_net* net, const reach_episode_set* batch, int32_t t_h,
                    const double* weights, double* loss, double* grad);

/* track_loss (training.hpp:134-178) of a controller `ctl` against logged (state, action) pairs with the
 * plant `plant` (REACH_PLANT_QUADROTOR, params {mass, gravity, jx, jy, jz}) advanced by rk4_substeps fixed
 * RK4 steps per control interval delta, and (grad != NULL) its grad_forward over the controller's
 * net_params: one Dual rollout per (parameter, episode) on the device.  blowup_count = episodes charged
 * the cap. */
int reach_track_loss(reach_ctx* ctx, const reach_net* ctl, int32_t plant, const double* plant_params,
                     const reach_episode_set* batch, int32_t t_t, const double* weights, double gamma, double delta,
                     int32_t rk4_substeps, double cap, double* loss, double* grad, int32_t* blowup_count);

/* TrainConfig (training.hpp:262-282) and one TrainLog row (:284-292). */
typedef struct reach_train_config {
  int32_t horizon_max;
  double eps0, eps_final, lambda, gamma;
  int32_t iters, batch;
  double lr, reach_cap;
  int32_t curriculum;
  uint64_t seed;
  int32_t window, rebuild_from_box; /* cfg.dt_prm */
} reach_train_config;
typedef struct reach_train_log_row {
  int32_t iter, t_h;
  double eps, l_pred, l_reach, l_total;
  int32_t diverged_count;
} reach_train_log_row;

/* train_dt_dyn (training.hpp:333-382): certified training of a DT dynamics net, L = pred_loss +
 * lambda reach_loss with the horizon / radius curriculum, the reference's minibatch stream (Rng(seed),
 * uniform_int) and Adam on the host; every loss and every gradient (grad_forward: pred_loss and
 * reach_loss Dual passes) on the device.  params_out [param_count] = the trained net_params;
 * log [iters] rows.  REACH_E_NONFINITE where the reference throws std::runtime_error (non-finite loss
 * or derivative; ctx error string = the reference's message). */
int reach_train_dt_dyn(reach_ctx* ctx, const reach_net_desc* init, const reach_train_config* cfg,
                       const reach_episode_set* dataset, double* params_out, reach_train_log_row* log);

/* The CEM loop in pieces, for multi-GPU drivers that shard each population
 * and all-gather the scores between sample() and update(). */
typedef struct reach_cem reach_cem;
int reach_cem_create(const reach_plan_problem* prob, const reach_sampler_config* cfg, reach_cem** out);
int reach_cem_destroy(reach_cem* cem);
/* Draws iteration `it`'s population into candidates [population][H][m]. */
int reach_cem_sample(reach_cem* cem, double* candidates);
/* Consumes the scores / ok flags of the population drawn last. */
int reach_cem_update(reach_cem* cem, const double* scores, const int32_t* ok);
/* best actions [H][m], best objective, best_effort, history [iterations so far] */
int reach_cem_result(const reach_cem* cem, double* best_actions, double* best_objective, int32_t* best_effort,
                     double* best_history);

/* ----------------------------------------------------------------------- */
/* Continuous-time closed loop under zero-order-hold neural feedback        */
/* (cl_reach, closed_loop.hpp:76-182): controller certification at control  */
/* boundaries (ctl_crown, neural.hpp:418-424) + stacking, then k_atomic     */
/* validated Taylor-model flowpipe steps of the augmented (x, u) field       */
/* (poly_picard / remainder_picard / symbolic_step, flowpipe_ct.hpp).        */
/* The plant is an analytic system from systems.hpp, evaluated on the       */
/* device; VectorField's host std::function closures cannot run there, so   */
/* an unknown plant is REACH_E_UNSUPPORTED, never a CPU fallback.           */

/* Analytic plants (systems.hpp), augmented with udot = 0 rows (fields.hpp:96-128). */
enum reach_plant {
  REACH_PLANT_QUADROTOR = 0 /* quadrotor_ode (systems.hpp:22-64): n = 12, l = 4;
                               params = {mass, gravity, jx, jy, jz} (QuadrotorParams) */
};

/* FlowpipeParams (flowpipe_ct.hpp:35-50). `steps` is not used by cl_reach. */
typedef struct reach_flowpipe_params {
  double h;
  int32_t steps;
  int32_t order;            /* Picard truncation order k, 1 or 2 */
  double eps_init;
  int32_t refine_rounds;
  double enlargement;
  int32_t max_enlargements;
  int32_t window;
} reach_flowpipe_params;

/* ClosedLoopSpec<double> (closed_loop.hpp:16-44) with an analytic plant. */
typedef struct reach_cl_spec {
  int32_t plant;            /* reach_plant */
  double plant_params[8];
  int32_t n, l;             /* state / control dims; the controller maps n + ref_dim -> l */
  int32_t ctl_steps;        /* control intervals */
  int32_t k_atomic;         /* flowpipe steps per control interval */
  int32_t ref_dim;          /* 0: no reference input */
  const double* y_ref;      /* [ctl_steps][ref_dim], host pointer */
  reach_flowpipe_params fp;
  int32_t intervalize_boundary;
} reach_cl_spec;

/* cl_reach for a batch of initial boxes.  Tubes have up to
 * 1 + ctl_steps * k_atomic boxes of n + l dims: box 0 is the augmented
 * initial set, box k >= 1 covers [(k-1) h, k h]; lo/hi are
 * [batch][1 + ctl_steps*k_atomic][n + l]. */
int reach_cl_batch(reach_ctx* ctx, const reach_net* ctl, const reach_cl_spec* spec, int32_t batch,
                   const double* x0_lo, const double* x0_hi, const reach_tube_out* out, int32_t flags);

/* reach_with_splitting(cl_reach engine, x0, SplitPlan) (refine.hpp:121-160):
 * the per-step hull over the sub-boxes [part_begin, part_end) of the grid
 * split of X0 (n dims, e.g. SplitPlan::rpy, refine.hpp:51-61).  Hull boxes:
 * [1 + ctl_steps*k_atomic][n + l].  X0 and counts are host pointers. */
typedef struct reach_cl_split_args {
  const double* x0_lo;   /* [n] */
  const double* x0_hi;   /* [n] */
  const int32_t* counts; /* [n] */
  int64_t part_begin;
  int64_t part_end;      /* <= 0 means "all parts" */
} reach_cl_split_args;

int reach_cl_split_hull(reach_ctx* ctx, const reach_net* ctl, const reach_cl_spec* spec,
                        const reach_cl_split_args* args, const reach_hull_out* out, int32_t flags);

/* ----------------------------------------------------------------------- */
/* Open-loop continuous-time flowpipe (ct_reach, flowpipe_ct.hpp:428-458) of */
/* an analytic VectorField from fields.hpp: box 0 is X0, box k >= 1 covers  */
/* [(k-1) h, k h]; the symbolic state's G0 is square, so fold_overflow uses  */
/* the G0^-1 Q solve (flowpipe_ct.hpp:326-346, linalg.hpp:96-132).          */
enum reach_ct_field {
  REACH_FIELD_ZERO = 0,        /* zero_field(n) (fields.hpp:87-92): params unused */
  REACH_FIELD_DIAG_LINEAR = 1, /* diag_linear_field(lambda) (fields.hpp:72-78): params = lambda[n] */
  REACH_FIELD_ROTATION = 2,    /* rotation_field(w) (fields.hpp:80-85), n = 2: params = {w} */
  REACH_FIELD_QUADROTOR = 3    /* quadrotor_field(prm, u) (fields.hpp:51-56), n = 12:
                                  params = {mass, gravity, jx, jy, jz, u0, u1, u2, u3} */
};

typedef struct reach_field_desc {
  int32_t kind; /* reach_ct_field */
  int32_t n;
  double params[16];
} reach_field_desc;

/* ct_reach for a batch of initial boxes [batch][n]; tubes of up to
 * 1 + fp.steps boxes of n dims (lo/hi [batch][1 + steps][n]).
 * Limits of the device family: n * (fp.window + 2) <= 80, n <= 16. */
int reach_ct_batch(reach_ctx* ctx, const reach_field_desc* field, const reach_flowpipe_params* fp, int32_t batch,
                   const double* x0_lo, const double* x0_hi, const reach_tube_out* out, int32_t flags);

/* reach_with_splitting(ct_reach engine, x0, plan) (refine.hpp:121-160; the
 * CLI's `reach-ct --split` / `split`, reach_cli.cpp:200-211): hull boxes
 * [1 + fp.steps][n] over the sub-boxes [part_begin, part_end). */
int reach_ct_split_hull(reach_ctx* ctx, const reach_field_desc* field, const reach_flowpipe_params* fp,
                        const reach_cl_split_args* args, const reach_hull_out* out, int32_t flags);

/* ctl_reach_loss (training.hpp:183-213) with the quadrotor plant: (1/M) sum_e [tube diverged ? cap :
 * log(1 + predicted_volume(cl_reach(spec, box_from_center(x0_e, eps))))] with spec->ctl_steps = t_h,
 * spec->fp.h = delta / k_atomic, and (grad != NULL) its grad_forward over the controller's net_params:
 * one Dual cl_reach per (parameter, episode) on the device (warp per pass, working set in shared
 * memory).  x0s [M][n]; y_refs [M][ctl_steps][ref_dim] per episode (spec->y_ref unused), NULL when
 * spec->ref_dim = 0.  diverged_count = episodes charged the cap. */
int reach_ctl_reach_loss(reach_ctx* ctx, const reach_net* ctl, const reach_cl_spec* spec, int32_t episodes,
                         const double* x0s, const double* y_refs, double eps, double cap, double* loss, double* grad,
                         int32_t* diverged_count);

/* train_ct_ctl (training.hpp:389-442): certified training of a controller against the quadrotor plant
 * (base: plant, params, n, l, k_atomic, fp_base, ref_dim), L = track_loss (rk4_substeps RK4 steps per
 * control interval delta) + lambda ctl_reach_loss (cl_reach with fp.h = delta / k_atomic), the
 * reference's curriculum / minibatch stream / Adam on the host, every loss and gradient on the device.
 * dataset: states [E][T+1][12], actions [E][T][4] (logged controls), y_ref [E][T][ref_dim]. */
int reach_train_ct_ctl(reach_ctx* ctx, const reach_net_desc* init, const reach_train_config* cfg,
                       const reach_episode_set* dataset, const reach_cl_spec* base, double delta,
                       int32_t rk4_substeps, double* params_out, reach_train_log_row* log);

#ifdef __cplusplus
}
#endif

#endif /* REACH_B200_H */
