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
  REACH_E_OOM = 5
};

/* Per-sample tube status; reason strings via reach_tube_status_string(). */
enum reach_tube_status {
  REACH_TUBE_OK = 0,
  REACH_TUBE_NONFINITE_PREACT = 1, /* "relax_activation: non-finite preactivation" (neural.hpp:171) */
  REACH_TUBE_DIVERGED_CERT = 2,    /* "diverged certification" (dt_reach.hpp:65) */
  REACH_TUBE_DIVERGED_BOX = 3,     /* "diverged box" (dt_reach.hpp:98) */
  REACH_TUBE_OTHER = 99            /* any other reference exception text */
};

/* Flags for the batch entry points. */
#define REACH_FLAG_DEVICE_PTRS 1 /* every pointer in args/out is a device pointer */

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

/* Uploads an immutable network (SPEC: nets are values). */
int reach_net_upload(reach_ctx* ctx, const reach_net_desc* desc, reach_net** out);
int reach_net_free(reach_ctx* ctx, reach_net* net);

/* dt_reach_batch on the device. Host pointers (default) are copied in/out
 * inside the call; with REACH_FLAG_DEVICE_PTRS the call is stream-ordered
 * and returns without synchronizing. */
int reach_dt_batch(reach_ctx* ctx, const reach_net* net, const reach_dt_args* args,
                   const reach_tube_out* out, int32_t flags);

/* reach_with_splitting(dt_reach) on the device: split, per-part horizon,
 * hull reduction, all without materializing per-part tubes.  The X0 box and
 * the counts are plan parameters and always HOST pointers; with
 * REACH_FLAG_DEVICE_PTRS the actions and every hull output are device
 * pointers and the call is stream-ordered. */
int reach_split_hull(reach_ctx* ctx, const reach_net* net, const reach_split_args* args,
                     const reach_hull_out* out, int32_t flags);

#ifdef __cplusplus
}
#endif

#endif /* REACH_B200_H */
