/*
 * lars_b200.h -- C ABI of the B200 LARS data-parallel step library
 * (liblars_b200.so, built for sm_100a).
 *
 * Everything here replaces one piece of the reference optimizer step of
 * `batchlab` (arXiv 1709.05011 reference, Python/numpy fp64), cited as
 * pkg/src/batchlab/<file>:<line>:
 *
 *   lars_step           optim.apply_update (optim.py:117-134) incl.
 *                       lars_local_lr / group_local_lr (optim.py:98-114) and,
 *                       unless LARS_STEP_EXPLICIT_LR, scheduled_lr
 *                       (optim.py:76-95) and the iteration advance of
 *                       sgd_step (optim.py:137-142); plus the `/ B` gradient
 *                       averaging of cluster.global_step (cluster.py:147-148)
 *                       through hp->grad_scale.
 *   lars_partial_norms  the two np.linalg.norm reductions of lars_local_lr
 *   + lars_update       (optim.py:100-101), split so that a sharded step can
 *                       all-reduce per-layer partial sums of squares between
 *                       them (the reference holds whole layers on every
 *                       replica, cluster.py:151-153, so it has no such split).
 *   lars_step_peer      cluster.global_step's all_reduce + `/ b` + the update
 *   (+ _stream)         on every replica (cluster.py:146-153) as ONE kernel per
 *                       rank over NVLink peer memory (reduce-scatter, norm
 *                       exchange, update, all-gather).
 *   lars_host_*         the reference ParamSet's storage (one fp64 numpy
 *                       array per group, mutated in place, nn.py:63-114):
 *                       DMA to / from the flat fp32 buffers.
 *
 * There is no C ABI in the reference; its boundary is the Python call
 * optim.sgd_step(params, hp, st) / optim.apply_update(params, hp, lr, it).
 * The Python package paper_1709_05011_b200 re-exposes exactly those
 * signatures on top of this library (INTEGRATION.md shows the ctypes binding).
 *
 * Conventions
 *  - Every function returns 0 (LARS_OK) or an error code: codes below 1000
 *    are LARS_ERR_*, codes >= 1000 are 1000 + cudaError_t.  lars_strerror()
 *    names both.  No C++ exception crosses the ABI.
 *  - Buffers are caller-owned device memory; step calls never allocate and
 *    are asynchronous on `stream` (a cudaStream_t, NULL = legacy default),
 *    so they can be captured into a CUDA graph.
 *  - One host thread per plan at a time (the reference: "callers must
 *    serialize steps per ParamSet").
 *  - Parameter, gradient and momentum buffers are fp32, 16-byte aligned;
 *    norms, trust ratios and the learning rate are fp64 like the reference.
 */
#ifndef LARS_B200_H
#define LARS_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define LARS_API __attribute__((visibility("default")))
#else
#define LARS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define LARS_ABI_VERSION 1

/* status codes */
#define LARS_OK 0
#define LARS_ERR_INVALID 1          /* bad argument / null pointer            */
#define LARS_ERR_ALIGNMENT 2        /* segment offset/length not a multiple of 4, or pointer not 16 B aligned */
#define LARS_ERR_LAYOUT 3           /* segments unsorted or overlapping       */
#define LARS_ERR_TOO_MANY_PIECES 4  /* a CTA's piece table exceeds shared memory */
#define LARS_ERR_NO_DEVICE 5        /* no CUDA device                         */
#define LARS_ERR_HOST_ONLY_PLAN 6   /* launch with a LARS_PLAN_HOST_ONLY plan */
#define LARS_ERR_HOST_MEMORY 7      /* host range could not be pinned for DMA */
#define LARS_ERR_CUDA_BASE 1000     /* 1000 + cudaError_t                     */

/* lars_segment_t.flags */
#define LARS_SEG_TRUST 1  /* layer takes the LARS trust ratio: category not in
                             hp.lars_skip_categories (optim.py:22, 111-114)  */
#define LARS_SEG_SHARED 2 /* sharded plans: the layer also has elements in
                             other ranks' shards (its norms need their sums);
                             used by lars_step_peer_stream                   */

/* One contiguous range of one parameter group (layer) in the flat buffers.
 * Mirrors nn.ParamGroup (nn.py:63-69) minus the arrays, which live in the
 * flat w / g / m buffers at [offset, offset+length).  A layer may have zero-
 * length segments (they still carry its flags, so its lambda is reported). */
typedef struct {
  int64_t offset;  /* first element (multiple of 4)                         */
  int64_t length;  /* element count (multiple of 4; padding must hold zeros) */
  int32_t layer;   /* parameter-group index in [0, nlayers)                 */
  int32_t flags;   /* LARS_SEG_*                                           */
} lars_segment_t;

/* lars_hparams_t.flags */
#define LARS_STEP_EXPLICIT_LR 1  /* use hp->lr (optim.apply_update) instead of
                                    the on-device schedule (optim.sgd_step) */
#define LARS_STEP_USE_WCARRY 2   /* take ||w||^2 from the previous update's
                                    epilogue instead of re-reading w; valid
                                    only if w was not written since       */
#define LARS_STEP_ADVANCE_ITER 4 /* *d_iter += 1 after the step (optim.py:141) */

/* HyperParams (optim.py:25-36) + ScheduleState sizes (optim.py:58-62). */
typedef struct {
  double base_lr;
  double momentum;
  double weight_decay;
  double poly_power;
  double trust;        /* lars_trust                                        */
  double grad_scale;   /* gradient used = g * grad_scale (1/B for the
                          sum-convention gradient of cluster.py:147-148)    */
  double lr;           /* explicit lr for LARS_STEP_EXPLICIT_LR             */
  int64_t warmup_iters;/* warmup_epochs * iterations_per_epoch (optim.py:88) */
  int64_t max_iters;   /* ScheduleState.max_iterations                      */
  int32_t lars_enabled;
  int32_t flags;       /* LARS_STEP_*                                       */
} lars_hparams_t;

/* lars_step_info_t.status bits */
#define LARS_STATUS_EXHAUSTED 1  /* iteration > max_iters: nothing was
                                    written (ScheduleExhaustedError,
                                    optim.py:84-87)                          */
#define LARS_STATUS_RANK_TIMEOUT 2 /* lars_step_peer: a peer rank did not
                                    reach a cross-rank barrier within 60 s;
                                    the launch completed without it and its
                                    results are invalid                     */

/* Device-resident per-step results (read lazily by the host). */
typedef struct {
  double lr;               /* learning rate the step used                    */
  int64_t iteration;       /* iteration the step ran at                      */
  int32_t nonfinite_layer; /* smallest layer whose updated weights are not
                              finite, INT32_MAX if none (DivergenceError,
                              optim.py:132-133)                              */
  int32_t status;          /* LARS_STATUS_*                                  */
} lars_step_info_t;

/* lars_plan_create flags */
#define LARS_PLAN_HOST_ONLY 1  /* build the partition only (no device upload;
                                  `grid` must be > 0); for inspection/tests */

typedef struct {
  int32_t grid;            /* CTAs per launch (persistent, co-resident)      */
  int32_t threads;         /* threads per CTA                                */
  int32_t nseg;            /* non-empty segments                             */
  int32_t nlayers;
  int64_t npieces;         /* (CTA, segment) intersections                   */
  int64_t nbatches;        /* 128-element batches (one float4 per lane)      */
  int64_t elements;        /* sum of segment lengths                         */
  int32_t max_pieces_cta;
  int32_t max_slots_cta;
  int32_t smem_bytes;      /* dynamic shared memory per CTA                  */
  int32_t reserved;
  int64_t workspace_bytes; /* size of d_ws                                   */
} lars_plan_info_t;

/* Build the launch plan for a segment table: segments sorted by offset and
 * non-overlapping.  grid <= 0 picks (#SMs x resident CTAs per SM). */
LARS_API int lars_plan_create(const lars_segment_t* segs, int32_t nseg, int32_t nlayers,
                     int32_t grid, int32_t flags, void** plan);
LARS_API int lars_plan_info(const void* plan, lars_plan_info_t* info);
/* Partition of one plan, for inspection (host arrays of lars_plan_info_t
 * sizes): per global warp its first batch (grid*8+1 entries) and per piece
 * its (segment, CTA).  Any pointer may be NULL. */
LARS_API int lars_plan_partition(const void* plan, int64_t* warp_b0, int32_t* piece_seg,
                        int32_t* piece_cta);
LARS_API void lars_plan_destroy(void* plan);

/* Initialise the workspace: zero the counters and the norm carry, arm the
 * slots through which the fused step's CTAs publish their partial sums.
 * Call once after allocating d_ws (lars_plan_info_t.workspace_bytes, 256 B
 * aligned); one workspace per plan, one launch at a time. */
LARS_API int lars_workspace_init(const void* plan, void* d_ws, void* stream);

/* The whole LARS step in ONE cooperative launch: per-layer fp64 sum of
 * squares of w and g, grid barrier, trust ratio + lr on device, fused
 * WD + momentum + write-back, Sum(w_new^2) carried for the next step.
 * d_sumsq[2*l] = Sum w^2 and d_sumsq[2*l+1] = Sum g^2 over the raw buffer
 * values (before grad_scale); d_lambda[l] = lambda_l; both may be NULL. */
LARS_API int lars_step(const void* plan, float* w, const float* g, float* m,
              const lars_hparams_t* hp, int64_t* d_iter, double* d_sumsq,
              double* d_lambda, lars_step_info_t* d_info, void* d_ws,
              void* stream);

/* Split form for a sharded step.  lars_partial_norms writes this shard's
 * per-layer sums of squares to d_sumsq[2*nlayers] (zeros for layers with no
 * local elements), evaluates the lr and advances *d_iter; the caller sums
 * d_sumsq over ranks (e.g. ncclAllReduce, fp64) and then calls lars_update,
 * which reads lr/status from d_info and writes lambda for every layer. */
LARS_API int lars_partial_norms(const void* plan, const float* w, const float* g,
                       const lars_hparams_t* hp, int64_t* d_iter,
                       double* d_sumsq, lars_step_info_t* d_info, void* d_ws,
                       void* stream);
LARS_API int lars_update(const void* plan, float* w, const float* g, float* m,
                const lars_hparams_t* hp, const double* d_sumsq,
                double* d_lambda, lars_step_info_t* d_info, void* d_ws,
                void* stream);

/* Sharded step fused with its collectives over NVLink peer memory: ONE
 * cooperative launch per rank does the reduce-scatter (the rank's gradient
 * shard summed over every rank's buffer in rank order: local from HBM, peers
 * through their UVA peer pointers), the per-layer sums, their exchange
 * between ranks (peer stores into every rank's [world][nlayers][2] buffer +
 * a flag barrier), the LARS update of the shard, and the all-gather (the new
 * weights stored into every rank's weight buffer), with cross-rank barriers
 * at the start (all gradients written) and the end (all shards landed).
 * Replaces cluster.all_reduce + `/ b` + apply_update on every replica
 * (cluster.py:146-153).  Index q of each array is rank q's buffer (q == rank:
 * the local one); weight and gradient pointers are offset to THIS rank's
 * shard; `plan` is the plan of this rank's shard.  Peer buffers must be
 * mapped (e.g. torch SymmetricMemory or cudaIpc). */
#define LARS_MAX_RANKS 8
typedef struct {
  float* w_peer[LARS_MAX_RANKS];        /* weight buffers, at this shard's offset   */
  const float* g_peer[LARS_MAX_RANKS];  /* gradient buffers, at this shard's offset */
  double* x_peer[LARS_MAX_RANKS];       /* [world][nlayers][2] norm exchange        */
  unsigned* f_peer[LARS_MAX_RANKS];     /* [world] barrier flags, zero-initialised  */
  float* g_shard;                       /* local scratch (shard length)             */
  float* m;                             /* local momentum shard                     */
  int32_t rank;
  int32_t world;
} lars_peer_t;

LARS_API int lars_step_peer(const void* plan, const lars_peer_t* pr, const lars_hparams_t* hp,
                            int64_t* d_iter, double* d_sumsq, double* d_lambda,
                            lars_step_info_t* d_info, void* d_ws, void* stream);

/* A cross-rank barrier alone (one thread, the peer flags and the epoch in
 * d_ws shared with the step kernels, so every rank must call it the same
 * number of times).  For benchmarks: align the ranks between untimed work
 * and a timed step. */
LARS_API int lars_peer_barrier(const lars_peer_t* pr, void* d_ws, lars_step_info_t* d_info,
                               void* stream);

/* Same step, streamed: the reduce-scatter (NVLink inbound) and the update +
 * all-gather (outbound) run concurrently over the shard's segments -- a
 * layer held entirely by this rank is updated as soon as its own gradient
 * is reduced; layers flagged LARS_SEG_SHARED wait for the other ranks'
 * partial sums.  Same results (same reductions in the same orders: rank
 * order for the gradient, chunk order within a segment, rank order across
 * ranks).  x_peer buffers need 2 * world * (2 * nlayers + 2) doubles,
 * zero-initialised.  Replaces cluster.py:146-153 like lars_step_peer. */
LARS_API int lars_step_peer_stream(const void* plan, const lars_peer_t* pr,
                                   const lars_hparams_t* hp, int64_t* d_iter, double* d_sumsq,
                                   double* d_lambda, lars_step_info_t* d_info, void* d_ws,
                                   void* stream);

/* Host-resident parameter sets: the reference's own ParamSet holds one
 * caller-owned fp64 numpy array per group and apply_update mutates them in
 * place (nn.py:63-114, optim.py:117-134).  These move such arrays to and
 * from the flat fp32 device buffers with DMA straight from / to the caller's
 * memory (no host-side packing or conversion): each span is one contiguous
 * fp64 host array placed at `offset` elements of the flat buffer.
 *
 * lars_host_register pins caller memory for DMA (cudaHostRegister; returns
 * LARS_ERR_HOST_MEMORY if the range cannot be pinned, e.g. it shares pages
 * with an already registered range -- stage such arrays through pinned
 * memory instead).  The caller keeps the array alive while registered. */
typedef struct {
  void* host;          /* fp64 host array, pinned (registered or allocated pinned) */
  int64_t offset;      /* element offset in the flat device buffer                 */
  int64_t numel;
} lars_host_span_t;

LARS_API int lars_host_register(void* ptr, int64_t bytes);
LARS_API int lars_host_unregister(void* ptr);
/* H2D of every span into d_stage (fp64, flat_elems long, zero where no span
 * lands), then ONE conversion launch d_dst[i] = (float)d_stage[i].  Async on
 * `stream`. */
LARS_API int lars_host_copy_in(const lars_host_span_t* spans, int32_t nspans, double* d_stage,
                               float* d_dst, int64_t flat_elems, void* stream);
/* ONE conversion launch d_stage[i] = (double)d_src[i], then D2H of every span.
 * Async on `stream`: synchronize before reading the host arrays. */
LARS_API int lars_host_copy_out(const float* d_src, double* d_stage, int64_t flat_elems,
                                const lars_host_span_t* spans, int32_t nspans, void* stream);

LARS_API const char* lars_strerror(int code);
LARS_API int lars_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LARS_B200_H */
