// lars_kernels.cu -- the LARS data-parallel step on B200 (sm_100a).
//
// Replaces the reference's per-group numpy loop (pkg/src/batchlab/optim.py:
// 117-134, with lars_local_lr :98-108, group_local_lr :111-114 and
// scheduled_lr :76-95) by one persistent, cooperative kernel over the flat,
// layer-segmented fp32 buffers w / g / m:
//
//   phase A  per-layer fp64 sums of squares of g (and of w unless they were
//            carried from the previous step's epilogue); each CTA owns a
//            static range of 128-element batches (one float4 per lane) that
//            its 8 warps sweep interleaved, each through a private cp.async
//            ring in shared memory; warp butterflies and a fixed-order
//            per-CTA combine, no atomics;
//   publish  no grid barrier (cooperative launch: CTAs co-resident): each
//            CTA publishes its per-piece partials into sentinel-armed slots,
//            fills its ring for phase B (the loads do not need lambda) and
//            polls every piece straight into shared memory;
//   lambda   every CTA sums each layer's pieces in a fixed order (bitwise
//            identical lambdas in every CTA); lr from the device counter;
//   phase B  g*scale + wd*w -> m = mu*m + lambda*lr*s -> w -= m over chunks
//            handed out dynamically (per-SM HBM throughput varies ~1.7x), two
//            chunks per atomic, tapering chunk size at the end; Sum(w_new^2)
//            per chunk carried to the next step; non-finite check per chunk.
//
// Loads of g in phase A carry an L2 evict_last policy (phase B re-reads g),
// the phase-B streams evict_normal.  NORMS / UPDATE template modes give the
// split form of the sharded multi-GPU step around NCCL collectives; the PEER
// mode is the sharded step fused with its collectives over NVLink peer
// memory: phase A does the reduce-scatter, phase B the all-gather, with
// cross-rank flag barriers.
//
// Tuning knobs (LARS_POL_A/B, LARS_SUMSQ_MODE, LARS_CHUNK, LARS_CLAIM,
// LARS_ASTAGES) default to the measured best; DESIGN.md lists the A/B runs.
//
// The host side (plan construction) is at the bottom, behind the C ABI of
// include/lars_b200.h.

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <utility>
#include <vector>

#include "lars_b200.h"

namespace {

#ifndef LARS_BULK_B
#define LARS_BULK_B 0   // phase-B streams by TMA bulk copies (1) or per-lane cp.async (0)
#endif

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kBatchVec = 32;     // float4 per batch
constexpr int kMinBlocksPerSM = 2;

enum Mode { kFull = 0, kNorms = 1, kUpdate = 2, kPeer = 3, kPeerStream = 4 };

// ---------------------------------------------------------------------------
// device plan
// ---------------------------------------------------------------------------

struct DevSeg {          // one non-empty segment, in float4 units
  int64_t vec_off;
  int64_t vec_len;
  int64_t bstart;        // first global batch
  int64_t bend;          // one past the last global batch
  int32_t layer;
  int32_t flags;
};

struct DevChunk {         // phase-B work unit: <= kChunkBatches batches of one segment
  int64_t vbeg;          // first float4
  int32_t nvec;          // float4 count
  int32_t layer;
};

// Per-CTA record (phase A): the CTA's batch range, pieces and chunk range,
// followed by copies of its segments, so ONE load round at kernel start
// brings everything a CTA needs before its first data load.
struct CtaDesc {
  int64_t B0, B1;        // batch range [B0, B1)
  int32_t seg0, npc;     // first segment, pieces (segments met)
  int32_t piece0;        // global index of the first piece
  int32_t ch0, ch1;      // phase-B chunks starting in [B0, B1)
  int32_t pad[3];
};
static_assert(sizeof(CtaDesc) == 48, "CtaDesc layout");

struct DevPlan {
  const unsigned char* cta_rec;   // [grid][cta_rec_stride]: CtaDesc + DevSeg[npc]
  const DevSeg* segs;             // [nseg]
  const DevChunk* chunks;         // [nchunks]
  const int32_t* chunk_seg;       // [nchunks]     segment of each chunk
  const int32_t* warp_ch0;        // [grid*kWarps + 1] chunks starting in each warp's run
  const int32_t* cta_ch0;         // [grid + 1]    chunks starting in each CTA's range
  const int64_t* warp_b0;         // [grid*kWarps + 1]
  const int32_t* warp_seg0;       // [grid*kWarps]  segment of the first batch
  const int32_t* warp_slot0;      // [grid*kWarps]  first shared-memory slot (CTA-relative)
  const int32_t* cta_seg0;        // [grid]
  const int32_t* cta_npieces;     // [grid]
  const int32_t* cta_piece0;      // [grid]        global index of the CTA's first piece
  const int32_t* piece_slot_lo;   // [npieces]     CTA-relative slot range
  const int32_t* piece_slot_hi;   // [npieces]
  const int32_t* layer_piece_ptr; // [nlayers+1]   CSR: pieces of each layer, ascending
  const int32_t* layer_piece_idx; // [npieces]
  const int32_t* piece_pos;       // [npieces]     position of each piece in the layer CSR
  const int32_t* layer_flags;     // [nlayers]
  int32_t nseg;
  int32_t nlayers;
  int32_t npieces;
  int32_t grid;
  int32_t max_pieces_cta;
  int32_t max_slots_cta;
  int32_t nchunks;
  int32_t stage_pieces;           // npieces if partials stage outside the ring, else 0
  int32_t cta_rec_stride;         // bytes, multiple of 16
  int64_t keep_nb;                // phase-A g loads of batches < keep_nb: L2 evict_last
  int32_t pol_b;                  // phase-B streams: 0 evict_first, 1 evict_normal
  int32_t nshared;                // segments whose layer continues on other ranks
  // streamed sharded step (lars_step_peer_stream)
  const int32_t* seg_c0;          // [nseg+1]  first chunk of each segment
  const int32_t* order;           // [nchunks] chunk claim order: interior segments first
  const int32_t* layer_seg;       // [nlayers] this shard's segment of each layer, -1 if none
};

struct StepArgs {
  DevPlan p;
  float* w;
  const float* g;
  float* m;
  lars_hparams_t hp;
  int64_t* d_iter;
  double* d_sumsq;
  const double* d_sumsq_in;       // kUpdate: global sums
  double* d_lambda;
  lars_step_info_t* d_info;
  double2* partial;               // [npieces]  (sum w^2, sum g^2) per piece
  double2* pub;                   // [2][npieces] fused step: published pieces, by launch parity
  unsigned* launch_ctr;           // fused-step launches so far (parity of `pub`)
  double* ccarry;                 // [nchunks]  sum w_new^2 per chunk (next step's ||w||^2)
  double* coef_g;                 // [nlayers]  kPeer: lambda*lr of the layers shared with other ranks
  unsigned* peer_launch;          // kPeer launches so far (tags of shared_ready)
  unsigned* shared_ready;         // kPeer: tag once coef_g holds the shared layers' lambda*lr
  unsigned long long* bar;        // grid barrier counter
  unsigned long long* ctr;        // phase-B chunks claimed (low) | warps done (high)
  // kPeer: sharded step fused with its collectives over NVLink peer memory;
  // w / g above are the local weight shard and the local reduced-gradient
  // scratch.  Index q of each array = rank q's buffer (q == rank: local).
  float* w_peer[LARS_MAX_RANKS];        // weights, at this rank's shard offset
  const float* g_peer[LARS_MAX_RANKS];  // gradients, at this rank's shard offset
  double* x_peer[LARS_MAX_RANKS];       // [world][nlayers][2] norm exchange
  unsigned* f_peer[LARS_MAX_RANKS];     // [world] barrier flags
  unsigned* nv_epoch;                   // workspace: last cross-rank barrier epoch
  int32_t rank, world;
  // streamed sharded step
  double2* apart;                       // [nchunks] per-chunk (sum w^2, sum g^2)
  unsigned* seg_cnt;                    // [nseg] chunks reduced (monotonic)
  unsigned* seg_ready;                  // [nseg] launch tag once the segment's sums are final
  double2* seg_part;                    // [nseg] the segment's sums
  unsigned long long* ctr_a;            // reduce-scatter chunk claims
  unsigned long long* ctr_b;            // update / all-gather chunk claims
  unsigned* shared_done;                // shared segments reduced (monotonic)
  unsigned* stream_launch;              // launches so far (tags)
};

// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------

#ifndef LARS_POL_A
#define LARS_POL_A 0   // phase-A g loads: 0 evict_last, 1 evict_normal, 2 evict_unchanged
#endif
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
#if LARS_POL_A == 0
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#elif LARS_POL_A == 1
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
#else
  asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
#endif
  return pol;
}


__device__ __forceinline__ uint64_t policy_evict_first_rt() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_normal_rt() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void st4(float* ptr, float4 v, uint64_t pol) {
  asm volatile(
      "st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;"
      :
      : "l"(ptr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
      : "memory");
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// Cross-rank barrier (one thread): publish `epoch` in this rank's slot of
// every rank's flag array, then wait until every slot here reached it.  One
// release fence, relaxed flag stores and polls, one acquire fence (release /
// acquire on every flag access measured 16 us slower per step at P = 2).
__device__ __forceinline__ void st_relaxed_sys(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// A rank that never arrives (crashed process, mismatched step counts) must
// not hang the GPU: after kRankTimeoutNs the barrier gives up, flags
// LARS_STATUS_RANK_TIMEOUT (the host raises ProtocolError) and the launch
// runs to completion.
constexpr unsigned long long kRankTimeoutNs = 60ull * 1000000000ull;
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void rank_barrier(const StepArgs& a, unsigned epoch) {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  for (int q = 0; q < a.world; ++q) st_relaxed_sys(a.f_peer[q] + a.rank, epoch);
  const unsigned* mine = a.f_peer[a.rank];
  const unsigned long long t0 = global_ns();
  for (int q = 0; q < a.world; ++q)
    while ((int)(ld_relaxed_sys(mine + q) - epoch) < 0) {
      if (global_ns() - t0 > kRankTimeoutNs) {
        atomicOr(&a.d_info->status, LARS_STATUS_RANK_TIMEOUT);
        q = a.world;
        break;
      }
    }
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

#ifndef LARS_POLL_STAGE
#define LARS_POLL_STAGE 1
#endif
#ifndef LARS_PEER_KU4
#define LARS_PEER_KU4 2  // phase-A batches per rank in flight per warp at P >= 4
#endif
#ifndef LARS_PEER_EARLY
#define LARS_PEER_EARLY 1  // kPeer: update the shard's interior layers during the norm exchange
#endif
#ifndef LARS_SUMSQ_MODE
#define LARS_SUMSQ_MODE 0
#endif
// exact squares (fp32 x fp32 fits fp64), fp64 accumulation
__device__ __forceinline__ double sumsq4(float4 v, double acc) {
#if LARS_SUMSQ_MODE == 0
  acc = fma((double)v.x, (double)v.x, acc);
  acc = fma((double)v.y, (double)v.y, acc);
  acc = fma((double)v.z, (double)v.z, acc);
  acc = fma((double)v.w, (double)v.w, acc);
#else
  // fp32 sum of the 4 squares, one conversion, fp64 accumulation
  const float q = fmaf(v.w, v.w, fmaf(v.z, v.z, fmaf(v.y, v.y, v.x * v.x)));
  acc += (double)q;
#endif
  return acc;
}

// butterfly sum: every lane ends with the same bits (a+b == b+a)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Published values polled without fences: a slot holds an all-ones bit
// pattern (a NaN no arithmetic here produces) until written; 64-bit accesses
// are single-copy atomic, a reader waits until neither half is the sentinel.
constexpr unsigned long long kSentinel64 = ~0ull;
__device__ __forceinline__ double2 ld_relaxed2(const double2* p) {
  double2 v;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed2(double2* p, double2 v) {
  asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" :: "l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ bool is_sentinel(double x) {
  return (unsigned long long)__double_as_longlong(x) == kSentinel64;
}

__device__ __forceinline__ bool finite4(float4 v) {
  return fabsf(v.x) <= 3.402823466e38f && fabsf(v.y) <= 3.402823466e38f &&
         fabsf(v.z) <= 3.402823466e38f && fabsf(v.w) <= 3.402823466e38f;
}

// scheduled_lr (optim.py:76-95), operand order as in Python
__device__ double device_lr(const lars_hparams_t& hp, int64_t it) {
  if (hp.flags & LARS_STEP_EXPLICIT_LR) return hp.lr;
  const int64_t W = hp.warmup_iters;
  if (it < W) return __ddiv_rn(__dmul_rn(hp.base_lr, (double)(it + 1)), (double)W);
  const int64_t span = hp.max_iters - W;
  if (span <= 0) return 0.0;
  const double progress = __ddiv_rn((double)(it - W), (double)span);
  return __dmul_rn(hp.base_lr, pow(__dsub_rn(1.0, progress), hp.poly_power));
}

// lars_local_lr (optim.py:98-108) on reduced sums of squares; group_local_lr
// (:111-114) through the flags.  No FMA contraction: same roundings as Python.
__device__ double device_lambda(const lars_hparams_t& hp, int32_t flags, double w2,
                                double g2) {
  if (!hp.lars_enabled || !(flags & LARS_SEG_TRUST)) return 1.0;
  const double wn = sqrt(w2);
  const double gn = __dmul_rn(sqrt(g2), fabs(hp.grad_scale));
  const double denom = __dadd_rn(gn, __dmul_rn(hp.weight_decay, wn));
  if (wn == 0.0) return 0.0;
  if (denom == 0.0) return 1.0;
  return __ddiv_rn(__dmul_rn(hp.trust, wn), denom);
}

// After the grid barrier every CTA pulls all per-piece partials (stored in
// layer-CSR order) into shared memory -- the staging ring is idle between the
// phases -- and sums each layer's run in a fixed order, so every CTA holds
// bitwise identical per-layer sums without a second grid barrier.
__device__ __forceinline__ void stage_partials(const DevPlan& P, const double2* partial,
                                               double2* smem) {
  for (int i = threadIdx.x; i < P.npieces; i += kThreads) smem[i] = __ldcg(partial + i);
  __syncthreads();
}
__device__ __forceinline__ double2 layer_sums_smem(const int32_t* lptr, const double2* smem,
                                                   int l) {
  double aw = 0.0, ag = 0.0;
  for (int i = lptr[l]; i < lptr[l + 1]; ++i) {
    aw += smem[i].x;
    ag += smem[i].y;
  }
  return make_double2(aw, ag);
}

// Software grid barrier over a monotonic arrival counter, in two halves so
// that work can be issued between arriving and waiting.
__device__ __forceinline__ unsigned long long grid_arrive(unsigned long long* bar,
                                                          unsigned int nblocks,
                                                          bool publish = true) {
  __syncthreads();
  unsigned long long target = 0;
  if (threadIdx.x == 0) {
    // (a CTA that wrote nothing since the last barrier needs no fence; a
    // fence also waits for the thread's outstanding cp.async loads)
    if (publish) __threadfence();
    const unsigned long long old = atomicAdd(bar, 1ull);
    target = (old / nblocks + 1ull) * nblocks;
  }
  return target;
}
// Thread 0's acquire load synchronizes with every arrival's release; the CTA
// barrier then orders the other threads after it (no trailing fence, which
// would wait for the prologue's cp.async loads: measured 2 us per launch).
__device__ __forceinline__ void grid_wait(unsigned long long* bar, unsigned long long target) {
  if (threadIdx.x == 0) {
    unsigned long long cur;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(bar) : "memory");
      if (cur >= target) break;
    }
  }
  __syncthreads();
}
__device__ __forceinline__ void grid_barrier(unsigned long long* bar, unsigned int nblocks) {
  grid_wait(bar, grid_arrive(bar, nblocks));
}

// ---------------------------------------------------------------------------
// shared memory layout (dynamic):
//   float4 ring[kWarps][kStagesB*3][32]   per-warp cp.async staging ring
//   DevSeg seg_s[maxp] | float coef_s[maxp] | double2 slot_s[maxs]
// ---------------------------------------------------------------------------

// Update arithmetic: LARS_UPDATE_F64=1 evaluates optim.py:128-131 in fp64
// from the fp32 state (the reference's precision; only the stored w / m are
// rounded to fp32), 0 in fp32 with fp32 coefficients.
#ifndef LARS_UPDATE_F64
#define LARS_UPDATE_F64 1
#endif
#if LARS_UPDATE_F64
typedef double coef_t;
#else
typedef float coef_t;
#endif

constexpr int kStagesB = 8;                    // update phase: 3 arrays per stage
constexpr int kQueue = 16;                     // per-warp chunk queue (power of 2)
#ifndef LARS_CHUNK
#define LARS_CHUNK 8
#endif
#ifndef LARS_CLAIM
#define LARS_CLAIM 2
#endif
constexpr int kChunkBatches = LARS_CHUNK;      // phase-B chunk: 8 x 128 elements
constexpr int kClaim = LARS_CLAIM;             // chunks claimed per atomic
#ifndef LARS_NCTR
#define LARS_NCTR 1
#endif
constexpr int kCounters = LARS_NCTR;           // phase-B claim counters (see fetch_next)
#ifndef LARS_TAPER2
#define LARS_TAPER2 150  // last 15.0 % of the batches in 2-batch phase-B chunks (per mille)
#endif
#ifndef LARS_TAPER1
#define LARS_TAPER1 30   // last 3.0 % in 1-batch chunks
#endif
#ifndef LARS_TAPER2_LONG
#define LARS_TAPER2_LONG 100  // the same for plans with >= 150 batches per warp
#endif
#ifndef LARS_TAPER1_LONG
#define LARS_TAPER1_LONG 20
#endif
#ifndef LARS_CLAIM_AHEAD
#define LARS_CLAIM_AHEAD 1
#endif
constexpr int kClaimAhead = LARS_CLAIM_AHEAD;  // phase-B claims in flight per warp (1 or 2)
constexpr int kCtrStride = 16;                 // 128 B apart (u64 units)
static_assert(kCounters >= 1 && kCounters <= 12, "claim counters live in the workspace header");
constexpr int kRingVec = kStagesB * 3 * 32;    // float4 per warp
constexpr size_t kRingBytes = sizeof(float4) * kRingVec * kWarps;

struct QEnt {
  int64_t vbeg;   // first float4 of the chunk
  int32_t nvec;   // float4s in the chunk
  int32_t layer;
  int32_t id;
  int32_t pad;
};
static_assert(sizeof(QEnt) == 24, "QEnt layout (shared-memory budget: two CTAs per SM)");
// the streamed step's queue entry carries lambda*lr too: 12 of them fill the
// same per-warp queue area as 16 QEnt
struct QEntS {
  int64_t vbeg;
  int32_t nvec;
  int32_t layer;
  int32_t id;
  int32_t pad;
  double coef;
};
constexpr int kQueueS = 12;
static_assert(sizeof(QEntS) * kQueueS <= sizeof(QEnt) * 16, "stream queue fits the QEnt area");

__host__ __device__ __forceinline__ size_t align_up(size_t x, size_t a) { return (x + a - 1) & ~(a - 1); }

constexpr size_t kMaxStageBytes = 16 * 1024;   // separate partial staging (else: in the ring)

struct SmemOff {
  size_t queue, mbar, seg, slot, stage, lptr, lflags, coef, total;
};

// ring | queues | segments | slots | staged partials | layer CSR | flags | coefficients
__host__ __device__ __forceinline__ SmemOff smem_layout(int maxp, int maxs, int nlayers,
                                                        int stage_pieces) {
  SmemOff o;
  size_t off = kRingBytes;
  o.queue = off;
  off += sizeof(QEnt) * kQueue * kWarps;
  o.mbar = off;
  off += LARS_BULK_B ? sizeof(uint64_t) * kStagesB * kWarps : 0;
  o.seg = off + sizeof(CtaDesc);  // the CTA record lands at o.seg - 48
  off += sizeof(CtaDesc) + sizeof(DevSeg) * (size_t)maxp;
  off = align_up(off, 16);
  o.slot = off;
  off += sizeof(double2) * (size_t)maxs;
  o.stage = off;
  off += sizeof(double2) * (size_t)stage_pieces;
  o.lptr = off;
  off += sizeof(int32_t) * (size_t)(nlayers + 1);
  o.lflags = off;
  off += sizeof(int32_t) * (size_t)nlayers;
  off = align_up(off, 8);
  o.coef = off;
  off += sizeof(coef_t) * (size_t)nlayers;
  o.total = align_up(off, 16);
  return o;
}

struct Smem {
  uint64_t* mbar;  // this warp's phase-B stage barriers (bulk-copy build)
  CtaDesc* rec;    // this CTA's record (phase A), followed by its segments
  float4* ring;    // this warp's ring
  QEnt* queue;     // this warp's chunk queue
  DevSeg* seg;     // the CTA's segments (phase A)
  double2* slot;   // per-(warp, segment) partial sums (phase A)
  double2* stage;  // all per-piece partials after the barrier (may alias the ring)
  int32_t* lptr;   // layer -> piece range (CSR)
  int32_t* lflags; // layer flags
  coef_t* coef;    // lambda*lr per layer (phase B)
};

__device__ __forceinline__ Smem carve(const DevPlan& P, int warp) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const SmemOff o = smem_layout(P.max_pieces_cta, P.max_slots_cta, P.nlayers, P.stage_pieces);
  Smem s;
  s.ring = reinterpret_cast<float4*>(smem_raw) + (size_t)warp * kRingVec;
  s.queue = reinterpret_cast<QEnt*>(smem_raw + o.queue) + (size_t)warp * kQueue;
  s.mbar = reinterpret_cast<uint64_t*>(smem_raw + o.mbar) + (size_t)warp * kStagesB;
  s.seg = reinterpret_cast<DevSeg*>(smem_raw + o.seg);
  s.rec = reinterpret_cast<CtaDesc*>(smem_raw + o.seg - sizeof(CtaDesc));
  s.slot = reinterpret_cast<double2*>(smem_raw + o.slot);
  s.stage = P.stage_pieces ? reinterpret_cast<double2*>(smem_raw + o.stage)
                           : reinterpret_cast<double2*>(smem_raw);
  s.lptr = reinterpret_cast<int32_t*>(smem_raw + o.lptr);
  s.lflags = reinterpret_cast<int32_t*>(smem_raw + o.lflags);
  s.coef = reinterpret_cast<coef_t*>(smem_raw + o.coef);
  return s;
}

// 16-byte cp.async (LDGSTS, L1 bypass) with an L2 eviction policy; lanes past
// the end of a segment copy 0 source bytes, i.e. zero-fill their slot.
__device__ __forceinline__ void cp_async16(float4* dst, const float* src, bool ok, uint64_t pol) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;"
               :: "r"(d), "l"(src), "r"(ok ? 16 : 0), "l"(pol) : "memory");
}
// 8- and 4-byte variants (L1-allocating .ca is the only form for < 16 B)
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" :: "r"(d), "l"(src), "r"(ok ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" :: "r"(d), "l"(src), "r"(ok ? 4 : 0)
               : "memory");
}
// 1D TMA bulk copies (cp.async.bulk, async proxy) completing on an mbarrier
#if LARS_BULK_B
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT_%=;\n}" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
#endif
__device__ __forceinline__ void cp_async16_cg(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" :: "l"(p));
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory");
}

// A segment's fields cached in registers while a warp walks its batch run
// (forward or backward); reloaded from shared memory only on a segment change.
struct SegReg {
  int64_t bstart, bend, voff, vlen;
  int c;
  __device__ __forceinline__ void load(const DevSeg* seg, int ci) {
    c = ci;
    bstart = seg[ci].bstart;
    bend = seg[ci].bend;
    voff = seg[ci].vec_off;
    vlen = seg[ci].vec_len;
  }
};

// ---------------------------------------------------------------------------
// phase A: per-(warp, segment) sums of squares into shared slots.
// Each lane stages its own float4s through the warp's ring with cp.async
// (no cross-lane sharing, so no barriers); kStages batches in flight, two
// consumed per iteration.
// ---------------------------------------------------------------------------

// The CTA's batch range [B0, B1) is read as ONE stream: warp w takes
// batches B0 + w, B0 + w + kWarps, ... (the 8 warps of a CTA sweep it side by
// side, 296 streams instead of 2368 scattered per-warp runs, which keeps
// DRAM pages open).  Warp w's sums for CTA piece c go to slot[w][c].
template <bool kReadW>
__device__ __forceinline__ void phase_norms(const StepArgs& a, const Smem& S, int64_t B0,
                                            int64_t B1, int warp, int lane) {
  const int64_t b0 = B0 + warp;
  if (b0 >= B1) return;
  constexpr int kArr = kReadW ? 2 : 1;
#ifndef LARS_ASTAGES
#define LARS_ASTAGES 16  // phase-A ring stages x arrays (measured: 12-16 best on AlexNet-BN)
#endif
  constexpr int kStages = LARS_ASTAGES / kArr;
  static_assert(kStages % 2 == 0, "stages must be even");
  const uint64_t keep = policy_evict_last();
  const uint64_t pass = policy_evict_first_rt();
  const int64_t keep_nb = a.p.keep_nb;
  const float* __restrict__ g = a.g;
  const float* __restrict__ w = a.w;
  float4* ring = S.ring;
  double2* slots = S.slot + (size_t)warp * a.p.max_pieces_cta;
  int c0 = 0;
  while (b0 >= S.seg[c0].bend) ++c0;
  int64_t ib = b0;
  SegReg is;
  is.load(S.seg, c0);
  auto issue = [&](int st) {
    if (ib < B1) {
      if (ib >= is.bend) {
        int ci = is.c;
        do { ++ci; } while (ib >= S.seg[ci].bend);
        is.load(S.seg, ci);
      }
      const int64_t rel = (ib - is.bstart) * kBatchVec + lane;
      const bool ok = rel < is.vlen;
      const int64_t e = ok ? (is.voff + rel) * 4 : 0;
      // g is re-read by phase B: keep the window L2 can hold (the start of
      // the buffer, which phase B visits first), stream the rest
      const uint64_t pol = ib < keep_nb ? keep : pass;
      cp_async16(ring + (st * kArr) * 32 + lane, g + e, ok, pol);
      if (kReadW) cp_async16(ring + (st * kArr + 1) * 32 + lane, w + e, ok, pol);
      ib += kWarps;
    }
    cp_async_commit();
  };
#pragma unroll 1
  for (int st = 0; st < kStages; ++st) issue(st);
  double aw = 0.0, ag = 0.0;
  SegReg cs;
  cs.load(S.seg, c0);
  auto consume = [&](int64_t b, int st) {
    if (b >= cs.bend) {
      aw = warp_sum(aw);
      ag = warp_sum(ag);
      if (lane == 0) slots[cs.c] = make_double2(aw, ag);
      aw = 0.0;
      ag = 0.0;
      int ci = cs.c;
      do { ++ci; } while (b >= S.seg[ci].bend);
      cs.load(S.seg, ci);
    }
    const float4 gv = ring[(st * kArr) * 32 + lane];  // zero-filled past the end
    ag = sumsq4(gv, ag);
    if (kReadW) {
      const float4 wv = ring[(st * kArr + 1) * 32 + lane];
      aw = sumsq4(wv, aw);
    }
  };
  int st = 0;
#pragma unroll 1
  for (int64_t b = b0; b < B1; b += 2 * kWarps) {
    cp_async_wait<kStages - 2>();
    consume(b, st);
    if (b + kWarps < B1) consume(b + kWarps, st + 1);
    issue(st);
    issue(st + 1);
    st = (st + 2 == kStages) ? 0 : st + 2;
  }
  cp_async_wait<0>();
  aw = warp_sum(aw);
  ag = warp_sum(ag);
  if (lane == 0) slots[cs.c] = make_double2(aw, ag);
}

// kU batches per peer in flight per warp.  Every warp of the grid pulls at
// once, so the links are heavily oversubscribed; fewer bytes in flight per
// warp give fairer service and a shorter straggler tail (measured: P=4 kU 8
// -> 4 -> 2: 313 -> 295 -> 292 us; P=2 best at 4).
template <bool kReadW, int kU>
__device__ __forceinline__ void phase_norms_peer(const StepArgs& a, const Smem& S, int64_t B0,
                                                 int64_t B1, int warp, int lane) {
  const int64_t b0 = B0 + warp;
  if (b0 >= B1) return;
  const uint64_t keep = policy_evict_last();
  double2* slots = S.slot + (size_t)warp * a.p.max_pieces_cta;
  double aw = 0.0, ag = 0.0;
  int cur = 0;
  while (b0 >= S.seg[cur].bend) ++cur;
#pragma unroll 1
  for (int64_t b = b0; b < B1; b += kU * kWarps) {
    float4 acc[kU];
    int64_t ev[kU];
    int cu[kU];
    int cc = cur;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t bb = b + (int64_t)u * kWarps;
      cu[u] = -1;
      ev[u] = -1;
      acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (bb < B1) {
        while (bb >= S.seg[cc].bend) ++cc;
        cu[u] = cc;
        const int64_t rel = (bb - S.seg[cc].bstart) * kBatchVec + lane;
        if (rel < S.seg[cc].vec_len) ev[u] = (S.seg[cc].vec_off + rel) * 4;
      }
    }
    // sum over ranks in rank order (fixed, deterministic)
#pragma unroll 1
    for (int q = 0; q < a.world; ++q) {
      const float* gq = a.g_peer[q];
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        v[u] = ev[u] >= 0 ? __ldcg(reinterpret_cast<const float4*>(gq + ev[u]))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        acc[u].x += v[u].x;
        acc[u].y += v[u].y;
        acc[u].z += v[u].z;
        acc[u].w += v[u].w;
      }
    }
    float4 wv[kU];
    if (kReadW) {
#pragma unroll
      for (int u = 0; u < kU; ++u)
        wv[u] = ev[u] >= 0 ? *reinterpret_cast<const float4*>(a.w + ev[u])
                           : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (cu[u] >= 0) {
        if (cu[u] != cur) {
          aw = warp_sum(aw);
          ag = warp_sum(ag);
          if (lane == 0) slots[cur] = make_double2(aw, ag);
          aw = 0.0;
          ag = 0.0;
          cur = cu[u];
        }
        if (ev[u] >= 0) st4(const_cast<float*>(a.g) + ev[u], acc[u], keep);
        ag = sumsq4(acc[u], ag);
        if (kReadW) aw = sumsq4(wv[u], aw);
      }
    }
  }
  aw = warp_sum(aw);
  ag = warp_sum(ag);
  if (lane == 0) slots[cur] = make_double2(aw, ag);
}

// ---------------------------------------------------------------------------
// phase B: fused update over dynamically scheduled chunks.
//
// Per-SM HBM throughput differs by up to ~1.7x on B200 (measured with
// tools/trace_step.py), so a static split leaves the fast SMs idle.  Phase B
// therefore hands out chunks (<= kChunkBatches batches inside one segment)
// from a global counter.  Each chunk's Sum(w_new^2) is reduced in a fixed
// order inside the chunk and stored per chunk, so the result does not depend
// on which warp processed it (bitwise deterministic).  The issue side of the
// cp.async pipeline grabs the next chunk id one chunk ahead (atomic latency
// hidden) and passes chunk descriptors to the consume side through a small
// per-warp queue in shared memory.
// ---------------------------------------------------------------------------

template <bool kEarly>  // kPeer with the interior-first order (LARS_PEER_EARLY)
struct UpdatePipe {
  static constexpr int kStages = kStagesB;
  static_assert(kStages % 2 == 0 && kQueue >= kStages + 2, "pipeline sizes");
  const StepArgs& a;
  const Smem& S;
  const int lane;
  const int nchunks;
  const int nwarps;
  uint64_t pol;
  // issue side: chunk ids come from an atomic issued one chunk ahead, and the
  // descriptor of the next chunk is loaded one chunk ahead, so switching
  // chunks never waits on memory
  int pending = 0;  // lane 0: first id of the block claimed by the prefetching atomic
  int pending2 = 0; // lane 0 (kClaimAhead == 2): the block claimed after that one
  int blk_next = 0, blk_end = 0;  // rest of the current claimed block
  bool issuing = true;
  bool have_nx = false;
  DevChunk nx{0, 0, 0};
  int nx_id = 0;
  QEnt ic{0, 0, 0, 0, 0};
  int ij = 0, inb = 0;  // batch within the issue chunk / its batch count
  int tail = 0;         // queue entries written
  int64_t issued = 0;
  // consume side
  QEnt cc{0, 0, 0, -1, 0};
  int cj = 0, cnb = 0, head = 0;
  int64_t consumed = 0;
  double aw = 0.0;
  bool bad = false;
  bool started = false;
  unsigned phase = 0;  // bulk-copy build: parity of each stage's barrier
  int cid = 0;  // claim counter in use
  int dry = 0;  // counters found exhausted
  unsigned peer_tag = 0;  // kPeer with early interior update: this launch's tag
  bool shared_ok = false; // the shared layers' lambda*lr arrived

  __device__ UpdatePipe(const StepArgs& a_, const Smem& S_, int lane_)
      : a(a_), S(S_), lane(lane_), nchunks(a_.p.nchunks), nwarps(gridDim.x * kWarps) {
    cid = (int)((blockIdx.x * kWarps + (threadIdx.x >> 5)) % kCounters);
    pol = a.p.pol_b ? policy_evict_normal_rt() : policy_evict_first_rt();
  }

  // Chunks are claimed kClaim at a time (the first one per warp is static).
  // With kCounters > 1 the claim blocks are dealt round-robin to that many
  // counters on separate L2 lines (block j + kCounters*c of counter j), a
  // warp starting on counter gw % kCounters and moving on when it runs
  // dry: the tapered tail's many small claims no longer queue on one atomic
  // unit.  Block ids map back to chunk ids as nwarps + kClaim * block.
  __device__ __forceinline__ int claim(int cid) {
    const unsigned c = (unsigned)atomicAdd(a.ctr + kCtrStride * cid, 1ull);
    return nwarps + kClaim * (cid + kCounters * (int)c);
  }
  __device__ __forceinline__ void fetch_next() {
    if (blk_next == blk_end) {
      int base = __shfl_sync(0xffffffffu, pending, 0);
      while (base >= nchunks) {  // this counter ran dry: try the next one
        if (++dry == kCounters) {
          have_nx = false;
          return;
        }
        cid = cid + 1 == kCounters ? 0 : cid + 1;
        if (lane == 0) {
          pending = claim(cid);
          if (kClaimAhead == 2) pending2 = claim(cid);
        }
        base = __shfl_sync(0xffffffffu, pending, 0);
      }
      blk_next = base;
      blk_end = min(base + (base < nwarps ? 1 : kClaim), nchunks);
      if (lane == 0) {
        if (kClaimAhead == 2) {  // two claims in flight: the next block's id is
          pending = pending2;    // already back when the current one is used up
          pending2 = claim(cid);
        } else {
          pending = claim(cid);
        }
      }
    }
    nx_id = kEarly ? a.p.order[blk_next++] : blk_next++;  // kPeer early: interior first
    have_nx = true;
    nx = a.p.chunks[nx_id];
  }

  // kPeer early: the shared layers' lambda*lr, once CTA 0 of this rank has
  // exchanged the sums with the other ranks
  __device__ void wait_shared() {
    const unsigned long long t0 = global_ns();
    unsigned backoff = 32;
    while (ld_acquire_u32(a.shared_ready) != peer_tag) {
      if (global_ns() - t0 > kRankTimeoutNs) {
        if (lane == 0) atomicOr(&a.d_info->status, LARS_STATUS_RANK_TIMEOUT);
        break;
      }
      __nanosleep(backoff);
      backoff = min(backoff * 2, 1024u);
    }
    shared_ok = true;
  }

  __device__ __forceinline__ void take_chunk() {
    if (!have_nx) {
      issuing = false;
      return;
    }
    ic.vbeg = nx.vbeg;
    ic.nvec = nx.nvec;
    ic.layer = nx.layer;
    ic.id = nx_id;
    ij = 0;
    inb = (nx.nvec + kBatchVec - 1) / kBatchVec;
    if (lane == 0) S.queue[tail & (kQueue - 1)] = ic;
    ++tail;
    __syncwarp();
    fetch_next();
  }

  __device__ __forceinline__ void issue(int st) {
    if (issuing && ij == inb) take_chunk();
    if (issuing) {
#if LARS_BULK_B
      // one elected lane moves the stage: three bulk copies (<= 512 B each,
      // the batch's valid part) completing on the stage's mbarrier
      if (lane == 0) {
        const int nv = min(kBatchVec, ic.nvec - ij * kBatchVec);
        const unsigned bytes = 16u * (unsigned)nv;
        const int64_t e = (ic.vbeg + (int64_t)ij * kBatchVec) * 4;
        float4* ring = S.ring;
        fence_proxy_async();  // the stage's previous generic reads before the async writes
        mbar_expect_tx(S.mbar + st, 3u * bytes);
        bulk_g2s(ring + (st * 3 + 0) * 32, a.g + e, bytes, S.mbar + st, pol);
        bulk_g2s(ring + (st * 3 + 1) * 32, a.w + e, bytes, S.mbar + st, pol);
        bulk_g2s(ring + (st * 3 + 2) * 32, a.m + e, bytes, S.mbar + st, pol);
      }
#else
      const int rel = ij * kBatchVec + lane;
      const bool ok = rel < ic.nvec;
      const int64_t e = ok ? (ic.vbeg + rel) * 4 : 0;
      float4* ring = S.ring;
      cp_async16(ring + (st * 3 + 0) * 32 + lane, a.g + e, ok, pol);
      cp_async16(ring + (st * 3 + 1) * 32 + lane, a.w + e, ok, pol);
      cp_async16(ring + (st * 3 + 2) * 32 + lane, a.m + e, ok, pol);
#endif
      ++ij;
      ++issued;
    }
#if !LARS_BULK_B
    cp_async_commit();
#endif
  }

  // grab the first chunks and fill the ring (does not need the trust ratios)
  // the first chunk of every warp is static (chunk id = global warp id), so
  // the prologue needs no atomic; later ids are nwarps + counter
  __device__ __forceinline__ void prologue() {
    started = true;
    pending = blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (kClaimAhead == 2 && lane == 0) pending2 = claim(cid);
    fetch_next();
#pragma unroll 1
    for (int st = 0; st < kStages; ++st) issue(st);
  }

  __device__ __forceinline__ void finish_chunk() {
    aw = warp_sum(aw);
    if (lane == 0) a.ccarry[cc.id] = aw;
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(&a.d_info->nonfinite_layer, cc.layer);
    aw = 0.0;
    bad = false;
  }

  __device__ __forceinline__ void consume(int st, coef_t& k, coef_t mu, coef_t wd, coef_t gsc) {
    if (cj == cnb) {
      if (cc.id >= 0) finish_chunk();
      cc = S.queue[head & (kQueue - 1)];
      ++head;
      cj = 0;
      cnb = (cc.nvec + kBatchVec - 1) / kBatchVec;
      k = S.coef[cc.layer];
      if (kEarly && (S.lflags[cc.layer] & LARS_SEG_SHARED)) {
        if (!shared_ok) wait_shared();
        k = (coef_t)__ldcg(a.coef_g + cc.layer);
      }
    }
#if LARS_BULK_B
    mbar_wait(S.mbar + st, (phase >> st) & 1u);
    phase ^= 1u << st;
#endif
    const int rel = cj * kBatchVec + lane;
    if (rel < cc.nvec) {
      const float4* ring = S.ring;
      const float4 gv = ring[(st * 3 + 0) * 32 + lane];
      const float4 wv = ring[(st * 3 + 1) * 32 + lane];
      const float4 mv = ring[(st * 3 + 2) * 32 + lane];
      float4 mn, wn;
      // optim.py:128-131: step_g = g + wd*w; m = mu*m + (lam*lr)*step_g; w -= m
#if LARS_UPDATE_F64
      // step_g and the new m in fp64 like the reference (mu*m and
      // lam*lr*step_g can cancel to a tiny m); only the stored m is rounded.
      // w - m in fp32 from the stored m: rounding error <= eps(|w'| + |m'|).
      auto upd = [&](float g, float w, float m, float& mo, float& wo) {
        const double sg = fma(wd, (double)w, (double)g * gsc);
        const double m64 = fma(mu, (double)m, k * sg);
        mo = (float)m64;
#if LARS_UPDATE_F64 == 2
        wo = (float)((double)w - m64);
#else
        wo = w - mo;
#endif
      };
      upd(gv.x, wv.x, mv.x, mn.x, wn.x);
      upd(gv.y, wv.y, mv.y, mn.y, wn.y);
      upd(gv.z, wv.z, mv.z, mn.z, wn.z);
      upd(gv.w, wv.w, mv.w, mn.w, wn.w);
#else
      float4 sg;
      sg.x = fmaf(wd, wv.x, gv.x * gsc);
      sg.y = fmaf(wd, wv.y, gv.y * gsc);
      sg.z = fmaf(wd, wv.z, gv.z * gsc);
      sg.w = fmaf(wd, wv.w, gv.w * gsc);
      mn.x = fmaf(mu, mv.x, k * sg.x);
      mn.y = fmaf(mu, mv.y, k * sg.y);
      mn.z = fmaf(mu, mv.z, k * sg.z);
      mn.w = fmaf(mu, mv.w, k * sg.w);
      wn.x = wv.x - mn.x;
      wn.y = wv.y - mn.y;
      wn.z = wv.z - mn.z;
      wn.w = wv.w - mn.w;
#endif
      const int64_t e = (cc.vbeg + rel) * 4;
      st4(a.m + e, mn, pol);
      if (a.world > 1) {
        // all-gather: the new weights go to every rank (peers over NVLink)
        for (int q = 0; q < a.world; ++q) st4(a.w_peer[q] + e, wn, pol);
      } else {
        st4(a.w + e, wn, pol);
      }
      aw = sumsq4(wn, aw);
      bad |= !finite4(wn);
    }
    ++cj;
    ++consumed;
  }

  // drain the pipeline: consume two batches, refill two stages, repeat
  __device__ __forceinline__ void run() {
    if (!started) prologue();
    const coef_t mu = (coef_t)a.hp.momentum;
    const coef_t wd = (coef_t)a.hp.weight_decay;
    const coef_t gsc = (coef_t)a.hp.grad_scale;
    coef_t k = 0;
    int st = 0;
#pragma unroll 1
    while (consumed < issued) {
#if !LARS_BULK_B
      cp_async_wait<kStages - 2>();
#endif
      consume(st, k, mu, wd, gsc);
      if (consumed < issued) consume(st + 1, k, mu, wd, gsc);
      issue(st);
      issue(st + 1);
      st = (st + 2 == kStages) ? 0 : st + 2;
    }
#if !LARS_BULK_B
    cp_async_wait<0>();
#endif
    if (cc.id >= 0) finish_chunk();
    // the last warp out resets the chunk counter for the next launch.
    // Claims (low half) and departures (high half) share one 64-bit word:
    // same-address atomics are ordered, so no fence is needed (a fence here
    // would wait for this warp's last stores)
    if (lane == 0) {
      const unsigned long long old = atomicAdd(a.ctr, 1ull << 32);
      if ((old >> 32) == gridDim.x * kWarps - 1)
        for (int j = 0; j < kCounters; ++j) atomicExch(a.ctr + kCtrStride * j, 0ull);
    }
  }
};

// ---------------------------------------------------------------------------
// optional per-warp phase timestamps (profiling builds: -DLARS_TRACE)
// ---------------------------------------------------------------------------

#ifdef LARS_TRACE
constexpr int kTraceWarps = 8192;
__device__ unsigned long long g_trace[kTraceWarps * 8];
__device__ __forceinline__ void trace(int gw, int k, int lane) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (lane == 0 && gw < kTraceWarps) g_trace[gw * 8 + k] = t;
  if (k == 0 && lane == 0 && gw < kTraceWarps) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_trace[gw * 8 + 7] = smid;
  }
}
__device__ __forceinline__ void trace_val(int gw, int k, unsigned long long v, int lane) {
  if (lane == 0 && gw < kTraceWarps) g_trace[gw * 8 + k] = v;
}
#else
__device__ __forceinline__ void trace(int, int, int) {}
__device__ __forceinline__ void trace_val(int, int, unsigned long long, int) {}
#endif

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------

template <int kMode, bool kCarry>
__global__ void __launch_bounds__(kThreads, kMinBlocksPerSM) lars_step_kernel(StepArgs a) {
  const DevPlan& P = a.p;
  const int warp = threadIdx.x >> 5;
  const Smem S = carve(P, warp);
  const int cta = blockIdx.x;
  const int lane = threadIdx.x & 31;
  const int gw = cta * kWarps + warp;
  trace(gw, 0, lane);
#if LARS_BULK_B
  if (lane == 0)
    for (int i = 0; i < kStagesB; ++i) mbar_init(S.mbar + i, 1);
  __syncwarp();
#endif

  // ---- one load round before any wait: the CTA record (phase-A range,
  // pieces, chunk range, segment copies), the per-layer tables (needed after
  // the barrier), the schedule state, and an L2 prefetch of this warp's first
  // phase-B chunk descriptor (static id = global warp id) ----
  if (kMode != kUpdate) {
    const float4* rsrc = reinterpret_cast<const float4*>(P.cta_rec + (size_t)cta * P.cta_rec_stride);
    float4* rdst = reinterpret_cast<float4*>(S.rec);
    for (int i = threadIdx.x; i < P.cta_rec_stride / 16; i += kThreads) cp_async16_cg(rdst + i, rsrc + i);
  }
  for (int l = threadIdx.x; l <= P.nlayers; l += kThreads) {
    cp_async4(S.lptr + l, P.layer_piece_ptr + l, true);
    if (l < P.nlayers) cp_async4(S.lflags + l, P.layer_flags + l, true);
  }
  cp_async_commit();
  if (kMode != kNorms && lane == 0 && gw < P.nchunks) prefetch_l2(P.chunks + gw);

  // lr / schedule state (optim.py:83-95) -- every CTA evaluates it identically
  int64_t it;
  double lr;
  bool exhausted;
  if (kMode == kUpdate) {
    lr = a.d_info->lr;
    it = a.d_info->iteration;
    exhausted = (a.d_info->status & LARS_STATUS_EXHAUSTED) != 0;
  } else {
    it = *a.d_iter;
    exhausted = !(a.hp.flags & LARS_STEP_EXPLICIT_LR) && it > a.hp.max_iters;
    lr = exhausted ? 0.0 : device_lr(a.hp, it);
    if (cta == 0 && threadIdx.x == 0) {
      a.d_info->lr = lr;
      a.d_info->iteration = it;
      a.d_info->nonfinite_layer = INT_MAX;
      a.d_info->status = exhausted ? LARS_STATUS_EXHAUSTED : 0;
      // order the reset before this CTA's publishes (after which other CTAs
      // may atomicMin a non-finite layer into it)
      __threadfence();
    }
  }
  UpdatePipe<kMode == kPeer && LARS_PEER_EARLY> up(a, S, lane);
  // fused step: this launch's published-piece array and the next one's
  double2* pub = nullptr;
  double2* pub_next = nullptr;
  if (kMode == kFull && LARS_POLL_STAGE) {
    const unsigned par = *reinterpret_cast<volatile unsigned*>(a.launch_ctr) & 1u;
    pub = a.pub + (size_t)par * P.npieces;
    pub_next = a.pub + (size_t)(par ^ 1u) * P.npieces;
  }

  unsigned peer_tag = 0;
  if (kMode == kPeer && LARS_PEER_EARLY) {
    peer_tag = *reinterpret_cast<volatile unsigned*>(a.peer_launch) + 1u;
    up.peer_tag = peer_tag;
  }
  if (kMode == kPeer) {
    // every rank's gradient must be complete before anyone reads it through
    // the switch (the previous launch's final barrier covers the other way)
    if (cta == 0 && threadIdx.x == 0) {
      const unsigned e0 = *a.nv_epoch + 1;
      rank_barrier(a, e0);
      *a.nv_epoch = e0;
    }
    grid_barrier(a.bar, gridDim.x);
    if (gw != 0) trace(gw, 5, lane);  // (slot 5 of warp 0: exchange below)
  }

  if (kMode != kUpdate) {
    // ---- phase A: static per-warp runs, per-layer sums of squares ----
    cp_async_wait<0>();  // the record and layer tables (issued at entry)
    __syncthreads();
    const int seg0 = S.rec->seg0;
    const int npc = S.rec->npc;
    const int piece0 = S.rec->piece0;
    const int64_t B0 = S.rec->B0;
    const int64_t B1 = S.rec->B1;
    const int maxp = P.max_pieces_cta;
    for (int i = threadIdx.x; i < kWarps * maxp; i += kThreads) S.slot[i] = make_double2(0.0, 0.0);
    // ||w||^2 carried from the previous update: the per-chunk sums of the
    // chunks that start in this CTA's range, warp w taking every 8th; their
    // lines are pulled into L2 now so the fold after phase A hits L2
    const int ch0 = S.rec->ch0, ch1 = S.rec->ch1;
    if (kCarry) {
      for (int i = ch0 + 16 * threadIdx.x; i < ch1; i += 16 * kThreads) prefetch_l2(a.ccarry + i);
      for (int i = ch0 + 32 * threadIdx.x; i < ch1; i += 32 * kThreads) prefetch_l2(P.chunk_seg + i);
    }
    __syncthreads();
    if (kMode == kPeer) {
      if (a.world >= 4)
        phase_norms_peer<!kCarry, LARS_PEER_KU4>(a, S, B0, B1, warp, lane);
      else
        phase_norms_peer<!kCarry, 4>(a, S, B0, B1, warp, lane);
    } else {
      phase_norms<!kCarry>(a, S, B0, B1, warp, lane);
    }
    if (kCarry) {
      // The warp's chunks (every 8th of the CTA's) 256 at a time: their
      // carries and segment ids land in the (now idle) ring by cp.async, all
      // in flight at once -- a CTA owning the tapered 1-batch chunks has
      // hundreds, and one dependent load round per 32 made it a phase-A
      // straggler.  Then 32 at a time (lane i: the i-th chunk, in chunk
      // order) a segmented warp scan sums each segment's run, whose last lane
      // adds it to the segment's slot: a fixed order, so deterministic.
      __syncwarp();
      double2* slots = S.slot + (size_t)warp * maxp;
      double* cbuf = reinterpret_cast<double*>(S.ring);
      int32_t* sbuf = reinterpret_cast<int32_t*>(cbuf + 256);
      for (int blk = ch0 + warp; blk < ch1; blk += 256 * kWarps) {
        for (int j = lane; j < 256; j += 32) {
          const int ch = blk + kWarps * j;
          const bool ok = ch < ch1;
          cp_async8(cbuf + j, a.ccarry + (ok ? ch : 0), ok);
          cp_async4(sbuf + j, P.chunk_seg + (ok ? ch : 0), ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        for (int g = 0; g < 8 && blk + kWarps * 32 * g < ch1; ++g) {
          const int j = 32 * g + lane;
          const bool valid = blk + kWarps * j < ch1;
          const double v0 = cbuf[j];
          const int sg = valid ? sbuf[j] : -1;
          double v = valid ? v0 : 0.0;
          const int sg_prev = __shfl_up_sync(0xffffffffu, sg, 1);
          unsigned f = (lane == 0 || sg_prev != sg) ? 1u : 0u;  // run head
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const double vu = __shfl_up_sync(0xffffffffu, v, d);
            const unsigned fu = __shfl_up_sync(0xffffffffu, f, d);
            if (lane >= d) {
              if (!f) v = vu + v;
              f |= fu;
            }
          }
          const int sg_next = __shfl_down_sync(0xffffffffu, sg, 1);
          if (valid && (lane == 31 || sg_next != sg)) slots[sg - seg0].x += v;
          __syncwarp();
        }
      }
    }
    trace(gw, 1, lane);
    __syncthreads();
    for (int c = threadIdx.x; c < npc; c += kThreads) {
      double aw = 0.0, ag = 0.0;
      for (int w8 = 0; w8 < kWarps; ++w8) {
        aw += S.slot[w8 * maxp + c].x;
        ag += S.slot[w8 * maxp + c].y;
      }
      const int pos = P.piece_pos[piece0 + c];
      if (kMode == kFull && LARS_POLL_STAGE) {
        // published for the other CTAs' staging polls; this CTA's slots of
        // the next launch's array are armed now (nobody reads them before)
        st_relaxed2(pub + pos, make_double2(aw, ag));
        st_relaxed2(pub_next + pos, make_double2(__longlong_as_double((long long)kSentinel64),
                                                 __longlong_as_double((long long)kSentinel64)));
      } else {
        a.partial[pos] = make_double2(aw, ag);
      }
    }
    // Phase B's first loads do not depend on the trust ratios: issue them
    // between arriving at the barrier and waiting (after arriving: the
    // arrival's fence would wait for them).  Needs the ring free, i.e. the
    // partials staged elsewhere.  kPeer: phase B reads the reduced gradient
    // other CTAs wrote in phase A, so only after the wait, and not in CTA 0,
    // whose exchange loads and peer stores would queue behind them (measured
    // 4 us at P = 2).
    if (kMode == kFull && LARS_POLL_STAGE) {
      // No grid barrier: every CTA polls the published pieces straight into
      // its staging buffer (a piece is final once it is not the sentinel),
      // so the last publish is followed by one L2 round trip, not a barrier
      // plus a staging load.  All pieces published = every CTA finished
      // phase A (its reads of w and of the carry included) and read its
      // launch-start state.
      if (!exhausted && P.stage_pieces) up.prologue();
      for (int i = threadIdx.x; i < P.npieces; i += kThreads) {
        double2 v;
        while (v = ld_relaxed2(pub + i), is_sentinel(v.x) || is_sentinel(v.y)) {
        }
        S.stage[i] = v;
      }
      __syncthreads();
      trace(gw, 2, lane);
      if (cta == 0 && threadIdx.x == 0) {
        atomicAdd(a.launch_ctr, 1u);
        if (!exhausted && (a.hp.flags & LARS_STEP_ADVANCE_ITER)) *a.d_iter = it + 1;
      }
    } else {
      const unsigned long long bt = grid_arrive(a.bar, gridDim.x);
      if (kMode == kFull && !exhausted && P.stage_pieces) up.prologue();
      grid_wait(a.bar, bt);
      if (kMode == kPeer && cta != 0 && !exhausted && P.stage_pieces) up.prologue();
      trace(gw, 2, lane);
      if (cta == 0 && threadIdx.x == 0 && !exhausted && (a.hp.flags & LARS_STEP_ADVANCE_ITER))
        *a.d_iter = it + 1;
    }
  }

  if (kMode == kNorms) {
    // per-layer local sums for the cross-rank all-reduce (CTA 0 writes them)
    if (cta != 0) return;
    stage_partials(P, a.partial, S.stage);
    for (int l = threadIdx.x; l < P.nlayers; l += kThreads) {
      const double2 sm = layer_sums_smem(S.lptr, S.stage, l);
      a.d_sumsq[2 * l] = sm.x;
      a.d_sumsq[2 * l + 1] = sm.y;
    }
    return;
  }

  if (kMode == kPeer && LARS_PEER_EARLY) {
    // A layer that lies entirely inside this shard needs only the local sums:
    // every CTA takes its lambda now and starts the update, while warp 0 of
    // CTA 0 exchanges the sums with the other ranks.  The chunks of the
    // layers shared with other ranks come last in the claim order (`order`)
    // and wait for that exchange (UpdatePipe::wait_shared).
    stage_partials(P, a.partial, S.stage);
    for (int l = threadIdx.x; l < P.nlayers; l += kThreads) {
      const double2 sm = layer_sums_smem(S.lptr, S.stage, l);
      if (cta == 0)
        for (int q = 0; q < a.world; ++q) {
          double* slot = a.x_peer[q] + ((size_t)a.rank * P.nlayers + l) * 2;
          slot[0] = sm.x;
          slot[1] = sm.y;
        }
      if (P.layer_seg[l] < 0 || (S.lflags[l] & LARS_SEG_SHARED)) continue;
      // (the rank-order sum of the rows would add exact zeros to these)
      const double lam = device_lambda(a.hp, S.lflags[l], sm.x, sm.y);
      S.coef[l] = (coef_t)__dmul_rn(lam, lr);  // (lam * lr), optim.py:130
      if (cta == 0) {
        if (a.d_sumsq) {
          a.d_sumsq[2 * l] = sm.x;
          a.d_sumsq[2 * l + 1] = sm.y;
        }
        if (a.d_lambda) a.d_lambda[l] = lam;
      }
    }
    __syncthreads();
    if (cta == 0 && warp == 0) {
      if (lane == 0) {
        trace(gw, 5, lane);
        const unsigned epoch = *a.nv_epoch + 1;
        rank_barrier(a, epoch);
        *a.nv_epoch = epoch;
        trace(gw, 6, lane);
      }
      __syncwarp();
      for (int l = lane; l < P.nlayers; l += 32) {
        if (P.layer_seg[l] >= 0 && !(S.lflags[l] & LARS_SEG_SHARED)) continue;
        double w2 = 0.0, g2 = 0.0;
        for (int q = 0; q < a.world; ++q) {  // rank order: identical on all ranks
          const double2 v = __ldcg(reinterpret_cast<const double2*>(
              a.x_peer[a.rank] + ((size_t)q * P.nlayers + l) * 2));
          w2 += v.x;
          g2 += v.y;
        }
        const double lam = device_lambda(a.hp, S.lflags[l], w2, g2);
        a.coef_g[l] = __dmul_rn(lam, lr);
        if (a.d_sumsq) {
          a.d_sumsq[2 * l] = w2;
          a.d_sumsq[2 * l + 1] = g2;
        }
        if (a.d_lambda) a.d_lambda[l] = lam;
      }
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release_u32(a.shared_ready, peer_tag);
      if (exhausted && lane == 0) *a.peer_launch = peer_tag;
    }
    if (exhausted) return;
    trace(gw, 3, lane);
    up.run();
    trace(gw, 4, lane);
    grid_barrier(a.bar, gridDim.x);
    if (cta == 0 && threadIdx.x == 0) {
      const unsigned e2 = *a.nv_epoch + 1;
      rank_barrier(a, e2);
      *a.nv_epoch = e2;
      *a.peer_launch = peer_tag;
    }
    return;
  }
  if (kMode == kPeer) {
    // the other CTAs' rings fill while CTA 0 exchanges the per-layer sums
    // with the other ranks
    if (cta == 0) {
      unsigned epoch;
      stage_partials(P, a.partial, S.stage);
      for (int l = threadIdx.x; l < P.nlayers; l += kThreads) {
        const double2 sm = layer_sums_smem(S.lptr, S.stage, l);
        for (int q = 0; q < a.world; ++q) {
          double* slot = a.x_peer[q] + ((size_t)a.rank * P.nlayers + l) * 2;
          slot[0] = sm.x;
          slot[1] = sm.y;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        trace(gw, 5, lane);
        epoch = *a.nv_epoch + 1;
        rank_barrier(a, epoch);
        *a.nv_epoch = epoch;
        trace(gw, 6, lane);
      }
    }
    // only CTA 0 wrote since the last barrier (the others issued loads)
    grid_wait(a.bar, grid_arrive(a.bar, gridDim.x, cta == 0));
    // global sums: the ranks' partials added in rank order (identical on all ranks)
    for (int l = threadIdx.x; l < P.nlayers; l += kThreads) {
      double w2 = 0.0, g2 = 0.0;
      for (int q = 0; q < a.world; ++q) {
        const double2 v = __ldcg(reinterpret_cast<const double2*>(
            a.x_peer[a.rank] + ((size_t)q * P.nlayers + l) * 2));
        w2 += v.x;
        g2 += v.y;
      }
      const double lam = device_lambda(a.hp, S.lflags[l], w2, g2);
      S.coef[l] = (coef_t)__dmul_rn(lam, lr);  // (lam * lr), optim.py:130
      if (cta == 0) {
        if (a.d_sumsq) {
          a.d_sumsq[2 * l] = w2;
          a.d_sumsq[2 * l + 1] = g2;
        }
        if (a.d_lambda) a.d_lambda[l] = lam;
      }
    }
    if (exhausted) return;
    __syncthreads();
    trace(gw, 3, lane);
    up.run();
    trace(gw, 4, lane);
    // every rank's shard must have landed everywhere before anyone goes on:
    // each CTA's stores are ordered before its arrival, CTA 0's system-scope
    // fence in the rank barrier then covers all of them
    grid_barrier(a.bar, gridDim.x);
    if (cta == 0 && threadIdx.x == 0) {
      const unsigned e2 = *a.nv_epoch + 1;
      rank_barrier(a, e2);
      *a.nv_epoch = e2;
    }
    return;
  }

  // ---- lambda and lambda*lr per layer, into shared memory ----
  if (kMode == kFull) {
    if (!LARS_POLL_STAGE) stage_partials(P, a.partial, S.stage);
    trace(gw, 5, lane);
    for (int l = threadIdx.x; l < P.nlayers; l += kThreads) {
      const double2 sm = layer_sums_smem(S.lptr, S.stage, l);
      const double lam = device_lambda(a.hp, S.lflags[l], sm.x, sm.y);
      S.coef[l] = (coef_t)__dmul_rn(lam, lr);  // (lam * lr), optim.py:130
      if (cta == 0) {
        if (a.d_sumsq) {
          a.d_sumsq[2 * l] = sm.x;
          a.d_sumsq[2 * l + 1] = sm.y;
        }
        if (a.d_lambda) a.d_lambda[l] = lam;
      }
    }
    trace(gw, 6, lane);
    if (exhausted) return;
  } else {
    cp_async_wait<0>();  // layer tables (issued at entry)
    __syncthreads();
    for (int l = threadIdx.x; l < P.nlayers; l += kThreads) {
      const double lam = device_lambda(a.hp, S.lflags[l], a.d_sumsq_in[2 * l],
                                       a.d_sumsq_in[2 * l + 1]);
      S.coef[l] = (coef_t)__dmul_rn(lam, lr);
      if (cta == 0 && a.d_lambda) a.d_lambda[l] = lam;
    }
    if (exhausted) return;
  }
  __syncthreads();
  trace(gw, 3, lane);

  // ---- phase B ----
  up.run();
  trace(gw, 4, lane);
}

// ---------------------------------------------------------------------------
// the streamed sharded step (lars_step_peer_stream)
//
// The fused peer kernel above runs its reduce-scatter (inbound NVLink: pulls
// from the peers) and its all-gather (outbound: stores to the peers) one
// after the other, because lambda needs whole-layer norms.  But a layer that
// lies entirely inside this rank's shard needs only local sums, so its update
// can start as soon as ITS reduce-scatter is done.  This kernel pipelines the
// two over the shard's segments:
//   A-workers (warps 0-3 of every CTA): claim chunks in `order` (interior
//     segments in buffer order, then the ones shared with other ranks), pull
//     and sum the rank gradients (rank order), store the reduced gradient,
//     write the chunk's (sum w^2, sum g^2); the warp that reduces a segment's
//     last chunk sums its chunks in fixed order into seg_part and tags it
//     ready; when every shared segment is final, one row of per-layer partial
//     sums (shared layers only) goes to every rank's exchange buffer;
//   B-workers (warps 4-7, and the A-workers once A runs dry): claim the same
//     chunks in the same order, wait until the chunk's segment is final (and,
//     for a shared layer, until every rank's row arrived), take lambda from the
//     segment's sums (or the rows, summed in rank order), then update and store
//     the new weights to every rank -- inbound and outbound traffic overlap.
// The end is the fused kernel's: grid barrier, per-layer sums to every rank
// (for the reported lambdas), cross-rank barrier.  Every wait has a timeout
// (LARS_STATUS_RANK_TIMEOUT) so a missing peer cannot hang the GPU.
// ---------------------------------------------------------------------------

#ifndef LARS_AWARPS
#define LARS_AWARPS 4
#endif
constexpr int kAWarps = LARS_AWARPS;                      // A-workers per CTA
#ifndef LARS_STREAM_RING
#define LARS_STREAM_RING 1   // A-workers stream through a cp.async ring (0: registers)
#endif
constexpr unsigned long long kStreamTimeoutNs = 20ull * 1000000000ull;
constexpr unsigned long long kRowFlagBase = 0x7FF8DEAD00000000ull;  // NaN-boxed tag

__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const void* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys_u64(void* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

// row layout in each rank's exchange buffer: region r (0: shared layers,
// mid-step; 1: every layer, end of step) x [world] rows x (2L + 2) doubles,
// the last two holding the row's tag
__device__ __forceinline__ double* xrow(const StepArgs& a, int owner, int region, int from) {
  const size_t rowlen = 2 * (size_t)a.p.nlayers + 2;
  return a.x_peer[owner] + ((size_t)region * a.world + from) * rowlen;
}

// one warp: this rank's row of per-layer sums into every rank's buffer, then
// the tag (after a system-scope fence, so the values land first)
__device__ void publish_row(const StepArgs& a, int region, unsigned tag, int lane) {
  const DevPlan& P = a.p;
  for (int q = 0; q < a.world; ++q) {
    double* dst = xrow(a, q, region, a.rank);
    for (int l = lane; l < P.nlayers; l += 32) {
      const int sg = P.layer_seg[l];
      double2 v = make_double2(0.0, 0.0);
      if (sg >= 0 && (region == 1 || (P.segs[sg].flags & LARS_SEG_SHARED))) v = __ldcg(a.seg_part + sg);
      dst[2 * l] = v.x;
      dst[2 * l + 1] = v.y;
    }
  }
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    for (int q = 0; q < a.world; ++q)
      st_relaxed_sys_u64(xrow(a, q, region, a.rank) + 2 * P.nlayers, kRowFlagBase | tag);
  }
  __syncwarp();
}

// wait (one warp) until every rank's row of `region` carries `tag`
__device__ bool wait_rows(const StepArgs& a, int region, unsigned tag, int lane) {
  const unsigned long long t0 = global_ns();
  bool ok = true;
  for (;;) {
    bool mine = true;
    if (lane < a.world)
      mine = ld_relaxed_sys_u64(xrow(a, a.rank, region, lane) + 2 * a.p.nlayers) == (kRowFlagBase | tag);
    if (__all_sync(0xffffffffu, mine)) break;
    if (global_ns() - t0 > kStreamTimeoutNs) {
      if (lane == 0) atomicOr(&a.d_info->status, LARS_STATUS_RANK_TIMEOUT);
      ok = false;
      break;
    }
    __nanosleep(100);
  }
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  return ok;
}

// A-worker: reduce-scatter + per-chunk sums until the claim counter runs dry
// The segment whose chunk count just reached its total: sum its chunks'
// partials in chunk order (fixed lane assignment + butterfly), tag it ready;
// after the last shared segment, publish this rank's row.  One warp.
__device__ void finish_segment(const StepArgs& a, int sg, int lane, unsigned launch, unsigned tag) {
  const DevPlan& P = a.p;
  __threadfence();
  const int c0 = P.seg_c0[sg], c1 = P.seg_c0[sg + 1];
  double sw = 0.0, sgm = 0.0;
  for (int j = c0 + lane; j < c1; j += 32) {
    const double2 v = __ldcg(a.apart + j);
    sw += v.x;
    sgm += v.y;
  }
  sw = warp_sum(sw);
  sgm = warp_sum(sgm);
  bool shared_all = false;
  if (lane == 0) {
    a.seg_part[sg] = make_double2(sw, sgm);
    __threadfence();
    st_release_u32(a.seg_ready + sg, tag);
    if (P.segs[sg].flags & LARS_SEG_SHARED) {
      const unsigned d = atomicAdd(a.shared_done, 1u);
      shared_all = (d + 1u - launch * (unsigned)P.nshared) == (unsigned)P.nshared;
    }
  }
  if (__shfl_sync(0xffffffffu, shared_all ? 1 : 0, 0)) {
    __threadfence();
    publish_row(a, 0, tag, lane);
  }
}

// One claimed position k of `order` with the loads in registers (kU batches
// per rank in flight): pull and sum the rank gradients, store the reduced
// gradient, the chunk's sums, count it; the segment's last chunk finishes it.
template <bool kCarry, int kU>
__device__ void reduce_chunk_regs(const StepArgs& a, int lane, int k, unsigned launch, unsigned tag) {
  const DevPlan& P = a.p;
  const uint64_t keep = policy_evict_last();
  float* gs = const_cast<float*>(a.g);  // the local reduced-gradient scratch
  const int c = P.order[k];
  const DevChunk ch = P.chunks[c];
  const int sg = P.chunk_seg[c];
  const double carry_w = kCarry ? __ldcg(a.ccarry + c) : 0.0;
  const int nb = (ch.nvec + kBatchVec - 1) / kBatchVec;
  double aw = 0.0, ag = 0.0;
#pragma unroll 1
  for (int b0 = 0; b0 < nb; b0 += kU) {
    float4 acc[kU];
    int64_t ev[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int rel = (b0 + u) * kBatchVec + lane;
      ev[u] = (b0 + u < nb && rel < ch.nvec) ? (ch.vbeg + rel) * 4 : -1;
      acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll 1
    for (int q = 0; q < a.world; ++q) {  // rank order: same sum on every rank
      const float* gq = a.g_peer[q];
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        v[u] = ev[u] >= 0 ? __ldcg(reinterpret_cast<const float4*>(gq + ev[u]))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        acc[u].x += v[u].x;
        acc[u].y += v[u].y;
        acc[u].z += v[u].z;
        acc[u].w += v[u].w;
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (ev[u] < 0) continue;
      st4(gs + ev[u], acc[u], keep);
      ag = sumsq4(acc[u], ag);
      if (!kCarry) aw = sumsq4(*reinterpret_cast<const float4*>(a.w + ev[u]), aw);
    }
  }
  ag = warp_sum(ag);
  aw = kCarry ? carry_w : warp_sum(aw);
  int last = 0;
  if (lane == 0) a.apart[c] = make_double2(aw, ag);
  __syncwarp();
  __threadfence();  // every lane's gradient stores and the sums before the count
  __syncwarp();
  if (lane == 0) {
    const unsigned nch = (unsigned)(P.seg_c0[sg + 1] - P.seg_c0[sg]);
    const unsigned old = atomicAdd(a.seg_cnt + sg, 1u);
    last = (old + 1u - launch * nch) == nch;
  }
  if (__shfl_sync(0xffffffffu, last, 0)) finish_segment(a, sg, lane, launch, tag);
}

template <bool kCarry, int kU>
__device__ void stream_reduce(const StepArgs& a, int lane, unsigned launch, unsigned tag) {
  for (;;) {
    int k = 0;
    if (lane == 0) k = (int)atomicAdd(a.ctr_a, 1ull);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= a.p.nchunks) break;
    reduce_chunk_regs<kCarry, kU>(a, lane, k, launch, tag);
  }
}

// A-worker with a cp.async ring: each stage holds one batch from every rank
// (and w when its norm is not carried), so a warp keeps kStages batches in
// flight instead of a few in registers.  Completed chunks are signalled in
// groups of kSignal: one fence per group (a fence also waits for the ring's
// loads in flight).  kP: ranks rounded up to 2, 4 or 8.
template <bool kCarry, int kP>
__device__ void stream_reduce_ring(const StepArgs& a, const Smem& S, int lane, unsigned launch,
                                   unsigned tag) {
  const DevPlan& P = a.p;
  constexpr int kSlots = kP + (kCarry ? 0 : 1);
  constexpr int kStages = (kStagesB * 3) / kSlots;
  constexpr int kSignal = 4;
  static_assert(kStages >= 2 && kStages <= kQueue, "ring stages");
  const uint64_t keep = policy_evict_last();
  const uint64_t pass = policy_evict_first_rt();
  float* gs = const_cast<float*>(a.g);
  float4* ring = S.ring;
  QEnt* q = S.queue;  // claimed chunks, issue side -> consume side
  const int world = a.world;
  // ---- issue side: claims one chunk ahead ----
  int pend = 0;
  if (lane == 0) pend = (int)atomicAdd(a.ctr_a, 1ull);
  int ik = __shfl_sync(0xffffffffu, pend, 0);
  if (lane == 0) pend = (int)atomicAdd(a.ctr_a, 1ull);
  bool issuing = true;
  int ij = 0, inb = 0, itail = 0, invec = 0;
  int64_t ivb = 0;
  auto issue = [&](int st) -> bool {
    bool did = false;
    if (issuing && ij == inb) {
      if (ik >= P.nchunks) {
        issuing = false;
      } else {
        const int c = P.order[ik];
        const DevChunk ch = P.chunks[c];
        ivb = ch.vbeg;
        invec = ch.nvec;
        ij = 0;
        inb = (ch.nvec + kBatchVec - 1) / kBatchVec;
        if (lane == 0) {
          QEnt e;
          e.vbeg = ch.vbeg;
          e.nvec = ch.nvec;
          e.layer = P.chunk_seg[c];  // (the segment)
          e.id = c;
          e.pad = inb;
          q[itail & (kQueue - 1)] = e;
        }
        ++itail;
        __syncwarp();
        ik = __shfl_sync(0xffffffffu, pend, 0);
        if (lane == 0) pend = (int)atomicAdd(a.ctr_a, 1ull);
      }
    }
    if (issuing) {
      const int rel = ij * kBatchVec + lane;
      const bool ok = rel < invec;
      const int64_t e = ok ? (ivb + rel) * 4 : 0;
#pragma unroll
      for (int r = 0; r < kP; ++r)
        if (r < world) cp_async16(ring + (st * kSlots + r) * 32 + lane, a.g_peer[r] + e, ok, pass);
      if (!kCarry) cp_async16(ring + (st * kSlots + kP) * 32 + lane, a.w + e, ok, pass);
      ++ij;
      did = true;
    }
    cp_async_commit();
    return did;
  };
  // ---- consume side ----
  int chead = 0, cj = 0, cnb = 0;
  QEnt cur{0, 0, 0, -1, 0};
  double aw = 0.0, ag = 0.0;
  int done_seg = -1;  // lane i < ndone: segment of the i-th unsignalled chunk
  int ndone = 0;
  auto signal = [&]() {
    if (ndone == 0) return;
    __syncwarp();
    __threadfence();  // every lane's gradient stores (and lane 0's partials)
    __syncwarp();
    bool last = false;
    if (lane < ndone) {
      const unsigned nch = (unsigned)(P.seg_c0[done_seg + 1] - P.seg_c0[done_seg]);
      const unsigned old = atomicAdd(a.seg_cnt + done_seg, 1u);
      last = (old + 1u - launch * nch) == nch;
    }
    unsigned m = __ballot_sync(0xffffffffu, last);
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      finish_segment(a, __shfl_sync(0xffffffffu, done_seg, src), lane, launch, tag);
    }
    ndone = 0;
    done_seg = -1;
  };
  auto finish_chunk = [&]() {
    ag = warp_sum(ag);
    aw = kCarry ? __ldcg(a.ccarry + cur.id) : warp_sum(aw);
    if (lane == 0) a.apart[cur.id] = make_double2(aw, ag);
    if (lane == ndone) done_seg = cur.layer;
    ++ndone;
    aw = 0.0;
    ag = 0.0;
    if (ndone == kSignal) signal();
  };
  int issued = 0, consumed = 0;
#pragma unroll 1
  for (int st = 0; st < kStages; ++st) issued += issue(st) ? 1 : 0;
  int st = 0;
#pragma unroll 1
  while (consumed < issued) {
    cp_async_wait<kStages - 1>();
    if (cj == cnb) {
      if (cur.id >= 0) finish_chunk();
      cur = q[chead & (kQueue - 1)];
      ++chead;
      cj = 0;
      cnb = cur.pad;
    }
    const int rel = cj * kBatchVec + lane;
    if (rel < cur.nvec) {
      float4 acc = ring[(st * kSlots) * 32 + lane];
#pragma unroll
      for (int r = 1; r < kP; ++r) {  // rank order: the same sum on every rank
        if (r < world) {
          const float4 v = ring[(st * kSlots + r) * 32 + lane];
          acc.x += v.x;
          acc.y += v.y;
          acc.z += v.z;
          acc.w += v.w;
        }
      }
      st4(gs + (cur.vbeg + rel) * 4, acc, keep);
      ag = sumsq4(acc, ag);
      if (!kCarry) aw = sumsq4(ring[(st * kSlots + kP) * 32 + lane], aw);
    }
    ++cj;
    ++consumed;
    __syncwarp();
    issued += issue(st) ? 1 : 0;
    st = st + 1 == kStages ? 0 : st + 1;
  }
  cp_async_wait<0>();
  if (cur.id >= 0) finish_chunk();
  signal();
}

// B-worker pipeline: UpdatePipe's cp.async ring fed from the claim order,
// each chunk released by its segment's readiness
template <bool kCarry>
struct StreamPipe {
  static constexpr int kStages = kStagesB;
  const StepArgs& a;
  const Smem& S;
  const int lane;
  const int nchunks;
  const unsigned tag;
  const double lr;
  uint64_t pol;
  int pending = 0;
  int blk_next = 0, blk_end = 0;
  bool issuing = true, have_nx = false, rows_ok = false;
  DevChunk nx{0, 0, 0};
  int nx_id = 0;
  int ready_seg = -1;
  double coef_cur = 0.0;
  QEntS ic{0, 0, 0, 0, 0, 0.0};
  int ij = 0, inb = 0, tail = 0;
  int64_t issued = 0;
  QEntS cc{0, 0, 0, -1, 0, 0.0};
  int cj = 0, cnb = 0, head = 0;
  int64_t consumed = 0;
  double aw = 0.0;
  bool bad = false;
  int gw = 0;
  unsigned long long wait_ns = 0;  // time spent waiting for segments (trace builds)
  bool first_ready = true;

  unsigned launch = 0;
  bool a_left = true;  // reduce-scatter chunks may remain: steal them while waiting

  __device__ StreamPipe(const StepArgs& a_, const Smem& S_, int lane_, unsigned tag_, double lr_)
      : a(a_), S(S_), lane(lane_), nchunks(a_.p.nchunks), tag(tag_), lr(lr_) {
    pol = a.p.pol_b ? policy_evict_normal_rt() : policy_evict_first_rt();
  }

  __device__ __forceinline__ void fetch_next() {
    if (blk_next == blk_end) {
      const int base = __shfl_sync(0xffffffffu, pending, 0);
      if (base >= nchunks) {
        have_nx = false;
        return;
      }
      blk_next = base;
      blk_end = min(base + kClaim, nchunks);
      if (lane == 0) pending = (int)atomicAdd(a.ctr_b, (unsigned long long)kClaim);
    }
    nx_id = a.p.order[blk_next++];
    have_nx = true;
    nx = a.p.chunks[nx_id];
  }

  // the chunk's segment must be final (its reduced gradient stored, its sums
  // known) before its loads are issued; lambda*lr from those sums
  __device__ void ready(int c) {
    const int sg = a.p.chunk_seg[c];
    if (sg == ready_seg) return;
    const unsigned long long t0 = global_ns();
    if (first_ready) {
      first_ready = false;
      trace(gw, 3, lane);
    }
    unsigned backoff = 32;
    while (ld_acquire_u32(a.seg_ready + sg) != tag) {
      if (a_left) {  // do a reduce-scatter chunk instead of spinning
        int k = 0;
        if (lane == 0) k = (int)atomicAdd(a.ctr_a, 1ull);
        k = __shfl_sync(0xffffffffu, k, 0);
        if (k < a.p.nchunks) {
          reduce_chunk_regs<kCarry, 2>(a, lane, k, launch, tag);
          continue;
        }
        a_left = false;
      }
      if (global_ns() - t0 > kStreamTimeoutNs) {
        if (lane == 0) atomicOr(&a.d_info->status, LARS_STATUS_RANK_TIMEOUT);
        break;
      }
      __nanosleep(backoff);
      backoff = min(backoff * 2, 2048u);
    }
    const DevSeg seg = a.p.segs[sg];
    double w2, g2;
    if (seg.flags & LARS_SEG_SHARED) {
      if (!rows_ok) rows_ok = wait_rows(a, 0, tag, lane) || true;
      w2 = 0.0;
      g2 = 0.0;
      for (int q = 0; q < a.world; ++q) {  // rank order: identical on every rank
        const double* r = xrow(a, a.rank, 0, q);
        w2 += __ldcg(r + 2 * seg.layer);
        g2 += __ldcg(r + 2 * seg.layer + 1);
      }
    } else {
      const double2 v = __ldcg(a.seg_part + sg);
      w2 = v.x;
      g2 = v.y;
    }
    const double lam = device_lambda(a.hp, S.lflags[seg.layer], w2, g2);
    coef_cur = __dmul_rn(lam, lr);  // (lam * lr), optim.py:130
    ready_seg = sg;
    wait_ns += global_ns() - t0;
  }

  __device__ __forceinline__ void take_chunk() {
    if (!have_nx) {
      issuing = false;
      return;
    }
    ready(nx_id);
    ic.vbeg = nx.vbeg;
    ic.nvec = nx.nvec;
    ic.layer = nx.layer;
    ic.id = nx_id;
    ic.coef = coef_cur;
    ij = 0;
    inb = (nx.nvec + kBatchVec - 1) / kBatchVec;
    if (lane == 0) reinterpret_cast<QEntS*>(S.queue)[tail % kQueueS] = ic;
    ++tail;
    __syncwarp();
    fetch_next();
  }

  __device__ __forceinline__ void issue(int st) {
    if (issuing && ij == inb) take_chunk();
    if (issuing) {
      const int rel = ij * kBatchVec + lane;
      const bool ok = rel < ic.nvec;
      const int64_t e = ok ? (ic.vbeg + rel) * 4 : 0;
      float4* ring = S.ring;
      cp_async16(ring + (st * 3 + 0) * 32 + lane, a.g + e, ok, pol);
      cp_async16(ring + (st * 3 + 1) * 32 + lane, a.w + e, ok, pol);
      cp_async16(ring + (st * 3 + 2) * 32 + lane, a.m + e, ok, pol);
      ++ij;
      ++issued;
    }
    cp_async_commit();
  }

  __device__ __forceinline__ void finish_chunk() {
    aw = warp_sum(aw);
    if (lane == 0) a.ccarry[cc.id] = aw;
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(&a.d_info->nonfinite_layer, cc.layer);
    aw = 0.0;
    bad = false;
  }

  __device__ __forceinline__ void consume(int st, double mu, double wd, double gsc) {
    if (cj == cnb) {
      if (cc.id >= 0) finish_chunk();
      cc = reinterpret_cast<QEntS*>(S.queue)[head % kQueueS];
      ++head;
      cj = 0;
      cnb = (cc.nvec + kBatchVec - 1) / kBatchVec;
    }
    const int rel = cj * kBatchVec + lane;
    if (rel < cc.nvec) {
      const float4* ring = S.ring;
      const float4 gv = ring[(st * 3 + 0) * 32 + lane];
      const float4 wv = ring[(st * 3 + 1) * 32 + lane];
      const float4 mv = ring[(st * 3 + 2) * 32 + lane];
      const double k = cc.coef;
      float4 mn, wn;
      // optim.py:128-131 in fp64 (see UpdatePipe::consume)
      auto upd = [&](float g, float w, float m, float& mo, float& wo) {
        const double sgv = fma(wd, (double)w, (double)g * gsc);
        const double m64 = fma(mu, (double)m, k * sgv);
        mo = (float)m64;
        wo = w - mo;
      };
      upd(gv.x, wv.x, mv.x, mn.x, wn.x);
      upd(gv.y, wv.y, mv.y, mn.y, wn.y);
      upd(gv.z, wv.z, mv.z, mn.z, wn.z);
      upd(gv.w, wv.w, mv.w, mn.w, wn.w);
      const int64_t e = (cc.vbeg + rel) * 4;
      st4(a.m + e, mn, pol);
      for (int q = 0; q < a.world; ++q) st4(a.w_peer[q] + e, wn, pol);  // all-gather
      aw = sumsq4(wn, aw);
      bad |= !finite4(wn);
    }
    ++cj;
    ++consumed;
  }

  __device__ void run() {
    if (lane == 0) pending = (int)atomicAdd(a.ctr_b, (unsigned long long)kClaim);
    fetch_next();
#pragma unroll 1
    for (int st = 0; st < kStages; ++st) issue(st);
    const double mu = a.hp.momentum, wd = a.hp.weight_decay, gsc = a.hp.grad_scale;
    int st = 0;
#pragma unroll 1
    while (consumed < issued) {
      cp_async_wait<kStages - 2>();
      consume(st, mu, wd, gsc);
      if (consumed < issued) consume(st + 1, mu, wd, gsc);
      issue(st);
      issue(st + 1);
      st = (st + 2 == kStages) ? 0 : st + 2;
    }
    cp_async_wait<0>();
    if (cc.id >= 0) finish_chunk();
  }
};

template <bool kCarry>
__global__ void __launch_bounds__(kThreads, kMinBlocksPerSM) lars_stream_kernel(StepArgs a) {
  const DevPlan& P = a.p;
  const int warp = threadIdx.x >> 5;
  const Smem S = carve(P, warp);
  const int cta = blockIdx.x;
  const int lane = threadIdx.x & 31;
  const int gw = cta * kWarps + warp;
  trace(gw, 0, lane);
  for (int l = threadIdx.x; l < P.nlayers; l += kThreads) cp_async4(S.lflags + l, P.layer_flags + l, true);
  cp_async_commit();
  const int64_t it = *a.d_iter;
  const bool exhausted = !(a.hp.flags & LARS_STEP_EXPLICIT_LR) && it > a.hp.max_iters;
  const double lr = exhausted ? 0.0 : device_lr(a.hp, it);
  const unsigned launch = *reinterpret_cast<volatile unsigned*>(a.stream_launch);
  const unsigned tag = launch + 1u;
  if (cta == 0 && threadIdx.x == 0) {
    a.d_info->lr = lr;
    a.d_info->iteration = it;
    a.d_info->nonfinite_layer = INT_MAX;
    a.d_info->status = exhausted ? LARS_STATUS_EXHAUSTED : 0;
    __threadfence();
    // every rank's gradient is complete before anyone pulls it
    const unsigned e0 = *a.nv_epoch + 1;
    rank_barrier(a, e0);
    *a.nv_epoch = e0;
  }
  cp_async_wait<0>();
  grid_barrier(a.bar, gridDim.x);
  if (exhausted) return;
  trace(gw, 2, lane);
  if (cta == 0 && threadIdx.x == 0 && (a.hp.flags & LARS_STEP_ADVANCE_ITER)) *a.d_iter = it + 1;
  if (P.nshared == 0 && cta == 0 && warp == 0) publish_row(a, 0, tag, lane);  // nothing shared: empty row
  if (warp < kAWarps) {
#if LARS_STREAM_RING
    if (a.world > 4)
      stream_reduce_ring<kCarry, 8>(a, S, lane, launch, tag);
    else if (a.world > 2)
      stream_reduce_ring<kCarry, 4>(a, S, lane, launch, tag);
    else
      stream_reduce_ring<kCarry, 2>(a, S, lane, launch, tag);
#else
    if (a.world >= 4)
      stream_reduce<kCarry, 2>(a, lane, launch, tag);
    else
      stream_reduce<kCarry, 4>(a, lane, launch, tag);
#endif
    trace(gw, 1, lane);
  }
  StreamPipe<kCarry> up(a, S, lane, tag, lr);
  up.gw = gw;
  up.launch = launch;
  up.run();
  trace(gw, 4, lane);
  trace_val(gw, 6, up.wait_ns, lane);
  // every shard landed everywhere; per-layer sums for the reported lambdas
  grid_barrier(a.bar, gridDim.x);
  trace(gw, 5, lane);
  if (cta != 0) return;
  if (warp == 0) publish_row(a, 1, tag, lane);
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned e1 = *a.nv_epoch + 1;
    rank_barrier(a, e1);  // its leading system fence also publishes this rank's stores
    *a.nv_epoch = e1;
  }
  __syncthreads();
  for (int l = threadIdx.x; l < P.nlayers; l += kThreads) {
    double w2 = 0.0, g2 = 0.0;
    for (int q = 0; q < a.world; ++q) {
      const double* r = xrow(a, a.rank, 1, q);
      w2 += __ldcg(r + 2 * l);
      g2 += __ldcg(r + 2 * l + 1);
    }
    if (a.d_sumsq) {
      a.d_sumsq[2 * l] = w2;
      a.d_sumsq[2 * l + 1] = g2;
    }
    if (a.d_lambda) a.d_lambda[l] = device_lambda(a.hp, S.lflags[l], w2, g2);
  }
  if (threadIdx.x == 0) {
    *a.ctr_a = 0ull;
    *a.ctr_b = 0ull;
    *a.stream_launch = launch + 1u;
  }
}

// Cross-rank barrier on its own (one thread): the bench aligns the ranks with
// it between the untimed L2 flush and a timed step, so per-GPU differences in
// the flush's duration are not billed to the step's start barrier.
__global__ void rank_barrier_kernel(StepArgs a) {
  const unsigned e = *a.nv_epoch + 1;
  rank_barrier(a, e);
  *a.nv_epoch = e;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

struct Plan {
  // host copies
  int32_t grid = 0;
  int32_t nlayers = 0;
  int32_t max_pieces_cta = 0;
  int32_t max_slots_cta = 0;
  int32_t smem_bytes = 0;
  int64_t nbatches = 0;
  int64_t elements = 0;
  bool host_only = false;
  std::vector<DevSeg> segs;
  std::vector<int64_t> warp_b0;
  std::vector<int32_t> warp_seg0, warp_slot0, cta_seg0, cta_npieces, cta_piece0;
  std::vector<int32_t> piece_seg, piece_cta, piece_slot_lo, piece_slot_hi, piece_pos;
  std::vector<int32_t> layer_piece_ptr, layer_piece_idx, layer_flags;
  std::vector<DevChunk> chunks;
  std::vector<int32_t> chunk_seg, warp_ch0, cta_ch0;
  std::vector<int64_t> chunk_b0;  // first batch of each chunk (host only)
  std::vector<unsigned char> cta_rec;  // [grid][cta_rec_stride]
  int32_t cta_rec_stride = 0;
  int64_t keep_nb = 0;
  int32_t pol_b = 1;
  int32_t chunk_batches = kChunkBatches;
  bool chunk_override = false;
  std::vector<int32_t> seg_c0, order, layer_seg;
  int32_t nshared = 0;
  // device
  void* dmem = nullptr;
  DevPlan dev{};
  size_t ws_partial_off = 0, ws_pub_off = 0, ws_carry_off = 0, ws_coef_off = 0, ws_bytes = 0;
  size_t ws_apart_off = 0, ws_segcnt_off = 0, ws_segready_off = 0, ws_segpart_off = 0;
};

int cuda_code(cudaError_t e) { return e == cudaSuccess ? LARS_OK : LARS_ERR_CUDA_BASE + (int)e; }

int stage_pieces_for(size_t npieces) {
  return npieces * sizeof(double2) <= kMaxStageBytes ? (int)npieces : 0;
}

// segment index (into plan.segs) of global batch b: last seg with bstart <= b
int seg_of_batch(const std::vector<DevSeg>& segs, int64_t b) {
  int lo = 0, hi = (int)segs.size() - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (segs[mid].bstart <= b) lo = mid; else hi = mid - 1;
  }
  return lo;
}

int build_partition(Plan& pl, int grid) {
  pl.grid = grid;
  const int nw = grid * kWarps;
  const int64_t NB = pl.nbatches;
  pl.warp_b0.assign(nw + 1, 0);
  for (int k = 0; k <= nw; ++k)
    pl.warp_b0[k] = (int64_t)(((__int128)NB * k) / nw);
  pl.warp_seg0.assign(nw, 0);
  pl.warp_slot0.assign(nw, 0);
  pl.cta_seg0.assign(grid, 0);
  pl.cta_npieces.assign(grid, 0);
  pl.cta_piece0.assign(grid, 0);
  pl.piece_seg.clear();
  pl.piece_cta.clear();
  pl.piece_slot_lo.clear();
  pl.piece_slot_hi.clear();
  pl.max_pieces_cta = 1;
  pl.max_slots_cta = 1;
  int32_t npieces = 0;
  for (int c = 0; c < grid; ++c) {
    const int64_t B0 = pl.warp_b0[c * kWarps], B1 = pl.warp_b0[(c + 1) * kWarps];
    pl.cta_piece0[c] = npieces;
    if (B0 >= B1) {
      pl.cta_seg0[c] = 0;
      pl.cta_npieces[c] = 0;
      for (int w = 0; w < kWarps; ++w) {
        pl.warp_seg0[c * kWarps + w] = 0;
        pl.warp_slot0[c * kWarps + w] = 0;
      }
      continue;
    }
    const int s0 = seg_of_batch(pl.segs, B0);
    const int s1 = seg_of_batch(pl.segs, B1 - 1);
    const int npc = s1 - s0 + 1;
    pl.cta_seg0[c] = s0;
    pl.cta_npieces[c] = npc;
    std::vector<int32_t> lo(npc, INT_MAX), hi(npc, INT_MIN);
    int slot = 0;
    for (int w = 0; w < kWarps; ++w) {
      const int gw = c * kWarps + w;
      const int64_t b0 = pl.warp_b0[gw], b1 = pl.warp_b0[gw + 1];
      pl.warp_slot0[gw] = slot;
      if (b0 >= b1) {
        pl.warp_seg0[gw] = s0;
        continue;
      }
      const int ws0 = seg_of_batch(pl.segs, b0), ws1 = seg_of_batch(pl.segs, b1 - 1);
      pl.warp_seg0[gw] = ws0;
      for (int s = ws0; s <= ws1; ++s, ++slot) {
        lo[s - s0] = std::min(lo[s - s0], slot);
        hi[s - s0] = std::max(hi[s - s0], slot + 1);
      }
    }
    for (int i = 0; i < npc; ++i) {
      pl.piece_seg.push_back(s0 + i);
      pl.piece_cta.push_back(c);
      pl.piece_slot_lo.push_back(lo[i]);
      pl.piece_slot_hi.push_back(hi[i]);
    }
    npieces += npc;
    pl.max_pieces_cta = std::max(pl.max_pieces_cta, npc);
    pl.max_slots_cta = std::max(pl.max_slots_cta, slot);
  }
  // layer CSR
  const int L = pl.nlayers;
  pl.layer_piece_ptr.assign(L + 1, 0);
  for (int p = 0; p < npieces; ++p) pl.layer_piece_ptr[pl.segs[pl.piece_seg[p]].layer + 1]++;
  for (int l = 0; l < L; ++l) pl.layer_piece_ptr[l + 1] += pl.layer_piece_ptr[l];
  pl.layer_piece_idx.assign(npieces, 0);
  pl.piece_pos.assign(npieces, 0);
  std::vector<int32_t> fill(pl.layer_piece_ptr.begin(), pl.layer_piece_ptr.end() - 1);
  for (int p = 0; p < npieces; ++p) {
    const int pos = fill[pl.segs[pl.piece_seg[p]].layer]++;
    pl.layer_piece_idx[pos] = p;
    pl.piece_pos[p] = pos;
  }
  if ((size_t)npieces * sizeof(double2) > kRingBytes) return LARS_ERR_TOO_MANY_PIECES;
  // phase-B chunks and, per warp, the chunks starting in its phase-A run.
  // Chunk size: 8 batches, 4 when a warp's share is under 40 batches (small
  // shards: finer balance at the drain; measured ResNet-50 P=8 shard 30.7 ->
  // 28.6 us, AlexNet-BN P=8 42.5 -> 41.0 us, 1M sweep 19.3 -> 17.5 us; 8
  // stays best at >= 50 batches per warp), unless LARS_CHUNK_BATCHES is set
  if (!pl.chunk_override) pl.chunk_batches = (NB >= 40 * (int64_t)nw) ? kChunkBatches : 4;
  pl.chunks.clear();
  pl.chunk_seg.clear();
  pl.chunk_b0.clear();
  // Chunks are handed out in buffer order; they shrink towards the end
  // (8 -> 2 -> 1 batches) so that when the counter runs dry every warp is at
  // most one small chunk away from done.
  // (long runs per warp drain evenly with a shorter taper: AlexNet-BN, 201
  // batches per warp, 235.3 -> 230.7 us with 10 % / 2 %; ResNet-50 (84) and
  // a 16M sweep (53) are 0.6 / 1.7 us slower with it)
  const bool long_runs = NB >= 150 * (int64_t)nw;
  const int64_t t2 = long_runs ? LARS_TAPER2_LONG : LARS_TAPER2, t1 = long_runs ? LARS_TAPER1_LONG : LARS_TAPER1;
  const int64_t taper2 = NB - NB * t2 / 1000, taper1 = NB - NB * t1 / 1000;
  for (int si = 0; si < (int)pl.segs.size(); ++si) {
    const DevSeg& sg = pl.segs[si];
    for (int64_t j = 0; j < sg.bend - sg.bstart;) {
      const int64_t bglob = sg.bstart + j;
      const int64_t want = bglob < taper2 ? pl.chunk_batches : (bglob < taper1 ? std::min(2, pl.chunk_batches) : 1);
      const int64_t nb = std::min<int64_t>(want, sg.bend - sg.bstart - j);
      DevChunk ch;
      ch.vbeg = sg.vec_off + j * kBatchVec;
      ch.nvec = (int32_t)std::min<int64_t>(nb * kBatchVec, sg.vec_len - j * kBatchVec);
      ch.layer = sg.layer;
      pl.chunks.push_back(ch);
      pl.chunk_seg.push_back(si);
      pl.chunk_b0.push_back(bglob);
      j += nb;
    }
  }
  if (pl.chunks.size() > (size_t)INT_MAX / 2) return LARS_ERR_INVALID;
  pl.warp_ch0.assign(nw + 1, 0);
  for (int k = 0; k <= nw; ++k)
    pl.warp_ch0[k] = (int32_t)(std::lower_bound(pl.chunk_b0.begin(), pl.chunk_b0.end(),
                                                pl.warp_b0[k]) - pl.chunk_b0.begin());
  pl.cta_ch0.assign(grid + 1, 0);
  for (int c = 0; c <= grid; ++c) pl.cta_ch0[c] = pl.warp_ch0[c * kWarps];
  pl.max_slots_cta = kWarps * pl.max_pieces_cta;  // slot[warp][piece]
  // per-CTA records: CtaDesc + copies of the CTA's segments
  pl.cta_rec_stride = (int32_t)align_up(sizeof(CtaDesc) + sizeof(DevSeg) * (size_t)pl.max_pieces_cta, 16);
  pl.cta_rec.assign((size_t)grid * pl.cta_rec_stride, 0);
  for (int c = 0; c < grid; ++c) {
    CtaDesc d{};
    d.B0 = pl.warp_b0[c * kWarps];
    d.B1 = pl.warp_b0[(c + 1) * kWarps];
    d.seg0 = pl.cta_seg0[c];
    d.npc = pl.cta_npieces[c];
    d.piece0 = pl.cta_piece0[c];
    d.ch0 = pl.cta_ch0[c];
    d.ch1 = pl.cta_ch0[c + 1];
    unsigned char* r = pl.cta_rec.data() + (size_t)c * pl.cta_rec_stride;
    std::memcpy(r, &d, sizeof(d));
    if (d.npc > 0)
      std::memcpy(r + sizeof(CtaDesc), pl.segs.data() + d.seg0, sizeof(DevSeg) * (size_t)d.npc);
  }
  const size_t smem = smem_layout(pl.max_pieces_cta, pl.max_slots_cta, pl.nlayers,
                                  stage_pieces_for(pl.piece_seg.size())).total;
  if (smem > 227 * 1024) return LARS_ERR_TOO_MANY_PIECES;
  pl.smem_bytes = (int32_t)smem;
  // streamed sharded step: chunk range per segment, claim order (interior
  // segments in buffer order, then the shared ones), segment of each layer
  const int nseg = (int)pl.segs.size();
  pl.seg_c0.assign(nseg + 1, (int32_t)pl.chunks.size());
  for (int c = (int)pl.chunks.size() - 1; c >= 0; --c) pl.seg_c0[pl.chunk_seg[c]] = c;
  for (int si = nseg - 1; si >= 0; --si)
    if (pl.seg_c0[si] > pl.seg_c0[si + 1]) pl.seg_c0[si] = pl.seg_c0[si + 1];
  pl.order.clear();
  pl.nshared = 0;
  for (int pass = 0; pass < 2; ++pass)
    for (int si = 0; si < nseg; ++si) {
      const bool shared = (pl.segs[si].flags & LARS_SEG_SHARED) != 0;
      if (shared != (pass == 1) || pl.segs[si].vec_len == 0) continue;
      if (shared) ++pl.nshared;
      for (int c = pl.seg_c0[si]; c < pl.seg_c0[si + 1]; ++c) pl.order.push_back(c);
    }
  pl.layer_seg.assign(pl.nlayers, -1);
  for (int si = 0; si < nseg; ++si)
    if (pl.segs[si].vec_len > 0) pl.layer_seg[pl.segs[si].layer] = si;
  return LARS_OK;
}

template <int kMode, bool kCarry>
void* kernel_ptr() {
  return reinterpret_cast<void*>(&lars_step_kernel<kMode, kCarry>);
}

void* pick_kernel(int mode, bool carry) {
  if (mode == kFull) return carry ? kernel_ptr<kFull, true>() : kernel_ptr<kFull, false>();
  if (mode == kNorms) return carry ? kernel_ptr<kNorms, true>() : kernel_ptr<kNorms, false>();
  if (mode == kPeer) return carry ? kernel_ptr<kPeer, true>() : kernel_ptr<kPeer, false>();
  if (mode == kPeerStream)
    return carry ? reinterpret_cast<void*>(&lars_stream_kernel<true>)
                 : reinterpret_cast<void*>(&lars_stream_kernel<false>);
  return kernel_ptr<kUpdate, false>();
}

// Each kernel's dynamic shared-memory limit is a per-function attribute that
// every plan needs at least its own size in: only ever raised, so that a plan
// created later with a smaller footprint cannot break the launches of an
// earlier, larger one (per device).
int ensure_smem_attr(void* k, int smem) {
  static std::mutex mu;
  static std::map<std::pair<int, void*>, int> set;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_code(e);
  std::lock_guard<std::mutex> lk(mu);
  int& cur = set[std::make_pair(dev, k)];
  if (smem <= cur) return LARS_OK;
  e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return cuda_code(e);
  cur = smem;
  return LARS_OK;
}

int occupancy(int smem, int* blocks) {
  int best = INT_MAX;
  const int modes[9][2] = {{kFull, 0}, {kFull, 1}, {kNorms, 0}, {kNorms, 1}, {kUpdate, 0},
                           {kPeer, 0}, {kPeer, 1}, {kPeerStream, 0}, {kPeerStream, 1}};
  for (auto& mc : modes) {
    void* k = pick_kernel(mc[0], mc[1] != 0);
    int rc = ensure_smem_attr(k, smem);
    if (rc) return rc;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, kThreads, smem);
    if (e != cudaSuccess) return cuda_code(e);
    if (getenv("LARS_DEBUG_OCC")) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, k);
      fprintf(stderr, "lars occupancy: mode %d carry %d smem %d regs %d -> %d blocks/SM\n", mc[0], mc[1],
              smem, fa.numRegs, n);
    }
    best = std::min(best, n);
  }
  *blocks = best;
  return LARS_OK;
}

template <typename T>
size_t push(std::vector<unsigned char>& blob, const std::vector<T>& v) {
  size_t off = (blob.size() + 255) & ~size_t(255);
  blob.resize(off + sizeof(T) * std::max<size_t>(v.size(), 1));
  if (!v.empty()) std::memcpy(blob.data() + off, v.data(), sizeof(T) * v.size());
  return off;
}

int upload(Plan& pl) {
  std::vector<unsigned char> blob;
  const size_t o_segs = push(blob, pl.segs);
  const size_t o_wb0 = push(blob, pl.warp_b0);
  const size_t o_ws0 = push(blob, pl.warp_seg0);
  const size_t o_wsl = push(blob, pl.warp_slot0);
  const size_t o_cs0 = push(blob, pl.cta_seg0);
  const size_t o_cnp = push(blob, pl.cta_npieces);
  const size_t o_cp0 = push(blob, pl.cta_piece0);
  const size_t o_psl = push(blob, pl.piece_slot_lo);
  const size_t o_psh = push(blob, pl.piece_slot_hi);
  const size_t o_lpp = push(blob, pl.layer_piece_ptr);
  const size_t o_lpi = push(blob, pl.layer_piece_idx);
  const size_t o_ppo = push(blob, pl.piece_pos);
  const size_t o_lfl = push(blob, pl.layer_flags);
  const size_t o_chk = push(blob, pl.chunks);
  const size_t o_chs = push(blob, pl.chunk_seg);
  const size_t o_wch = push(blob, pl.warp_ch0);
  const size_t o_cch = push(blob, pl.cta_ch0);
  const size_t o_rec = push(blob, pl.cta_rec);
  const size_t o_sc0 = push(blob, pl.seg_c0);
  const size_t o_ord = push(blob, pl.order);
  const size_t o_lsg = push(blob, pl.layer_seg);
  cudaError_t e = cudaMalloc(&pl.dmem, blob.size());
  if (e != cudaSuccess) return cuda_code(e);
  e = cudaMemcpy(pl.dmem, blob.data(), blob.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_code(e);
  auto base = static_cast<unsigned char*>(pl.dmem);
  DevPlan& d = pl.dev;
  d.segs = reinterpret_cast<const DevSeg*>(base + o_segs);
  d.warp_b0 = reinterpret_cast<const int64_t*>(base + o_wb0);
  d.warp_seg0 = reinterpret_cast<const int32_t*>(base + o_ws0);
  d.warp_slot0 = reinterpret_cast<const int32_t*>(base + o_wsl);
  d.cta_seg0 = reinterpret_cast<const int32_t*>(base + o_cs0);
  d.cta_npieces = reinterpret_cast<const int32_t*>(base + o_cnp);
  d.cta_piece0 = reinterpret_cast<const int32_t*>(base + o_cp0);
  d.piece_slot_lo = reinterpret_cast<const int32_t*>(base + o_psl);
  d.piece_slot_hi = reinterpret_cast<const int32_t*>(base + o_psh);
  d.layer_piece_ptr = reinterpret_cast<const int32_t*>(base + o_lpp);
  d.layer_piece_idx = reinterpret_cast<const int32_t*>(base + o_lpi);
  d.piece_pos = reinterpret_cast<const int32_t*>(base + o_ppo);
  d.layer_flags = reinterpret_cast<const int32_t*>(base + o_lfl);
  d.chunks = reinterpret_cast<const DevChunk*>(base + o_chk);
  d.chunk_seg = reinterpret_cast<const int32_t*>(base + o_chs);
  d.warp_ch0 = reinterpret_cast<const int32_t*>(base + o_wch);
  d.cta_ch0 = reinterpret_cast<const int32_t*>(base + o_cch);
  d.cta_rec = base + o_rec;
  d.cta_rec_stride = pl.cta_rec_stride;
  d.keep_nb = pl.keep_nb;
  d.pol_b = pl.pol_b;
  d.seg_c0 = reinterpret_cast<const int32_t*>(base + o_sc0);
  d.order = reinterpret_cast<const int32_t*>(base + o_ord);
  d.layer_seg = reinterpret_cast<const int32_t*>(base + o_lsg);
  d.nshared = pl.nshared;
  d.nchunks = (int32_t)pl.chunks.size();
  d.stage_pieces = stage_pieces_for(pl.piece_seg.size());
  d.nseg = (int32_t)pl.segs.size();
  d.nlayers = pl.nlayers;
  d.npieces = (int32_t)pl.piece_seg.size();
  d.grid = pl.grid;
  d.max_pieces_cta = pl.max_pieces_cta;
  d.max_slots_cta = pl.max_slots_cta;
  return LARS_OK;
}

// workspace: [barrier u64 | chunks claimed u32 + warps done u32 | epoch u32 | pad]
//            partial | carry | coef
void layout_workspace(Plan& pl) {
  const size_t np = std::max<size_t>(pl.piece_seg.size(), 1);
  const size_t nc = std::max<size_t>(pl.chunks.size(), 1);
  pl.ws_partial_off = 2048;  // header: barrier, counters (128 B apart), epoch, launch count
  pl.ws_pub_off = pl.ws_partial_off + align_up(sizeof(double2) * np, 256);
  pl.ws_carry_off = pl.ws_pub_off + align_up(sizeof(double2) * np * 2, 256);
  pl.ws_coef_off = pl.ws_carry_off + align_up(sizeof(double) * nc, 256);
  const size_t ns = std::max<size_t>(pl.segs.size(), 1);
  pl.ws_apart_off = pl.ws_coef_off + align_up(sizeof(double) * (size_t)pl.nlayers, 256);
  pl.ws_segcnt_off = pl.ws_apart_off + align_up(sizeof(double2) * nc, 256);
  pl.ws_segready_off = pl.ws_segcnt_off + align_up(sizeof(unsigned) * ns, 256);
  pl.ws_segpart_off = pl.ws_segready_off + align_up(sizeof(unsigned) * ns, 256);
  pl.ws_bytes = pl.ws_segpart_off + align_up(sizeof(double2) * ns, 256);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int launch(const Plan& pl, int mode, bool carry, StepArgs& a, void* d_ws, cudaStream_t st) {
  a.p = pl.dev;
  auto ws = static_cast<unsigned char*>(d_ws);
  a.bar = reinterpret_cast<unsigned long long*>(ws);
  a.ctr = reinterpret_cast<unsigned long long*>(ws + 8);
  a.nv_epoch = reinterpret_cast<unsigned*>(ws + 16);
  a.partial = reinterpret_cast<double2*>(ws + pl.ws_partial_off);
  a.pub = reinterpret_cast<double2*>(ws + pl.ws_pub_off);
  a.launch_ctr = reinterpret_cast<unsigned*>(ws + 20);
  a.ccarry = reinterpret_cast<double*>(ws + pl.ws_carry_off);
  a.coef_g = reinterpret_cast<double*>(ws + pl.ws_coef_off);
  a.peer_launch = reinterpret_cast<unsigned*>(ws + 1812);
  a.shared_ready = reinterpret_cast<unsigned*>(ws + 1816);
  a.apart = reinterpret_cast<double2*>(ws + pl.ws_apart_off);
  a.seg_cnt = reinterpret_cast<unsigned*>(ws + pl.ws_segcnt_off);
  a.seg_ready = reinterpret_cast<unsigned*>(ws + pl.ws_segready_off);
  a.seg_part = reinterpret_cast<double2*>(ws + pl.ws_segpart_off);
  a.ctr_a = reinterpret_cast<unsigned long long*>(ws + 1536);
  a.ctr_b = reinterpret_cast<unsigned long long*>(ws + 1664);
  a.shared_done = reinterpret_cast<unsigned*>(ws + 1792);
  a.stream_launch = reinterpret_cast<unsigned*>(ws + 1920);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = pl.smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = (mode == kUpdate) ? 0 : 1;  // kFull / kNorms / kPeer hold grid barriers
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {&a};
  void* k = pick_kernel(mode, carry);
  const int rc = ensure_smem_attr(k, pl.smem_bytes);
  if (rc) return rc;
  cudaError_t e = cudaLaunchKernelExC(&cfg, k, args);
  return cuda_code(e);
}

// fp64 <-> fp32 conversion of the flat buffers for host-resident parameter
// sets (lars_host_copy_in / _out): a grid-stride stream, 2 elements per
// thread per iteration (16-byte fp64 loads / stores).
__global__ void __launch_bounds__(256) f64_to_f32_kernel(const double2* __restrict__ src,
                                                        float2* __restrict__ dst, int64_t n2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = __ldcs(src + i);
    __stcs(dst + i, make_float2((float)v.x, (float)v.y));
  }
}
__global__ void __launch_bounds__(256) f32_to_f64_kernel(const float2* __restrict__ src,
                                                        double2* __restrict__ dst, int64_t n2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float2 v = __ldcs(src + i);
    __stcs(dst + i, make_double2((double)v.x, (double)v.y));
  }
}

int convert_grid(int64_t n2) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n2 + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

extern "C" {

int lars_abi_version(void) { return LARS_ABI_VERSION; }

#ifdef LARS_TRACE
__attribute__((visibility("default"))) int lars_debug_trace(unsigned long long* out, int n) {
  if (n > kTraceWarps * 8) n = kTraceWarps * 8;
  return cuda_code(cudaMemcpyFromSymbol(out, g_trace, sizeof(unsigned long long) * n));
}
#endif

const char* lars_strerror(int code) {
  switch (code) {
    case LARS_OK: return "ok";
    case LARS_ERR_INVALID: return "invalid argument";
    case LARS_ERR_ALIGNMENT: return "misaligned segment or buffer (need multiples of 4 elements, 16-byte pointers)";
    case LARS_ERR_LAYOUT: return "segments must be sorted by offset and non-overlapping";
    case LARS_ERR_TOO_MANY_PIECES: return "too many segments per CTA for shared memory";
    case LARS_ERR_NO_DEVICE: return "no CUDA device";
    case LARS_ERR_HOST_ONLY_PLAN: return "plan was built with LARS_PLAN_HOST_ONLY";
    case LARS_ERR_HOST_MEMORY: return "host memory range could not be pinned (already registered or not pageable memory)";
    default: break;
  }
  if (code >= LARS_ERR_CUDA_BASE) return cudaGetErrorString((cudaError_t)(code - LARS_ERR_CUDA_BASE));
  return "unknown error";
}

int lars_plan_create(const lars_segment_t* segs, int32_t nseg, int32_t nlayers, int32_t grid,
                     int32_t flags, void** out) {
  if (!out || nseg < 0 || nlayers <= 0 || (nseg > 0 && !segs)) return LARS_ERR_INVALID;
  *out = nullptr;
  Plan* pl = new (std::nothrow) Plan();
  if (!pl) return LARS_ERR_INVALID;
  pl->nlayers = nlayers;
  pl->host_only = (flags & LARS_PLAN_HOST_ONLY) != 0;
  pl->layer_flags.assign(nlayers, 0);
  int64_t prev_end = 0;
  int64_t nb = 0;
  for (int i = 0; i < nseg; ++i) {
    const lars_segment_t& s = segs[i];
    if (s.layer < 0 || s.layer >= nlayers || s.offset < 0 || s.length < 0) { delete pl; return LARS_ERR_INVALID; }
    if ((s.offset & 3) || (s.length & 3)) { delete pl; return LARS_ERR_ALIGNMENT; }
    pl->layer_flags[s.layer] |= s.flags;
    if (s.length == 0) continue;
    if (s.offset < prev_end) { delete pl; return LARS_ERR_LAYOUT; }
    prev_end = s.offset + s.length;
    DevSeg d;
    d.vec_off = s.offset / 4;
    d.vec_len = s.length / 4;
    d.bstart = nb;
    nb += (d.vec_len + kBatchVec - 1) / kBatchVec;
    d.bend = nb;
    d.layer = s.layer;
    d.flags = s.flags;
    pl->segs.push_back(d);
    pl->elements += s.length;
  }
  pl->nbatches = nb;
  // L2 residency of g between the phases: by default
  // every batch is kept (evict_last); LARS_KEEP_MB / LARS_POL_B override it
  // for tuning runs
  pl->keep_nb = nb;
  if (const char* env = getenv("LARS_KEEP_MB")) {
    const double mb = atof(env);
    if (mb >= 0) pl->keep_nb = std::min<int64_t>(nb, (int64_t)(mb * 1048576.0 / (kBatchVec * 16)));
  }
  if (const char* env = getenv("LARS_POL_B")) pl->pol_b = atoi(env) ? 1 : 0;
  if (const char* env = getenv("LARS_CHUNK_BATCHES")) {
    const int v = atoi(env);
    if (v >= 1 && v <= 16) {
      pl->chunk_batches = v;
      pl->chunk_override = true;
    }
  }
  if (pl->segs.empty()) {  // keep one dummy so device lookups stay in bounds
    DevSeg d{};
    d.layer = 0;
    pl->segs.push_back(d);
  }
  int rc;
  if (pl->host_only) {
    if (grid <= 0) { delete pl; return LARS_ERR_INVALID; }
    rc = build_partition(*pl, grid);
    if (rc) { delete pl; return rc; }
    layout_workspace(*pl);
    *out = pl;
    return LARS_OK;
  }
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) { delete pl; return e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? LARS_ERR_NO_DEVICE : cuda_code(e); }
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) { delete pl; return cuda_code(e); }
  int want = grid > 0 ? grid : sms * kMinBlocksPerSM;
  for (int attempt = 0; attempt < 4; ++attempt) {
    rc = build_partition(*pl, want);
    if (rc) { delete pl; return rc; }
    int per_sm = 0;
    rc = occupancy(pl->smem_bytes, &per_sm);
    if (rc) { delete pl; return rc; }
    if (per_sm <= 0) { delete pl; return LARS_ERR_TOO_MANY_PIECES; }
    if (want <= per_sm * sms) break;
    if (grid > 0) { delete pl; return LARS_ERR_INVALID; }  // caller asked for too many
    want = per_sm * sms;
  }
  layout_workspace(*pl);
  rc = upload(*pl);
  if (rc) { if (pl->dmem) cudaFree(pl->dmem); delete pl; return rc; }
  *out = pl;
  return LARS_OK;
}

int lars_plan_info(const void* plan, lars_plan_info_t* info) {
  if (!plan || !info) return LARS_ERR_INVALID;
  const Plan* pl = static_cast<const Plan*>(plan);
  info->grid = pl->grid;
  info->threads = kThreads;
  info->nseg = pl->elements ? (int32_t)pl->segs.size() : 0;
  info->nlayers = pl->nlayers;
  info->npieces = (int64_t)pl->piece_seg.size();
  info->nbatches = pl->nbatches;
  info->elements = pl->elements;
  info->max_pieces_cta = pl->max_pieces_cta;
  info->max_slots_cta = pl->max_slots_cta;
  info->smem_bytes = pl->smem_bytes;
  info->reserved = 0;
  info->workspace_bytes = (int64_t)pl->ws_bytes;
  return LARS_OK;
}

int lars_plan_partition(const void* plan, int64_t* warp_b0, int32_t* piece_seg, int32_t* piece_cta) {
  if (!plan) return LARS_ERR_INVALID;
  const Plan* pl = static_cast<const Plan*>(plan);
  if (warp_b0) std::memcpy(warp_b0, pl->warp_b0.data(), sizeof(int64_t) * pl->warp_b0.size());
  if (piece_seg) std::memcpy(piece_seg, pl->piece_seg.data(), sizeof(int32_t) * pl->piece_seg.size());
  if (piece_cta) std::memcpy(piece_cta, pl->piece_cta.data(), sizeof(int32_t) * pl->piece_cta.size());
  return LARS_OK;
}

void lars_plan_destroy(void* plan) {
  if (!plan) return;
  Plan* pl = static_cast<Plan*>(plan);
  if (pl->dmem) cudaFree(pl->dmem);
  delete pl;
}

int lars_workspace_init(const void* plan, void* d_ws, void* stream) {
  if (!plan || !d_ws) return LARS_ERR_INVALID;
  const Plan* pl = static_cast<const Plan*>(plan);
  if (pl->host_only) return LARS_ERR_HOST_ONLY_PLAN;
  auto st = static_cast<cudaStream_t>(stream);
  auto ws = static_cast<unsigned char*>(d_ws);
  cudaError_t e = cudaMemsetAsync(ws, 0, pl->ws_bytes, st);
  if (e == cudaSuccess)  // published-piece slots start armed (all-ones: kSentinel64)
    e = cudaMemsetAsync(ws + pl->ws_pub_off, 0xff, pl->ws_carry_off - pl->ws_pub_off, st);
  return cuda_code(e);
}

static int check_step_args(const Plan* pl, const float* w, const float* g, const float* m,
                           const lars_hparams_t* hp, const void* d_ws, const void* d_info) {
  if (!pl || !hp || !d_ws || !d_info) return LARS_ERR_INVALID;
  if (pl->host_only) return LARS_ERR_HOST_ONLY_PLAN;
  if (pl->elements > 0 && (!w || !g)) return LARS_ERR_INVALID;
  if (!aligned16(w) || !aligned16(g) || !aligned16(m) || !aligned16(d_ws)) return LARS_ERR_ALIGNMENT;
  return LARS_OK;
}

int lars_step(const void* plan, float* w, const float* g, float* m, const lars_hparams_t* hp,
              int64_t* d_iter, double* d_sumsq, double* d_lambda, lars_step_info_t* d_info,
              void* d_ws, void* stream) {
  const Plan* pl = static_cast<const Plan*>(plan);
  int rc = check_step_args(pl, w, g, m, hp, d_ws, d_info);
  if (rc) return rc;
  if (!d_iter || (pl->elements > 0 && !m)) return LARS_ERR_INVALID;
  StepArgs a{};
  a.w = w; a.g = g; a.m = m; a.hp = *hp; a.d_iter = d_iter;
  a.d_sumsq = d_sumsq; a.d_sumsq_in = nullptr; a.d_lambda = d_lambda; a.d_info = d_info;
  return launch(*pl, kFull, (hp->flags & LARS_STEP_USE_WCARRY) != 0, a, d_ws,
                static_cast<cudaStream_t>(stream));
}

int lars_partial_norms(const void* plan, const float* w, const float* g, const lars_hparams_t* hp,
                       int64_t* d_iter, double* d_sumsq, lars_step_info_t* d_info, void* d_ws,
                       void* stream) {
  const Plan* pl = static_cast<const Plan*>(plan);
  int rc = check_step_args(pl, w, g, nullptr, hp, d_ws, d_info);
  if (rc) return rc;
  if (!d_iter || !d_sumsq) return LARS_ERR_INVALID;
  StepArgs a{};
  a.w = const_cast<float*>(w); a.g = g; a.m = nullptr; a.hp = *hp; a.d_iter = d_iter;
  a.d_sumsq = d_sumsq; a.d_sumsq_in = nullptr; a.d_lambda = nullptr; a.d_info = d_info;
  return launch(*pl, kNorms, (hp->flags & LARS_STEP_USE_WCARRY) != 0, a, d_ws,
                static_cast<cudaStream_t>(stream));
}

static int step_peer(int mode, const void* plan, const lars_peer_t* pr, const lars_hparams_t* hp,
                   int64_t* d_iter, double* d_sumsq, double* d_lambda, lars_step_info_t* d_info,
                   void* d_ws, void* stream) {
  const Plan* pl = static_cast<const Plan*>(plan);
  if (!pr || pr->world < 1 || pr->world > LARS_MAX_RANKS || pr->rank < 0 || pr->rank >= pr->world)
    return LARS_ERR_INVALID;
  float* w_local = pr->w_peer[pr->rank];
  int rc = check_step_args(pl, w_local, pr->g_shard, pr->m, hp, d_ws, d_info);
  if (rc) return rc;
  if (!d_iter || (pl->elements > 0 && !pr->m)) return LARS_ERR_INVALID;
  StepArgs a{};
  for (int q = 0; q < pr->world; ++q) {
    if (!pr->w_peer[q] || !pr->g_peer[q] || !pr->x_peer[q] || !pr->f_peer[q]) return LARS_ERR_INVALID;
    if (!aligned16(pr->w_peer[q]) || !aligned16(pr->g_peer[q]) || !aligned16(pr->x_peer[q]))
      return LARS_ERR_ALIGNMENT;
    a.w_peer[q] = pr->w_peer[q];
    a.g_peer[q] = pr->g_peer[q];
    a.x_peer[q] = pr->x_peer[q];
    a.f_peer[q] = pr->f_peer[q];
  }
  a.w = w_local; a.g = pr->g_shard; a.m = pr->m; a.hp = *hp; a.d_iter = d_iter;
  a.d_sumsq = d_sumsq; a.d_sumsq_in = nullptr; a.d_lambda = d_lambda; a.d_info = d_info;
  a.rank = pr->rank; a.world = pr->world;
  return launch(*pl, mode, (hp->flags & LARS_STEP_USE_WCARRY) != 0, a, d_ws,
                static_cast<cudaStream_t>(stream));
}

int lars_step_peer(const void* plan, const lars_peer_t* pr, const lars_hparams_t* hp,
                   int64_t* d_iter, double* d_sumsq, double* d_lambda, lars_step_info_t* d_info,
                   void* d_ws, void* stream) {
  return step_peer(kPeer, plan, pr, hp, d_iter, d_sumsq, d_lambda, d_info, d_ws, stream);
}

int lars_step_peer_stream(const void* plan, const lars_peer_t* pr, const lars_hparams_t* hp,
                          int64_t* d_iter, double* d_sumsq, double* d_lambda,
                          lars_step_info_t* d_info, void* d_ws, void* stream) {
  return step_peer(kPeerStream, plan, pr, hp, d_iter, d_sumsq, d_lambda, d_info, d_ws, stream);
}

int lars_peer_barrier(const lars_peer_t* pr, void* d_ws, lars_step_info_t* d_info, void* stream) {
  if (!pr || !d_ws || !d_info || pr->world < 1 || pr->world > LARS_MAX_RANKS || pr->rank < 0 ||
      pr->rank >= pr->world)
    return LARS_ERR_INVALID;
  StepArgs a{};
  for (int q = 0; q < pr->world; ++q) {
    if (!pr->f_peer[q]) return LARS_ERR_INVALID;
    a.f_peer[q] = pr->f_peer[q];
  }
  a.rank = pr->rank;
  a.world = pr->world;
  a.d_info = d_info;
  a.nv_epoch = reinterpret_cast<unsigned*>(static_cast<unsigned char*>(d_ws) + 16);
  rank_barrier_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return cuda_code(cudaGetLastError());
}

int lars_host_register(void* ptr, int64_t bytes) {
  if (!ptr || bytes <= 0) return LARS_ERR_INVALID;
  cudaError_t e = cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterDefault);
  if (e == cudaSuccess) return LARS_OK;
  cudaGetLastError();  // not sticky: clear it so it does not surface later
  if (e == cudaErrorHostMemoryAlreadyRegistered || e == cudaErrorInvalidValue ||
      e == cudaErrorNotSupported)
    return LARS_ERR_HOST_MEMORY;
  return cuda_code(e);
}

int lars_host_unregister(void* ptr) {
  if (!ptr) return LARS_ERR_INVALID;
  cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) cudaGetLastError();
  return cuda_code(e);
}

int lars_host_copy_in(const lars_host_span_t* spans, int32_t nspans, double* d_stage, float* d_dst,
                      int64_t flat_elems, void* stream) {
  if (nspans < 0 || (nspans > 0 && !spans) || !d_stage || !d_dst || flat_elems < 0 || (flat_elems & 1))
    return LARS_ERR_INVALID;
  if (!aligned16(d_stage) || !aligned16(d_dst)) return LARS_ERR_ALIGNMENT;
  auto st = static_cast<cudaStream_t>(stream);
  for (int i = 0; i < nspans; ++i) {
    const lars_host_span_t& s = spans[i];
    if (!s.host || s.offset < 0 || s.numel < 0 || s.offset + s.numel > flat_elems) return LARS_ERR_INVALID;
    if (s.numel == 0) continue;
    cudaError_t e = cudaMemcpyAsync(d_stage + s.offset, s.host, sizeof(double) * (size_t)s.numel,
                                    cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_code(e);
  }
  if (flat_elems == 0) return LARS_OK;
  const int64_t n2 = flat_elems / 2;
  f64_to_f32_kernel<<<convert_grid(n2), 256, 0, st>>>(reinterpret_cast<const double2*>(d_stage),
                                                     reinterpret_cast<float2*>(d_dst), n2);
  return cuda_code(cudaGetLastError());
}

int lars_host_copy_out(const float* d_src, double* d_stage, int64_t flat_elems,
                       const lars_host_span_t* spans, int32_t nspans, void* stream) {
  if (nspans < 0 || (nspans > 0 && !spans) || !d_stage || !d_src || flat_elems < 0 || (flat_elems & 1))
    return LARS_ERR_INVALID;
  if (!aligned16(d_stage) || !aligned16(d_src)) return LARS_ERR_ALIGNMENT;
  auto st = static_cast<cudaStream_t>(stream);
  if (flat_elems > 0) {
    const int64_t n2 = flat_elems / 2;
    f32_to_f64_kernel<<<convert_grid(n2), 256, 0, st>>>(reinterpret_cast<const float2*>(d_src),
                                                       reinterpret_cast<double2*>(d_stage), n2);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_code(e);
  }
  for (int i = 0; i < nspans; ++i) {
    const lars_host_span_t& s = spans[i];
    if (!s.host || s.offset < 0 || s.numel < 0 || s.offset + s.numel > flat_elems) return LARS_ERR_INVALID;
    if (s.numel == 0) continue;
    cudaError_t e = cudaMemcpyAsync(s.host, d_stage + s.offset, sizeof(double) * (size_t)s.numel,
                                    cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_code(e);
  }
  return LARS_OK;
}

int lars_update(const void* plan, float* w, const float* g, float* m, const lars_hparams_t* hp,
                const double* d_sumsq, double* d_lambda, lars_step_info_t* d_info, void* d_ws,
                void* stream) {
  const Plan* pl = static_cast<const Plan*>(plan);
  int rc = check_step_args(pl, w, g, m, hp, d_ws, d_info);
  if (rc) return rc;
  if (!d_sumsq || (pl->elements > 0 && !m)) return LARS_ERR_INVALID;
  StepArgs a{};
  a.w = w; a.g = g; a.m = m; a.hp = *hp; a.d_iter = nullptr;
  a.d_sumsq = nullptr; a.d_sumsq_in = d_sumsq; a.d_lambda = d_lambda; a.d_info = d_info;
  return launch(*pl, kUpdate, false, a, d_ws, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
