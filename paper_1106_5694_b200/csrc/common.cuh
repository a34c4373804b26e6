// common.cuh -- shared device types for the B200 DGS path (sm_100a only).
//
// Storage: the benefit matrix is held twice in HBM, row-major A[i*ld + j] and
// its transpose AT[j*ld + i] (the reference's SolverState::a / a_cols,
// proj/src/solver_state.hpp:36-37,67-76), in the narrowest element type that
// represents every fp64 entry exactly (int16 / int32 / fp32 / fp64).  All delta
// arithmetic reproduces the reference's fp64 add/sub chain bit for bit:
// integer storage computes in exact int32 (every intermediate is an integer
// below 2^31, so fp64 would be exact too), float storage widens to fp64 and
// uses round-to-nearest add/sub with no contraction (kernels_scalar.cpp:16-17).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "paper_1106_5694_b200 kernels target sm_100a only"
#endif

namespace lsapgpu {

enum Storage : int { kI16 = 0, kI32 = 1, kF32 = 2, kF64 = 3 };

template <class E>
struct Traits;
template <>
struct Traits<int16_t> {
  using Acc = int32_t;  // exact
  static constexpr Storage kStorage = kI16;
  static constexpr bool kInt = true;
};
template <>
struct Traits<int32_t> {
  using Acc = int32_t;  // exact because |a| < 2^29 is enforced by the classifier
  static constexpr Storage kStorage = kI32;
  static constexpr bool kInt = true;
};
template <>
struct Traits<float> {
  using Acc = double;
  static constexpr Storage kStorage = kF32;
  static constexpr bool kInt = false;
};
template <>
struct Traits<double> {
  using Acc = double;
  static constexpr Storage kStorage = kF64;
  static constexpr bool kInt = false;
};

// Round-to-nearest fp64 add/sub, never contracted (matches -mno-fma reference).
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// The four-term exchange delta in the reference's operation order:
// (p - s) + (q - c).  Integer storage: exact int32.
__device__ __forceinline__ int32_t delta4(int32_t p, int32_t s, int32_t q, int32_t c) {
  return (p - s) + (q - c);
}
__device__ __forceinline__ double delta4(double p, double s, double q, double c) {
  return dadd(dsub(p, s), dsub(q, c));
}

template <class E>
__device__ __forceinline__ typename Traits<E>::Acc widen(E v) {
  return static_cast<typename Traits<E>::Acc>(v);
}

// Work-list item: agent index in the low 30 bits, bit 30 = also write the
// job record of tau[agent], bit 31 = write the agent record.
constexpr uint32_t kItemAgent = 0x80000000u;
constexpr uint32_t kItemJob = 0x40000000u;
constexpr uint32_t kItemMask = 0x3FFFFFFFu;

// LFMM edge states
constexpr uint8_t kEdgeUndecided = 0, kEdgeAccepted = 1, kEdgeRejected = 2, kEdgeNone = 3;

struct LogEntry {  // one committed 2-exchange (AppliedExchange, parallel.hpp:49-55)
  int32_t iter;    // inner iteration (global within the solve)
  int32_t slot;    // record slot: agent i, or n + job j; batch order = ascending slot
  double delta;    // the recomputed improvement that was committed
};

// Device control block (one per context, lives in device memory).
struct Ctrl {
  int32_t parity;           // which edge list the next commit consumes
  int32_t iter;             // inner iterations so far in this solve (global stamp)
  uint32_t round;           // LFMM round counter (key epoch)
  int32_t work_count;       // items in the current work list
  int32_t own_count;        // multi-GPU: items of this rank's share
  int32_t edge_count[2];    // ping-pong edge-list sizes
  int32_t inner_done;       // set when a commit found no active record
  int32_t expired;          // deadline hit
  int32_t drain;            // delta log needs draining by the host
  int32_t error;            // nonzero: overlap assertion fired (parallel.cpp:296-302)
  int64_t log_count;        // entries in the delta log
  int64_t switches;         // committed exchanges (this solve)
  int64_t pair_items;       // scanned pair items (this solve)
  int64_t agent_scans, job_scans;
  int64_t lfmm_rounds;      // total LFMM rounds (instrumentation)
  int64_t inner_iterations; // batches (this solve)
  uint64_t deadline_gt;     // %globaltimer deadline, 0 = none
  int32_t tl_count;         // device timeline entries (instrumentation)
  // conflict-check -> apply hand-off of the split commit (commit_single.cuh,
  // commit_apply): committed / queued-conflicted proposal lists of one batch
  int32_t k2_parity, k2_nlog, k2_nconf, k2_iter;
  int64_t k2_log_base;
  // device ordering of the delta log (log_order.cu): nonzero if the log was
  // not iteration-grouped with distinct slots per iteration; entries placed
  uint32_t order_bad, order_total;
  uint32_t push_done;  // CTAs finished with the peer push of the current round
  uint32_t pad2_;
  uint64_t p2p_epoch;  // peer transport: rounds pushed (flags carry it; graph-capturable)
  // quantized-filter scan (instrumentation): candidates verified exactly,
  // items that overflowed their queue (whole-item exact fallback)
  int64_t filter_kept, filter_overflows;
  // filter scan self-check (DevState::filter_check): mismatches of the
  // filtered records against an unfiltered scan of the same item, first one
  int32_t fchk_mismatch, fchk_item, fchk_cnt, fchk_side;
  int32_t fchk_want_k, fchk_got_k;
  int32_t fchk_p, fchk_aux_ok, fchk_u, fchk_t0, fchk_tmax, fchk_pad;
  double fchk_want_d, fchk_got_d;
};

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One active record as a proposal for the conflict check, written by the
// producer of the record (the pair scan, the multi-GPU record merge, the
// step-API table import) against the state the record was computed on.  The
// exchange moves agent a to job j_new and the displaced agent d to job j_old:
//   agent record of i (slot i, partner job k):   a = i, d = sigma[k],
//                                                j_new = k, j_old = tau[i]
//   job record of j (slot n + j, partner k):     a = k, d = sigma[j],
//                                                j_new = j, j_old = tau[k]
// delta is the record's value; acur_a = A[a][j_new] and acur_d = A[d][j_old]
// are the two entries the apply writes (exact in fp64 for every storage).
struct Prop {
  int32_t slot;
  int32_t a, d;
  int32_t j_new, j_old;
  int32_t pad;
  double delta;
  double acur_a, acur_d;
};
static_assert(sizeof(Prop) == 48, "proposal layout");

// The compact {slot, proposer, partner, job} view the general commit path
// uses: proposer = the record's owner (i, or the holder of j), partner = the
// record's partner (job k, or agent k), job = the owner's current job.
__device__ __forceinline__ int4 prop_key(const Prop& p, int32_t n) {
  return p.slot < n ? make_int4(p.slot, p.a, p.j_new, p.j_old) : make_int4(p.slot, p.d, p.a, p.j_new);
}

// A[i][j] widened to fp64 for any storage type (exact), read from the
// TRANSPOSE AT[j][i]: every rank holds all of AT, while A may be held as a
// row block only (row-block placement)
__device__ __forceinline__ double mat_at(const void* AT, int storage, int64_t ld, int32_t i, int32_t j) {
  const int64_t k = static_cast<int64_t>(j) * ld + i;
  const void* M = AT;
  switch (storage) {
    case kI16: return static_cast<double>(static_cast<const int16_t*>(M)[k]);
    case kI32: return static_cast<double>(static_cast<const int32_t*>(M)[k]);
    case kF32: return static_cast<double>(static_cast<const float*>(M)[k]);
    default: return static_cast<const double*>(M)[k];
  }
}

// Proposal of agent i's record (partner job k) / job j's record (partner
// agent k) on the current state; used by producers that do not hold the rows.
__device__ __forceinline__ Prop agent_prop(const int32_t* sigma, const int32_t* tau, const void* A, int storage,
                                           int64_t ld, int32_t i, int32_t k, double delta) {
  const int32_t d = sigma[k], jo = tau[i];
  if (A == nullptr) return Prop{i, i, d, k, jo, 0, delta, 0.0, 0.0};  // conflict check only
  return Prop{i, i, d, k, jo, 0, delta, mat_at(A, storage, ld, i, k), mat_at(A, storage, ld, d, jo)};
}
__device__ __forceinline__ Prop job_prop(const int32_t* sigma, const int32_t* tau, const void* A, int storage,
                                         int64_t ld, int32_t n, int32_t j, int32_t k, double delta) {
  const int32_t h = sigma[j], jo = tau[k];
  if (A == nullptr) return Prop{n + j, k, h, j, jo, 0, delta, 0.0, 0.0};  // conflict check only
  return Prop{n + j, k, h, j, jo, 0, delta, mat_at(A, storage, ld, k, j), mat_at(A, storage, ld, h, jo)};
}

// Proposal fields a scan defers to the end of its launch (pad != 0) so the
// dependent global loads do not sit on a stage's critical path: pad 1 = the
// agent record's displaced holder and its entry, pad 2 = every entry-derived
// field (the streaming kernel, whose AT rows are not on chip).
__device__ __forceinline__ Prop finish_prop(Prop p, const int32_t* sigma, const int32_t* tau, const void* A,
                                            int storage, int64_t ld, int32_t n) {
  if (p.pad == 0) return p;
  if (p.slot < n) {  // agent i = a -> job k = j_new; displaced sigma[k] -> j_old = tau[i]
    p.d = sigma[p.j_new];
    p.acur_d = mat_at(A, storage, ld, p.d, p.j_old);
    if (p.pad == 2) p.acur_a = mat_at(A, storage, ld, p.a, p.j_new);
  } else {  // agent k = a -> job j0 = j_new; holder i = d -> tau[k]
    p.j_old = tau[p.a];
    p.acur_a = mat_at(A, storage, ld, p.a, p.j_new);
    p.acur_d = mat_at(A, storage, ld, p.d, p.j_old);
  }
  p.pad = 0;
  return p;
}

// Programmatic dependent launch: a kernel launched with programmatic stream
// serialization may start while its predecessor drains; it must wait for the
// predecessor's completion (and memory) before touching state the
// predecessor writes.  Both are no-ops for a normally launched kernel.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// timeline kinds
constexpr unsigned kTlScanFull = 1, kTlScan = 2, kTlCommit = 3, kTlCommitEnd = 4;
__device__ __forceinline__ void tl_mark(Ctrl* c, unsigned long long* tl, int cap, unsigned kind) {
  if (tl == nullptr) return;
  const int i = atomicAdd(&c->tl_count, 1);
  if (i < cap) tl[i] = (globaltimer() << 4) | kind;
}

// Launch helper: cudaLaunchKernelEx with programmatic stream serialization
// when enabled (pdl != 0), so consecutive kernels of the inner loop overlap
// one's tail with the next one's launch.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int pdl,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

}  // namespace lsapgpu
