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
};

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

}  // namespace lsapgpu
