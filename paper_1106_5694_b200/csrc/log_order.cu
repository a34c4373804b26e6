// log_order.cu -- the delta log in the reference's batch order on the device.
//
// The reference applies a batch's accepted exchanges in ascending slot order
// (agents, then jobs; parallel.cpp:306-310), so the objective trace and, for
// float storage, the rounding of the running objective depend on that order.
// The commit kernels append a batch's entries as one contiguous range of the
// log (one reservation per batch), in whatever order their CTAs got there.
// Within one batch every slot appears at most once (one record per agent and
// per job), so a batch's order is a rank in a slot bitmap: one CTA per batch
// sets a bit per entry in shared memory, prefix-counts the words and writes
// each entry to (batch start + number of set bits below its slot).  The host
// then replays the ordered log straight from its pinned copy instead of
// sorting 10^4-10^5 entries per pass.
//
// Anything that breaks the premises (batches not contiguous and ascending,
// a slot twice in a batch, a slot out of range) sets Ctrl::order_bad, and the
// host falls back to ordering the raw log itself; Ctrl::order_total (entries
// placed) must equal the log count as well.
#include "state.h"

namespace lsapgpu {
namespace {

constexpr int kOrderThreads = 1024;
constexpr int kOrderCtas = 148;
constexpr size_t kOrderSmemMax = 200 * 1024;

// first position in [0, cnt) whose iter >= it (the log's iters ascend);
// one warp, 32 probes per step
__device__ int64_t lower_bound_iter(const LogEntry* log, int64_t cnt, int32_t it) {
  const int lane = threadIdx.x & 31;
  int64_t a = 0, b = cnt;
  while (b - a > 32) {
    const int64_t len = b - a;
    const int64_t p = a + (len * lane) / 32;
    const unsigned below = __ballot_sync(0xffffffffu, __ldcg(&log[p].iter) < it);
    const int c = __popc(below);  // probes below `it` form a prefix of the lanes
    if (c == 0) return a;         // log[a] >= it
    const int64_t pc1 = a + (len * (c - 1)) / 32;
    const int64_t pc = c < 32 ? a + (len * c) / 32 : b;
    a = pc1 + 1;
    b = pc;
  }
  const bool below = a + lane < b && __ldcg(&log[a + lane].iter) < it;
  return a + __popc(__ballot_sync(0xffffffffu, below));
}

__global__ void __launch_bounds__(kOrderThreads) order_log_kernel(DevState st, int32_t words) {
  extern __shared__ uint32_t sm[];
  uint32_t* bits = sm;           // slot bitmap of the batch
  uint32_t* pre = sm + words;    // exclusive prefix popcounts of the words
  __shared__ int64_t seg[2];
  __shared__ uint32_t wsum[kOrderThreads / 32];
  Ctrl* C = st.ctrl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t cnt = __ldcg(&C->log_count);
  if (cnt <= 0) return;
  const LogEntry* log = st.log;
  const int32_t slots = 2 * st.n;
  // premise 1: iterations ascend along the log (every CTA checks a stride)
  bool bad = false;
  for (int64_t k = 1 + static_cast<int64_t>(blockIdx.x) * blockDim.x + tid; k < cnt;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bad |= __ldcg(&log[k].iter) < __ldcg(&log[k - 1].iter);
  if (__syncthreads_or(bad) && tid == 0) atomicOr(&C->order_bad, 1u);
  const int32_t lo = __ldcg(&log[0].iter), hi = __ldcg(&log[cnt - 1].iter);
  const int per = (words + kOrderThreads - 1) / kOrderThreads;  // words per thread in the scan
  uint32_t placed = 0;
  for (int64_t it = static_cast<int64_t>(lo) + blockIdx.x; it <= hi; it += gridDim.x) {
    if (warp < 2) {
      const int64_t x = lower_bound_iter(log, cnt, static_cast<int32_t>(it + warp));
      if (lane == 0) seg[warp] = x;
    }
    for (int w = tid; w < words; w += kOrderThreads) bits[w] = 0u;
    __syncthreads();
    const int64_t s0 = seg[0], s1 = seg[1];
    if (s1 <= s0) {
      __syncthreads();
      continue;
    }
    bool dup = false;
    for (int64_t e = s0 + tid; e < s1; e += kOrderThreads) {
      const int32_t s = __ldcg(&log[e].slot);
      if (s < 0 || s >= slots) {
        dup = true;
        continue;
      }
      const uint32_t m = 1u << (s & 31);
      dup |= (atomicOr(&bits[s >> 5], m) & m) != 0u;
    }
    if (__syncthreads_or(dup) && tid == 0) atomicOr(&C->order_bad, 2u);
    // exclusive prefix of popcounts: thread t owns words [t*per, t*per+per)
    uint32_t mine = 0;
    for (int q = 0; q < per; ++q) {
      const int w = tid * per + q;
      if (w < words) mine += __popc(bits[w]);
    }
    uint32_t incl = mine;
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      uint32_t v = wsum[lane];
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, off);
        if (lane >= off) v += y;
      }
      wsum[lane] = v;  // inclusive over warps
    }
    __syncthreads();
    uint32_t run = incl - mine + (warp ? wsum[warp - 1] : 0u);
    for (int q = 0; q < per; ++q) {
      const int w = tid * per + q;
      if (w < words) {
        pre[w] = run;
        run += __popc(bits[w]);
      }
    }
    __syncthreads();
    for (int64_t e = s0 + tid; e < s1; e += kOrderThreads) {
      const LogEntry L = st.log[e];
      if (L.slot < 0 || L.slot >= slots) continue;
      const uint32_t r = pre[L.slot >> 5] + __popc(bits[L.slot >> 5] & ((1u << (L.slot & 31)) - 1u));
      st.log_sorted[s0 + r] = L;
    }
    placed += static_cast<uint32_t>(s1 - s0);
    __syncthreads();  // bitmap reused by the next batch
  }
  if (tid == 0 && placed) atomicAdd(&C->order_total, placed);
}

size_t order_smem(int32_t n) {
  const size_t words = (2 * static_cast<size_t>(n) + 31) / 32;
  return 2 * words * sizeof(uint32_t);
}

}  // namespace

bool order_log_fits(int32_t n) { return order_smem(n) <= kOrderSmemMax; }

cudaError_t launch_order_log(const DevState& d, cudaStream_t st) {
  const size_t smem = order_smem(d.n);
  if (smem > kOrderSmemMax || !d.log_sorted) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(&d.ctrl->order_bad, 0, 2 * sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  if (smem > 48 * 1024) {  // (per device: set on every launch that needs it)
    e = cudaFuncSetAttribute(order_log_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const int32_t words = static_cast<int32_t>((2 * static_cast<size_t>(d.n) + 31) / 32);
  order_log_kernel<<<kOrderCtas, kOrderThreads, smem, st>>>(d, words);
  return cudaGetLastError();
}

}  // namespace lsapgpu
