#pragma once
// scan_kernel.cuh -- the fused pair-scan kernel (streaming variant): the B200 replacement for the
// reference's exchange_scan ISA variants driven by eval_agent / eval_job
// (proj/src/kernels_scalar.cpp:6-25, kernels_avx2.cpp:40-92,
// solver_state.hpp:78-104) over eval_all / reeval_lists (parallel.cpp:80-124).
//
// One work item is an agent i together with its job j0 = tau[i].  Agent i's
// scan and job j0's scan read exactly the same two rows, A[i,:] and AT[j0,:]
// (SURVEY 8(a) row 8), so one pass produces both records:
//   for every agent i', with t = tau[i'], x = AT[j0][i'], g = A[i][t],
//   c = acur[i'], s = acur[i]:
//     agent candidate (partner job t):   (g - s) + (x - c)
//     job   candidate (partner agent i'): (x - s) + (g - c)
// which are the reference's fp64 expressions in the reference's order.  The
// winner is the maximum with the smallest candidate index on ties, and it is
// active iff it exceeds eps (kernels_avx2.cpp:90).  The reference skips the
// candidate i' = i (k == skip); that candidate evaluates to exactly
// (s - s) + (s - s) = +0 on both sides, so it can never be an active winner
// (active requires > eps >= 0) and the kernel needs no skip test.
//
// Arithmetic.  Integer storage computes exactly in int32 and packs
// (delta, smallest-index) into one unsigned key so a running max is a single
// IMNMX per side: 32-bit keys (18-bit biased delta | 14-bit inverted index)
// when |a| <= 32767 and n <= 16384, 64-bit keys otherwise.  Float storage
// widens to fp64 and keeps (delta, index) with the explicit tie-break.
//
// Data movement per item: A[i,:] is staged into shared memory with TMA bulk
// copies (cp.async.bulk + mbarrier) because it is gathered at random positions
// t; AT[j0,:] is streamed with 16-byte no-L1-allocate loads, and tau / acur,
// which the M items of a CTA share, are read once per CTA.  CTAs are
// persistent and double buffer their stages (rows + item metadata), with the
// stream registers software-pipelined one iteration ahead.
// Algorithmic HBM bytes: 2 * n * sizeof(elem) per item.
#include <cfloat>
#include <climits>
#include <cstdlib>

#include "state.h"

namespace lsapgpu {
namespace scan_detail {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "LAB_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 16-byte streaming load that does not allocate in L1 (AT rows are read once).
__device__ __forceinline__ uint4 ld_stream16(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
// 16-byte load of data every CTA re-reads (tau, acur): cacheable.
__device__ __forceinline__ uint4 ld_keep16(const void* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

// element k (0 <= k < 16/sizeof(E)) of a 16-byte vector, widened
template <class E>
__device__ __forceinline__ typename Traits<E>::Acc vget(const uint4& v, int k) {
  const uint32_t w = (&v.x)[(k * sizeof(E)) / 4];
  if constexpr (sizeof(E) == 2) {
    return (k & 1) ? (static_cast<int32_t>(w) >> 16) : static_cast<int32_t>(static_cast<int16_t>(w & 0xFFFFu));
  } else if constexpr (sizeof(E) == 4) {
    if constexpr (Traits<E>::kInt)
      return static_cast<int32_t>(w);
    else
      return static_cast<double>(__uint_as_float(w));
  } else {
    const uint32_t hi = (&v.x)[(k * 8) / 4 + 1];
    return __hiloint2double(static_cast<int>(hi), static_cast<int>(w));
  }
}

enum KeyMode : int { kPacked32 = 0, kPacked64 = 1, kFloat = 2 };
constexpr int32_t kOff32 = 1 << 17;  // bias of the 18-bit delta field

// Per-side running best.  packed modes: a key whose unsigned max is the best
// (delta desc, index asc); float mode: explicit (delta, index) with tie-break.
template <int KM>
struct Track;

template <>
struct Track<kPacked32> {
  uint32_t k;
  __device__ __forceinline__ void init() { k = 0u; }
  __device__ __forceinline__ void merge(const Track& o) { k = max(k, o.k); }
  __device__ __forceinline__ bool valid() const { return k != 0u; }
  __device__ __forceinline__ double delta() const {
    return static_cast<double>(static_cast<int32_t>(k >> 14) - kOff32);
  }
  __device__ __forceinline__ int32_t index() const { return 16383 - static_cast<int32_t>(k & 16383u); }
  __device__ __forceinline__ void warp_reduce() { k = __reduce_max_sync(0xffffffffu, k); }
};

template <>
struct Track<kPacked64> {
  unsigned long long k;
  __device__ __forceinline__ void init() { k = 0ull; }
  __device__ __forceinline__ void merge(const Track& o) { k = o.k > k ? o.k : k; }
  __device__ __forceinline__ bool valid() const { return k != 0ull; }
  __device__ __forceinline__ double delta() const {
    return static_cast<double>(static_cast<int32_t>(static_cast<uint32_t>(k >> 32) ^ 0x80000000u));
  }
  __device__ __forceinline__ int32_t index() const {
    return static_cast<int32_t>(~static_cast<uint32_t>(k & 0xFFFFFFFFull));
  }
  __device__ __forceinline__ void warp_reduce() {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, k, off);
      k = o > k ? o : k;
    }
  }
  __device__ __forceinline__ void add(int32_t d, int32_t idx) {
    const unsigned long long key =
        (static_cast<unsigned long long>(static_cast<uint32_t>(d) ^ 0x80000000u) << 32) |
        static_cast<uint32_t>(~idx);
    k = key > k ? key : k;
  }
};

template <>
struct Track<kFloat> {
  double d;
  int32_t i;
  __device__ __forceinline__ void init() {
    d = -__longlong_as_double(0x7ff0000000000000ll);
    i = INT_MAX;
  }
  __device__ __forceinline__ void add(double v, int32_t idx) {
    // branch-free: predicates combined with bitwise ops (no short-circuit jumps)
    const bool take = (v > d) | ((v == d) & (idx < i));
    d = take ? v : d;
    i = take ? idx : i;
  }
  __device__ __forceinline__ void merge(const Track& o) { add(o.d, o.i); }
  __device__ __forceinline__ bool valid() const { return i != INT_MAX; }
  __device__ __forceinline__ double delta() const { return d; }
  __device__ __forceinline__ int32_t index() const { return i; }
  __device__ __forceinline__ void warp_reduce() {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      Track o;
      o.d = __shfl_xor_sync(0xffffffffu, d, off);
      o.i = __shfl_xor_sync(0xffffffffu, i, off);
      merge(o);
    }
  }
};

struct ItemInfo {
  int32_t agent;  // -1: no item in this slot (tail group)
  int32_t job;    // tau[agent]
  uint32_t flags;
};

// Stream registers of one vector step: tau (V ints), acur (V elems), x (M rows x V elems).
template <class E, int M>
struct StreamRegs {
  static constexpr int V = 16 / sizeof(E);
  int32_t t[V];
  uint4 c;
  uint4 x[M];
};

template <class E, int M>
__device__ __forceinline__ void load_step(StreamRegs<E, M>& r, const int32_t* __restrict__ tau,
                                          const E* __restrict__ acur, const E* const (&xrow)[M],
                                          int32_t i0) {
  constexpr int V = StreamRegs<E, M>::V;
#pragma unroll
  for (int q = 0; q < V / 4; ++q) {
    const uint4 a = ld_keep16(tau + i0 + 4 * q);
    r.t[4 * q] = a.x;
    r.t[4 * q + 1] = a.y;
    r.t[4 * q + 2] = a.z;
    r.t[4 * q + 3] = a.w;
  }
  if constexpr (V == 2) {
    const uint2 a = __ldg(reinterpret_cast<const uint2*>(tau + i0));
    r.t[0] = a.x;
    r.t[1] = a.y;
  }
  r.c = ld_keep16(acur + i0);
#pragma unroll
  for (int m = 0; m < M; ++m) r.x[m] = ld_stream16(xrow[m] + i0);
}

// Consume one vector step: V candidates for each of the M items.
template <class E, int M, int KM, bool kChunked>
__device__ __forceinline__ void compute_step(const StreamRegs<E, M>& r, int32_t i0, int nvalid,
                                             const E* __restrict__ rows, int64_t chunk, int64_t clo,
                                             const typename Traits<E>::Acc (&sv)[M], Track<KM> (&ta)[M],
                                             Track<KM> (&tj)[M]) {

  using Acc = typename Traits<E>::Acc;
  constexpr int V = StreamRegs<E, M>::V;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    if (v >= nvalid) break;
    const int32_t ip = i0 + v;
    const int32_t t = r.t[v];
    int64_t tl = t;
    if constexpr (kChunked) {
      tl = static_cast<int64_t>(t) - clo;
      if (tl < 0 || tl >= chunk) continue;
    }
    const Acc c = vget<E>(r.c, v);
    if constexpr (KM == kPacked32) {
      // key = (d + OFF) * 2^14 + (16383 - idx) computed mod 2^32, d = g + x - s - c
      const uint32_t base = static_cast<uint32_t>(kOff32 - c) * 16384u + 16383u;
      const uint32_t ka_c = base - static_cast<uint32_t>(t);
      const uint32_t kj_c = base - static_cast<uint32_t>(ip);
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int32_t g = rows[static_cast<int64_t>(m) * chunk + tl];
        const int32_t x = vget<E>(r.x[m], v);
        const uint32_t u = static_cast<uint32_t>(g + x - sv[m]) * 16384u;
        ta[m].k = max(ta[m].k, u + ka_c);
        tj[m].k = max(tj[m].k, u + kj_c);
      }
    } else if constexpr (KM == kPacked64) {
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int32_t g = rows[static_cast<int64_t>(m) * chunk + tl];
        const int32_t x = vget<E>(r.x[m], v);
        const int32_t d = (g - sv[m]) + (x - c);
        ta[m].add(d, t);
        tj[m].add(d, ip);
      }
    } else {
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const double g = static_cast<double>(rows[static_cast<int64_t>(m) * chunk + tl]);
        const double x = vget<E>(r.x[m], v);
        ta[m].add(delta4(g, sv[m], x, c), t);   // agent: (g - s) + (x - c)
        tj[m].add(delta4(x, sv[m], g, c), ip);  // job:   (x - s) + (g - c)
      }
    }
  }
}

// L2 prefetch of a byte range (bulk, no completion tracking)
__device__ __forceinline__ void pf_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// mbarrier arrive (count 1) by one thread
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Per-CTA emission buffer for active records (EdgeEntry), flushed with one
// global atomic per flush instead of one dependent atomic per record.
constexpr int kEdgeBuf = 256;
constexpr int kMaxBufs = 4;

template <class E, int M, int NT, int KM, bool kChunked, int D>
__global__ void __launch_bounds__(NT, 512 / NT) pair_scan_kernel(DevState st, int full, int passes,
                                                          int64_t chunk, int bufs, int max_segments,
                                                          int l2pf) {
  using Acc = typename Traits<E>::Acc;
  constexpr int V = StreamRegs<E, M>::V;
  constexpr int NW = NT / 32;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int32_t n = st.n;
  const int64_t ld = st.ld;
  const E* __restrict__ A = static_cast<const E*>(st.A) - static_cast<int64_t>(st.a_row0) * st.ld;  // own row block
  const E* __restrict__ AT = static_cast<const E*>(st.AT);
  const E* __restrict__ acur = static_cast<const E*>(st.acur);
  const int32_t* __restrict__ tau = st.tau;

  // smem: [bufs][M][chunk] staged rows | full[B], empty[B] mbarriers | red[B][NW][2M]
  const size_t chunk_bytes = static_cast<size_t>(chunk) * sizeof(E);
  E* stage_base = reinterpret_cast<E*>(smem_raw);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem_raw + bufs * M * chunk_bytes);
  uint64_t* empty_bar = full_bar + kMaxBufs;
  Track<KM>* red = reinterpret_cast<Track<KM>*>(full_bar + 2 * kMaxBufs);  // [B][NW][2M]
  __shared__ ItemInfo info_s[kMaxBufs][M];
  __shared__ int arrive_cnt[kMaxBufs];
  __shared__ int last_seg;
  __shared__ Prop ebuf[kEdgeBuf];
  __shared__ int ebuf_n;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  pdl_trigger();
  pdl_wait();
  if (blockIdx.x == 0 && tid == 0) tl_mark(st.ctrl, st.tl, st.tl_cap, full ? kTlScanFull : kTlScan);

  const int32_t count = full ? n : (st.use_own ? st.ctrl->own_count : st.ctrl->work_count);
  if (count <= 0) return;
  const uint32_t* __restrict__ items = st.use_own ? st.items_own : st.items;
  const int32_t groups = (count + M - 1) / M;
  // Segments: split an item group over several CTAs when the list is short,
  // picking the split that best fills whole waves of the persistent grid.
  int S = 1;
  {
    const int G = gridDim.x;
    float best_eff = -1.f;
    for (int s = 1; s <= max_segments; ++s) {
      const long units = static_cast<long>(groups) * s;
      const long waves = (units + G - 1) / G;
      const float eff = static_cast<float>(units) / static_cast<float>(waves * G);
      if (eff > best_eff + 0.04f) {
        best_eff = eff;
        S = s;
      }
      if (units >= 4L * G) break;
    }
  }
  const int64_t units = static_cast<int64_t>(groups) * S;
  int64_t u = blockIdx.x;
  if (u >= units) return;
  const int32_t seg_gran = 32 * V;
  const int32_t seglen = ((n + S - 1) / S + seg_gran - 1) / seg_gran * seg_gran;
  const int parity_out = st.ctrl->parity;
  // stages of this CTA: (unit, pass) pairs, unit = blockIdx.x + k * gridDim.x
  const int64_t my_units = (units - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int64_t stages = my_units * passes;

  auto item_of = [&](int32_t idx) -> ItemInfo {
    ItemInfo it;
    if (idx >= count) {
      it.agent = -1;
      it.job = -1;
      it.flags = 0;
      return it;
    }
    const uint32_t w = full ? (static_cast<uint32_t>(idx) | kItemAgent | kItemJob) : items[idx];
    it.agent = static_cast<int32_t>(w & kItemMask);
    it.job = tau[it.agent];
    it.flags = w & (kItemAgent | kItemJob);
    return it;
  };
  // Producer (warp 0): item metadata + TMA bulk copies of stage q into buffer q % bufs.
  auto produce = [&](int64_t q) {
    const int64_t uq = blockIdx.x + (q / passes) * gridDim.x;
    const int pq = static_cast<int>(q % passes);
    const int b = static_cast<int>(q % bufs);
    const int32_t group = static_cast<int32_t>(uq / S);
    if (lane < M) info_s[b][lane] = item_of(group * M + lane);
    __syncwarp();
    if (lane == 0) {
      const int64_t lo = static_cast<int64_t>(pq) * chunk;
      const int64_t len = (ld - lo) < chunk ? (ld - lo) : chunk;
      const uint32_t bytes = static_cast<uint32_t>(len * sizeof(E));
      uint32_t total = 0;
#pragma unroll
      for (int m = 0; m < M; ++m)
        if (info_s[b][m].agent >= 0) total += bytes;
      mbar_expect_tx(&full_bar[b], total);
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int32_t ag = info_s[b][m].agent;
        if (ag < 0) continue;
        const unsigned char* src = reinterpret_cast<const unsigned char*>(A + static_cast<int64_t>(ag) * ld + lo);
        unsigned char* dst = reinterpret_cast<unsigned char*>(stage_base) + (b * M + m) * chunk_bytes;
        for (uint32_t off = 0; off < bytes; off += 32768u) {
          const uint32_t sz = (bytes - off) < 32768u ? (bytes - off) : 32768u;
          bulk_g2s(dst + off, src + off, sz, &full_bar[b]);
        }
      }
      // single-buffered rows: pull the NEXT stage's rows into L2 while this
      // one is scanned, so its staging copy streams from L2, not HBM
      if (l2pf && q + 1 < stages) {
        const int64_t un = blockIdx.x + ((q + 1) / passes) * gridDim.x;
        const int64_t ln = static_cast<int64_t>((q + 1) % passes) * chunk;
        const int64_t lenn = (ld - ln) < chunk ? (ld - ln) : chunk;
        const uint32_t nb = static_cast<uint32_t>(lenn * sizeof(E));
        const int32_t gn = static_cast<int32_t>(un / S);
        for (int m = 0; m < M; ++m) {
          const int32_t idx = gn * M + m;
          if (idx >= count) break;
          const int32_t ag = static_cast<int32_t>((full ? static_cast<uint32_t>(idx) : items[idx]) & kItemMask);
          const unsigned char* src = reinterpret_cast<const unsigned char*>(A + static_cast<int64_t>(ag) * ld + ln);
          for (uint32_t off = 0; off < nb; off += 32768u) pf_l2(src + off, (nb - off) < 32768u ? (nb - off) : 32768u);
        }
      }
    }
  };

  if (tid == 0) {
    for (int k = 0; k < bufs; ++k) {
      mbar_init(&full_bar[k], 1);
      mbar_init(&empty_bar[k], NW);
      arrive_cnt[k] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    ebuf_n = 0;
  }
  __syncthreads();
  if (warp == 0)
    for (int64_t k = 0; k < bufs && k < stages; ++k) produce(k);

  Track<KM> ta[M], tj[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    ta[m].init();
    tj[m].init();
  }

  for (int64_t q = 0; q < stages; ++q) {
    const int b = static_cast<int>(q % bufs);
    const int64_t uq = blockIdx.x + (q / passes) * gridDim.x;
    const int p = static_cast<int>(q % passes);
    const int32_t group = static_cast<int32_t>(uq / S);
    const int32_t seg = static_cast<int32_t>(uq % S);

    mbar_wait(&full_bar[b], static_cast<uint32_t>((q / bufs) & 1));
    ItemInfo it[M];
#pragma unroll
    for (int m = 0; m < M; ++m) it[m] = info_s[b][m];
    Acc sv[M];
    const E* xrow[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int32_t ag = it[m].agent < 0 ? 0 : it[m].agent;
      const int32_t jb = it[m].job < 0 ? 0 : it[m].job;
      sv[m] = widen(acur[ag]);
      xrow[m] = AT + static_cast<int64_t>(jb) * ld;
    }
    const int64_t clo = static_cast<int64_t>(p) * chunk;
    const int32_t seg_lo = seg * seglen;
    const int32_t seg_hi = min(n, seg_lo + seglen);
    const int32_t full_hi = seg_lo + ((seg_hi - seg_lo) / V) * V;
    const E* rows = stage_base + static_cast<size_t>(b) * M * chunk;

    // main loop over whole vectors: a ring of D stream-register sets keeps
    // the next D-1 vector steps' loads in flight (fully unrolled, so every
    // set stays in registers)
    int32_t i0 = seg_lo + tid * V;
    StreamRegs<E, M> rr[D];
#pragma unroll
    for (int d = 0; d < D - 1; ++d)
      if (i0 + d * NT * V < full_hi) load_step<E, M>(rr[d], tau, acur, xrow, i0 + d * NT * V);
    for (bool more = i0 < full_hi; more;) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int32_t ic = i0 + d * NT * V;
        if (ic >= full_hi) {
          more = false;
          break;
        }
        const int32_t ipf = ic + (D - 1) * NT * V;
        if (ipf < full_hi) load_step<E, M>(rr[(d + D - 1) % D], tau, acur, xrow, ipf);
        compute_step<E, M, KM, kChunked>(rr[d], ic, V, rows, chunk, clo, sv, ta, tj);
      }
      i0 += D * NT * V;
    }
    // ragged tail (only the last segment when n % V != 0)
    if (full_hi < seg_hi && tid == 0) {
      StreamRegs<E, M> tr;
      load_step<E, M>(tr, tau, acur, xrow, full_hi);
      compute_step<E, M, KM, kChunked>(tr, full_hi, seg_hi - full_hi, rows, chunk, clo, sv, ta, tj);
    }

    if (p == passes - 1) {
      // warp partials -> red[b]; the last warp to arrive reduces and writes
      Track<KM>* rq = red + b * NW * 2 * M;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        ta[m].warp_reduce();
        tj[m].warp_reduce();
        if (lane == 0) {
          rq[warp * 2 * M + 2 * m] = ta[m];
          rq[warp * 2 * M + 2 * m + 1] = tj[m];
        }
        ta[m].init();
        tj[m].init();
      }
      int last = 0;
      if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(&arrive_cnt[b], 1) == NW - 1;
        if (last) arrive_cnt[b] = 0;
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        __threadfence_block();
        // lanes 0..2M-1 each own one track: reduce over the NW warp partials
        Track<KM> r;
        r.init();
        if (lane < 2 * M)
          for (int w = 0; w < NW; ++w) r.merge(rq[w * 2 * M + lane]);
        bool finalize = (S == 1);
        double d = 0.0;
        int32_t k = -1;
        bool ok = false;
        if (S == 1) {
          ok = lane < 2 * M && r.valid();
          d = ok ? r.delta() : 0.0;
          k = ok ? r.index() : -1;
        } else {
          // publish this segment's partials; the last segment to arrive combines
          if (lane < 2 * M) {
            const int64_t slot = (static_cast<int64_t>(group) * S + seg) * M + (lane >> 1);
            const double pd = r.valid() ? r.delta() : -__longlong_as_double(0x7ff0000000000000ll);
            const int32_t pk = r.valid() ? r.index() : INT_MAX;
            if ((lane & 1) == 0) {
              st.part_ad[slot] = pd;
              st.part_at[slot] = pk;
            } else {
              st.part_jd[slot] = pd;
              st.part_ji[slot] = pk;
            }
          }
          __threadfence();
          __syncwarp();
          int lastseg = 0;
          if (lane == 0) {
            lastseg = atomicAdd(&st.part_arrive[group], 1) == S - 1;
            if (lastseg) st.part_arrive[group] = 0;
          }
          finalize = __shfl_sync(0xffffffffu, lastseg, 0);
          if (finalize) {
            __threadfence();
            Track<kFloat> c;
            c.init();
            if (lane < 2 * M)
              for (int s2 = 0; s2 < S; ++s2) {
                const int64_t slot = (static_cast<int64_t>(group) * S + s2) * M + (lane >> 1);
                Track<kFloat> o;
                o.d = (lane & 1) ? __ldcg(&st.part_jd[slot]) : __ldcg(&st.part_ad[slot]);
                o.i = (lane & 1) ? __ldcg(&st.part_ji[slot]) : __ldcg(&st.part_at[slot]);
                c.merge(o);
              }
            ok = lane < 2 * M && c.valid();
            d = c.d;
            k = c.i;
          }
        }
        if (finalize) {
          bool emit = false;
          Prop entry;
          if (lane < 2 * M) {
            const ItemInfo im = info_s[b][lane >> 1];
            const bool active = ok && d > st.eps;
            if (im.agent >= 0) {
              if ((lane & 1) == 0) {
                if (im.flags & kItemAgent) {
                  st.agent_delta[im.agent] = active ? d : 0.0;
                  st.agent_partner[im.agent] = active ? k : -1;
                  emit = active && st.emit_edges;
                  if (emit)  // agent i -> job k (entries filled in at the flush)
                    entry = Prop{im.agent, im.agent, -1, k, im.job, 2, d, 0.0, 0.0};
                }
              } else if (im.flags & kItemJob) {
                st.job_delta[im.job] = active ? d : 0.0;
                st.job_partner[im.job] = active ? k : -1;
                emit = active && st.emit_edges;
                if (emit)  // agent k -> job j0, holder i -> tau[k] (filled in at the flush)
                  entry = Prop{n + im.job, k, im.agent, im.job, -1, 2, d, 0.0, 0.0};
              }
            }
          }
          // buffered append (one smem atomic per warp); flush when nearly full
          const unsigned mask = __ballot_sync(0xffffffffu, emit);
          if (mask) {
            int base = 0;
            if (lane == 0) base = atomicAdd(&ebuf_n, __popc(mask));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (emit) {
              const int pos = base + __popc(mask & ((1u << lane) - 1));
              if (pos < kEdgeBuf) {
                ebuf[pos] = entry;
              } else {  // overflow: direct global append
                const int g = atomicAdd(&st.ctrl->edge_count[parity_out], 1);
                st.edges[parity_out][g] = finish_prop(entry, st.sigma, tau, st.AT, st.storage, ld, n);
              }
            }
          }
        }
      }
    }
    // release buffer b to the producer
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[b]);
    // producer: refill buffer b with stage q + bufs once every warp released it
    if (warp == 0 && q + bufs < stages) {
      mbar_wait(&empty_bar[b], static_cast<uint32_t>((q / bufs) & 1));
      produce(q + bufs);
    }
  }
  // flush the CTA's buffered edges
  __syncthreads();
  const int ne = min(ebuf_n, kEdgeBuf);
  __shared__ int gbase;
  if (tid == 0 && ne > 0) gbase = atomicAdd(&st.ctrl->edge_count[parity_out], ne);
  __syncthreads();
  for (int e = tid; e < ne; e += NT)
    st.edges[parity_out][gbase + e] = finish_prop(ebuf[e], st.sigma, tau, st.AT, st.storage, ld, n);
}

constexpr size_t kStaticSmem = 14 * 1024;  // ebuf + item metadata + counters (+ slack)

template <class E, int M, int NT, int KM>
cudaError_t launch_nt(const DevState& d, const ScanPlan& p, int full, cudaStream_t st) {
  auto k = p.passes > 1 ? pair_scan_kernel<E, M, NT, KM, true, 2>
                        : (p.depth == 3 ? pair_scan_kernel<E, M, NT, KM, false, 3> : pair_scan_kernel<E, M, NT, KM, false, 2>);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(p.smem));
  if (e != cudaSuccess) return e;
  return launch_pdl(k, dim3(p.ctas), dim3(NT), p.smem, st, d.pdl, d, full, p.passes, p.chunk, p.bufs,
                    p.max_segments, p.l2_prefetch);
}

template <class E, int M, int KM>
cudaError_t launch_typed(const DevState& d, const ScanPlan& p, int full, cudaStream_t st) {
  return p.threads == 256 ? launch_nt<E, M, 256, KM>(d, p, full, st) : launch_nt<E, M, 512, KM>(d, p, full, st);
}

template <class E, int KM>
cudaError_t launch_m(const DevState& d, const ScanPlan& p, int full, cudaStream_t st) {
  switch (p.m) {
    case 1: return launch_typed<E, 1, KM>(d, p, full, st);
    case 2: return launch_typed<E, 2, KM>(d, p, full, st);
    case 4: return launch_typed<E, 4, KM>(d, p, full, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace scan_detail

// One explicit instantiation set per (storage, key mode), each in its own
// translation unit (scan_<type>.cu) so they compile in parallel.
template <class E, int KM>
cudaError_t launch_scan_typed(const DevState& d, const ScanPlan& p, int full, cudaStream_t st) {
  return scan_detail::launch_m<E, KM>(d, p, full, st);
}

}  // namespace lsapgpu
