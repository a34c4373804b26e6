// scan.cu -- the fused pair-scan kernel: the B200 replacement for the
// reference's exchange_scan ISA variants driven by eval_agent / eval_job
// (proj/src/kernels_scalar.cpp:6-25, kernels_avx2.cpp:40-92,
// solver_state.hpp:78-104) over eval_all / reeval_lists (parallel.cpp:80-124).
//
// One work item is an agent i together with its job j0 = tau[i].  Agent i's
// scan and job j0's scan read exactly the same two rows, A[i,:] and AT[j0,:]
// (SURVEY 8(a) row 8), so one pass produces both records:
//   for every agent i' != i, with t = tau[i'], x = AT[j0][i'], g = A[i][t],
//   c = acur[i'], s = acur[i]:
//     agent candidate (partner job t):   (g - s) + (x - c)
//     job   candidate (partner agent i'): (x - s) + (g - c)
// which are the reference's fp64 expressions in the reference's order.  The
// winner is the maximum with the smallest candidate index on ties, and it is
// active iff it exceeds eps (kernels_avx2.cpp:90).
//
// Data movement per item: A[i,:] is staged into shared memory with TMA bulk
// copies (cp.async.bulk + mbarrier) because it is gathered at random positions
// t; AT[j0,:] is streamed with 16-byte loads, as are tau and acur, which are
// shared by the M items a CTA scans together.  CTAs are persistent and double
// buffer their stages, so the next item group's rows land while the current
// group is being reduced.  Algorithmic HBM bytes: 2 * n * sizeof(elem) per item.
#include <cfloat>
#include <climits>
#include <cstdlib>

#include "state.h"

namespace lsapgpu {
namespace {

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
// 16-byte load of data re-read by every CTA (tau, acur): keep it cacheable.
__device__ __forceinline__ uint4 ld_shared16(const void* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

template <class E>
struct Vec {
  static constexpr int V = 16 / sizeof(E);
  E e[V];
};

template <class E>
__device__ __forceinline__ void load_vec(Vec<E>& out, const E* p, bool stream) {
  uint4 raw = stream ? ld_stream16(p) : ld_shared16(p);
  *reinterpret_cast<uint4*>(out.e) = raw;
}

template <int V>
__device__ __forceinline__ void load_tau(int32_t (&t)[V], const int32_t* p) {
  if constexpr (V == 8) {
    uint4 a = ld_shared16(p), b = ld_shared16(p + 4);
    t[0] = a.x; t[1] = a.y; t[2] = a.z; t[3] = a.w;
    t[4] = b.x; t[5] = b.y; t[6] = b.z; t[7] = b.w;
  } else if constexpr (V == 4) {
    uint4 a = ld_shared16(p);
    t[0] = a.x; t[1] = a.y; t[2] = a.z; t[3] = a.w;
  } else {
    uint2 a = __ldg(reinterpret_cast<const uint2*>(p));
    t[0] = a.x; t[1] = a.y;
  }
}

template <class Acc>
struct Best {
  Acc d;
  int32_t k;
};

template <class Acc>
__device__ __forceinline__ Acc acc_lowest() {
  if constexpr (sizeof(Acc) == 4)
    return INT_MIN;
  else
    return -__longlong_as_double(0x7ff0000000000000ll);
}

template <class Acc>
__device__ __forceinline__ void consider(Best<Acc>& b, Acc d, int32_t k) {
  // max delta, smallest candidate index among equal deltas
  const bool take = (d > b.d) || (d == b.d && k < b.k);
  b.d = take ? d : b.d;
  b.k = take ? k : b.k;
}

template <class Acc>
__device__ __forceinline__ void warp_reduce(Best<Acc>& b) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    Acc od = __shfl_down_sync(0xffffffffu, b.d, off);
    int32_t ok = __shfl_down_sync(0xffffffffu, b.k, off);
    consider(b, od, ok);
  }
}

struct ItemInfo {
  int32_t agent;  // -1: no item in this slot (tail group)
  int32_t job;    // tau[agent]
  uint32_t flags;
};

template <class E, int M, int NT>
__global__ void __launch_bounds__(NT) pair_scan_kernel(DevState st, int full, int passes,
                                                        int64_t chunk, int bufs, int max_segments) {
  using Acc = typename Traits<E>::Acc;
  constexpr int V = Vec<E>::V;
  constexpr int NW = NT / 32;
  constexpr bool kInt = Traits<E>::kInt;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int32_t n = st.n;
  const int64_t ld = st.ld;
  const E* __restrict__ A = static_cast<const E*>(st.A);
  const E* __restrict__ AT = static_cast<const E*>(st.AT);
  const E* __restrict__ acur = static_cast<const E*>(st.acur);
  const int32_t* __restrict__ tau = st.tau;

  const size_t chunk_bytes = static_cast<size_t>(chunk) * sizeof(E);
  E* stage_base = reinterpret_cast<E*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + bufs * M * chunk_bytes);
  Best<Acc>* red = reinterpret_cast<Best<Acc>*>(bars + 2);  // [NW][2M]
  __shared__ ItemInfo info_s[2][M];
  __shared__ int last_arriver;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  const int32_t count = full ? n : st.ctrl->work_count;
  if (count <= 0) return;
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
  const int32_t seg_gran = 32 * V;
  const int32_t seglen = ((n + S - 1) / S + seg_gran - 1) / seg_gran * seg_gran;
  const int parity_out = st.ctrl->parity;

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto item_of = [&](int32_t idx) -> ItemInfo {
    ItemInfo it;
    if (idx >= count) {
      it.agent = -1;
      it.job = -1;
      it.flags = 0;
      return it;
    }
    const uint32_t w = full ? (static_cast<uint32_t>(idx) | kItemAgent | kItemJob) : st.items[idx];
    it.agent = static_cast<int32_t>(w & kItemMask);
    it.job = tau[it.agent];
    it.flags = w & (kItemAgent | kItemJob);
    return it;
  };

  // Issue the TMA bulk copies of stage (unit u, pass p) into buffer b.
  auto issue = [&](int64_t u, int p, int b) {
    const int32_t group = static_cast<int32_t>(u / S);
    uint32_t total = 0;
    const int64_t lo = static_cast<int64_t>(p) * chunk;
    const int64_t len = (ld - lo) < chunk ? (ld - lo) : chunk;
    const uint32_t bytes = static_cast<uint32_t>(len * sizeof(E));
    int32_t agents[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int32_t idx = group * M + m;
      agents[m] = -1;
      if (idx < count) {
        const uint32_t w = full ? static_cast<uint32_t>(idx) : st.items[idx];
        agents[m] = static_cast<int32_t>(w & kItemMask);
        total += bytes;
      }
    }
    mbar_expect_tx(&bars[b], total);
#pragma unroll
    for (int m = 0; m < M; ++m) {
      if (agents[m] < 0) continue;
      const unsigned char* src =
          reinterpret_cast<const unsigned char*>(A + static_cast<int64_t>(agents[m]) * ld + lo);
      unsigned char* dst = reinterpret_cast<unsigned char*>(stage_base) + (b * M + m) * chunk_bytes;
      for (uint32_t off = 0; off < bytes; off += 32768u) {
        const uint32_t sz = (bytes - off) < 32768u ? (bytes - off) : 32768u;
        bulk_g2s(dst + off, src + off, sz, &bars[b]);
      }
    }
  };

  Best<Acc> ba[M], bj[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    ba[m] = {acc_lowest<Acc>(), INT_MAX};
    bj[m] = {acc_lowest<Acc>(), INT_MAX};
  }

  int64_t u = blockIdx.x;
  int p = 0;
  uint32_t q = 0;  // stage counter (buffer = q % bufs, phase = (q / bufs) & 1)
  if (u < units && tid == 0) issue(u, 0, 0);

  while (u < units) {
    const int b = static_cast<int>(q % bufs);
    const uint32_t phase = (q / bufs) & 1u;
    int64_t u2 = u;
    int p2 = p + 1;
    if (p2 == passes) {
      p2 = 0;
      u2 = u + gridDim.x;
    }
    if (bufs == 2 && u2 < units && tid == 0) issue(u2, p2, (q + 1) % 2);

    const int32_t group = static_cast<int32_t>(u / S);
    const int32_t seg = static_cast<int32_t>(u % S);
    if (tid < M) info_s[q & 1][tid] = item_of(group * M + tid);
    __syncthreads();
    ItemInfo it[M];
#pragma unroll
    for (int m = 0; m < M; ++m) it[m] = info_s[q & 1][m];
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

    mbar_wait(&bars[b], phase);
    const E* rows = stage_base + static_cast<size_t>(b) * M * chunk;

    for (int32_t i0 = seg_lo + tid * V; i0 < seg_hi; i0 += NT * V) {
      int32_t tv[V];
      Vec<E> cv;
      Vec<E> xv[M];
      load_tau<V>(tv, tau + i0);
      load_vec(cv, acur + i0, false);
#pragma unroll
      for (int m = 0; m < M; ++m) load_vec(xv[m], xrow[m] + i0, true);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int32_t ip = i0 + v;
        const int64_t tl = static_cast<int64_t>(tv[v]) - clo;
        const bool ok = ip < seg_hi && (passes == 1 || (tl >= 0 && tl < chunk));
        const Acc c = widen(cv.e[v]);
#pragma unroll
        for (int m = 0; m < M; ++m) {
          if (ok && ip != it[m].agent && it[m].agent >= 0) {
            const Acc g = widen(rows[static_cast<size_t>(m) * chunk + tl]);
            const Acc x = widen(xv[m].e[v]);
            if constexpr (kInt) {
              const Acc d = delta4(g, sv[m], x, c);
              consider(ba[m], d, tv[v]);
              consider(bj[m], d, ip);
            } else {
              consider(ba[m], delta4(g, sv[m], x, c), tv[v]);
              consider(bj[m], delta4(x, sv[m], g, c), ip);
            }
          }
        }
      }
    }

    if (p == passes - 1) {
      // CTA reduction of the 2M (delta, index) pairs
#pragma unroll
      for (int m = 0; m < M; ++m) {
        warp_reduce(ba[m]);
        warp_reduce(bj[m]);
        if (lane == 0) {
          red[warp * 2 * M + 2 * m] = ba[m];
          red[warp * 2 * M + 2 * m + 1] = bj[m];
        }
        ba[m] = {acc_lowest<Acc>(), INT_MAX};
        bj[m] = {acc_lowest<Acc>(), INT_MAX};
      }
      __syncthreads();
      if (tid < 2 * M) {
        Best<Acc> r = red[tid];
        for (int w = 1; w < NW; ++w) consider(r, red[w * 2 * M + tid].d, red[w * 2 * M + tid].k);
        red[tid] = r;
      }
      __syncthreads();
      bool finalize = (S == 1);
      if (S > 1) {
        // publish this segment's partials; the last segment to arrive combines
        if (tid < 2 * M) {
          const int64_t slot = (static_cast<int64_t>(group) * S + seg) * M + (tid >> 1);
          if ((tid & 1) == 0) {
            st.part_ad[slot] = static_cast<double>(red[tid].d);
            st.part_at[slot] = red[tid].k;
          } else {
            st.part_jd[slot] = static_cast<double>(red[tid].d);
            st.part_ji[slot] = red[tid].k;
          }
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
          const int prev = atomicAdd(&st.part_arrive[group], 1);
          last_arriver = (prev == S - 1);
          if (last_arriver) st.part_arrive[group] = 0;
        }
        __syncthreads();
        finalize = last_arriver;
        if (finalize) {
          __threadfence();
          if (tid < 2 * M) {
            const int m = tid >> 1;
            Best<double> r = {-__longlong_as_double(0x7ff0000000000000ll), INT_MAX};
            for (int s2 = 0; s2 < S; ++s2) {
              const int64_t slot = (static_cast<int64_t>(group) * S + s2) * M + m;
              const double d = (tid & 1) ? __ldcg(&st.part_jd[slot]) : __ldcg(&st.part_ad[slot]);
              const int32_t k = (tid & 1) ? __ldcg(&st.part_ji[slot]) : __ldcg(&st.part_at[slot]);
              consider(r, d, k);
            }
            // stash combined result back as Acc (exact: int deltas are < 2^31)
            red[tid].d = static_cast<Acc>(r.d);
            red[tid].k = r.k;
          }
          __syncthreads();
        }
      }
      if (finalize && tid < 2 * M) {
        const int m = tid >> 1;
        const ItemInfo& im = it[m];
        if (im.agent >= 0) {
          const double d = static_cast<double>(red[tid].d);
          const bool active = d > st.eps && red[tid].k != INT_MAX;
          if ((tid & 1) == 0) {
            if (im.flags & kItemAgent) {
              st.agent_delta[im.agent] = active ? d : 0.0;
              st.agent_partner[im.agent] = active ? red[tid].k : -1;
              if (active) {
                const int pos = atomicAdd(&st.ctrl->edge_count[parity_out], 1);
                st.edges[parity_out][pos] = im.agent;
              }
            }
          } else {
            if (im.flags & kItemJob) {
              st.job_delta[im.job] = active ? d : 0.0;
              st.job_partner[im.job] = active ? red[tid].k : -1;
              if (active) {
                const int pos = atomicAdd(&st.ctrl->edge_count[parity_out], 1);
                st.edges[parity_out][pos] = n + im.job;
              }
            }
          }
        }
      }
    }
    __syncthreads();  // stage buffer b and red[] are free again
    if (bufs == 1 && u2 < units && tid == 0) issue(u2, p2, 0);
    ++q;
    u = u2;
    p = p2;
  }
}

template <class E, int M>
cudaError_t launch_typed(const DevState& d, const ScanPlan& p, int full, cudaStream_t st) {
  auto k = pair_scan_kernel<E, M, 256>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(p.smem));
  if (e != cudaSuccess) return e;
  k<<<p.ctas, 256, p.smem, st>>>(d, full, p.passes, p.chunk, p.bufs, p.max_segments);
  return cudaGetLastError();
}

template <class E>
cudaError_t launch_m(const DevState& d, const ScanPlan& p, int full, cudaStream_t st) {
  switch (p.m) {
    case 1: return launch_typed<E, 1>(d, p, full, st);
    case 2: return launch_typed<E, 2>(d, p, full, st);
    case 4: return launch_typed<E, 4>(d, p, full, st);
    default: return cudaErrorInvalidValue;
  }
}

size_t elem_size(int storage) {
  switch (storage) {
    case kI16: return 2;
    case kI32: return 4;
    case kF32: return 4;
    default: return 8;
  }
}

}  // namespace

ScanPlan plan_scan(const DevState& d, int num_sms) {
  ScanPlan p;
  const size_t es = elem_size(d.storage);
  // dynamic smem per CTA we plan against; LSAPGPU_SCAN_BUDGET (bytes) and
  // LSAPGPU_SCAN_M override the plan so tests can reach every code path
  // (multi-pass chunking, single buffering, item batching) at small n.
  size_t budget = 200 * 1024;
  if (const char* b = std::getenv("LSAPGPU_SCAN_BUDGET")) budget = std::strtoull(b, nullptr, 10);
  int force_m = 0;
  if (const char* m = std::getenv("LSAPGPU_SCAN_M")) force_m = std::atoi(m);
  const size_t row = static_cast<size_t>(d.ld) * es;
  const size_t reserve = 256 + 8 * 64 * 2 * 4;  // barriers + reduction scratch
  p.threads = 256;
  if (row <= budget) {
    p.passes = 1;
    p.chunk = d.ld;
    // batch items so tau/acur (L2) traffic is amortised, double buffered
    if (4 * 2 * row <= budget)
      p.m = 4;
    else if (2 * 2 * row <= budget)
      p.m = 2;
    else
      p.m = 1;
    if (force_m == 1 || force_m == 2 || force_m == 4) p.m = force_m;
    p.bufs = (2 * p.m * row <= budget) ? 2 : 1;
  } else {
    p.m = 1;
    p.bufs = 1;
    p.passes = static_cast<int>((row + budget - 1) / budget);
    int64_t ch = (d.ld + p.passes - 1) / p.passes;
    ch = (ch + 63) / 64 * 64;
    p.chunk = ch;
  }
  p.smem = static_cast<size_t>(p.bufs) * p.m * p.chunk * es + reserve;
  int per_sm = static_cast<int>((227 * 1024) / (p.smem + 1024));
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 8) per_sm = 8;
  p.ctas = num_sms * per_sm;
  p.max_segments = static_cast<int>(d.n / 2048);
  if (const char* s = std::getenv("LSAPGPU_SCAN_SEGMENTS")) p.max_segments = std::atoi(s);
  if (p.max_segments < 1) p.max_segments = 1;
  if (p.max_segments > 16) p.max_segments = 16;
  return p;
}

cudaError_t launch_scan(const DevState& d, const ScanPlan& p, int full, cudaStream_t st) {
  switch (d.storage) {
    case kI16: return launch_m<int16_t>(d, p, full, st);
    case kI32: return launch_m<int32_t>(d, p, full, st);
    case kF32: return launch_m<float>(d, p, full, st);
    case kF64: return launch_m<double>(d, p, full, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lsapgpu
