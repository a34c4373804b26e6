// auction.cu -- the reference's synchronous (Jacobi) auction baseline,
// lsap::auction_solve (proj/src/auction.cpp:110-153, baselines.hpp:12-36),
// on the device matrix A (row-major, storage type E).  SURVEY 8(f) item 4.
//
// The reference runs thousands of bidding rounds in which only a handful of
// agents are unassigned, so the loop is latency-bound, not bandwidth-bound:
// the whole solve (every round of every epsilon phase, and the greedy
// completion after a deadline) runs in ONE launch of one thread-block cluster
// (16 CTAs x 1024 threads where the part allows, else 8) whose rounds are
// separated by cluster barriers instead of kernel launches.
//
// One round (run_phase, auction.cpp:33-80):
//   bid    every unassigned agent i scans its row once: the best net benefit
//          A[i][k] - price[k] (smallest k on ties, net_scan's `d > best`,
//          kernels_scalar.cpp:40-54) and the second best (max over k != best,
//          the second net_scan with skip = best); bid = (price[best] +
//          (best - second)) + eps, every op a round-to-nearest fp64 add/sub
//          in the reference's order.  The agents are spread over the cluster
//          in groups of G warps per agent (G = 32 when few agents bid), and
//          read the prices from a shared-memory replica in every CTA (n up
//          to 20k).  The bid is posted to its job's 128-bit slot {inverted
//          agent, order-preserving key of the fp64 bid} with a CAS loop that
//          keeps the lexicographic maximum: the reference's "highest bid
//          wins, smallest agent on ties" (ascending agent loop with strict
//          `>`) in ONE atomic step, so a round needs two cluster barriers.
//   award  after the barrier each bidder reads its job's slot: the winner
//   apply  displaces the holder (queued for the next round), takes the job
//          and sets the price (global copy + every CTA's replica); losers are
//          queued again.  Every agent bids for exactly one job and displaced
//          holders never bid, so the awards are independent and their order
//          is immaterial.  Each CTA queues into its own list segment and
//          publishes the segment length to every peer through DSMEM.
// Top-2 reductions use exact max / min-index merges, so the result does not
// depend on how the row is split: bids, prices and the final assignment are
// bit-identical to the reference's.
#include <cooperative_groups.h>

#include <climits>

#include "state.h"

namespace cg = cooperative_groups;

namespace lsapgpu {
namespace {

constexpr int kNT = 1024;

// Order-preserving unsigned key of an fp64 value (0 = below every value).
__device__ __forceinline__ unsigned long long okey(double x) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

template <class T>
__device__ __forceinline__ T ldcg(const T* p) {
  return __ldcg(p);
}

// best value / its (smallest) index / best value over the other indices
struct Top2 {
  double b1, b2;
  int32_t i1;
};

__device__ __forceinline__ Top2 top2_empty() {
  const double ninf = __longlong_as_double(static_cast<long long>(0xFFF0000000000000ull));
  return {ninf, ninf, INT_MAX};
}

// Elements arrive in ascending index per thread: strict `>` keeps the first.
__device__ __forceinline__ void top2_add(Top2& t, double d, int32_t k) {
  if (d > t.b1) {
    t.b2 = t.b1;
    t.b1 = d;
    t.i1 = k;
  } else if (d > t.b2) {
    t.b2 = d;
  }
}

__device__ __forceinline__ Top2 top2_merge(const Top2& a, const Top2& b) {
  const bool bw = b.b1 > a.b1 || (b.b1 == a.b1 && b.i1 < a.i1);
  Top2 r;
  r.b1 = bw ? b.b1 : a.b1;
  r.i1 = bw ? b.i1 : a.i1;
  r.b2 = fmax(bw ? a.b1 : b.b1, bw ? b.b2 : a.b2);
  return r;
}

__device__ __forceinline__ Top2 top2_warp(Top2 t) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    Top2 o;
    o.b1 = __shfl_xor_sync(0xffffffffu, t.b1, off);
    o.b2 = __shfl_xor_sync(0xffffffffu, t.b2, off);
    o.i1 = __shfl_xor_sync(0xffffffffu, t.i1, off);
    t = top2_merge(t, o);
  }
  return t;
}

__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void row_pf(const void* p, uint32_t bytes) {
  for (uint32_t off = 0; off < bytes; off += 32768u)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(static_cast<const char*>(p) + off),
                 "r"(bytes - off < 32768u ? bytes - off : 32768u)
                 : "memory");
}

// 128-bit compare-and-swap on a bid slot {lo, hi}; returns the old value.
__device__ __forceinline__ void cas128(unsigned long long* p, unsigned long long c0, unsigned long long c1,
                                       unsigned long long s0, unsigned long long s1, unsigned long long& o0,
                                       unsigned long long& o1) {
  asm volatile(
      "{\n\t.reg .b128 d, c, s;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 s, {%4, %5};\n\t"
      "atom.relaxed.gpu.global.cas.b128 d, [%6], c, s;\n\t"
      "mov.b128 {%0, %1}, d;\n\t}"
      : "=l"(o0), "=l"(o1)
      : "l"(c0), "l"(c1), "l"(s0), "l"(s1), "l"(p)
      : "memory");
}

// Post a bid to its job's slot: {lo = inverted agent, hi = order key of the
// bid}, kept at the lexicographic maximum (highest bid, then smallest agent)
// by a CAS loop; an empty slot is {0, 0}.
__device__ __forceinline__ void post_bid(unsigned long long* slot, double bid, int32_t agent) {
  const unsigned long long h = okey(bid), l = 0xFFFFFFFFull - static_cast<unsigned long long>(agent);
  unsigned long long c0 = 0, c1 = 0;
  for (;;) {
    if (c1 > h || (c1 == h && c0 >= l)) return;  // a better bid is posted
    unsigned long long o0, o1;
    cas128(slot, c0, c1, l, h, o0, o1);
    if (o0 == c0 && o1 == c1) return;
    c0 = o0;
    c1 = o1;
  }
}

constexpr int kRec = 2048;  // bid records per CTA held in shared memory (the rest in global)

template <class E, int CS>
__global__ void __launch_bounds__(kNT, 1) auction_kernel(DevState st, AuctionDev a, int64_t remaining_ns) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t n = st.n;
  const int64_t ld = st.ld;
  const E* A = static_cast<const E*>(st.A);
  AuctionCtrl* C = a.ctrl;
  const int gtid = rank * kNT + tid;
  constexpr int kThreads = CS * kNT;

  extern __shared__ __align__(16) unsigned char dsm[];
  double* sprice = a.local_prices ? reinterpret_cast<double*>(dsm) : nullptr;  // replica of prices
  __shared__ Top2 part[32];
  __shared__ int32_t s_cnt[2][CS];  // bidders each CTA queued for the next round (written by that CTA)
  __shared__ int32_t s_pre[CS + 1];
  __shared__ int s_expired, s_nrec, s_push, s_awards;
  __shared__ int32_t r_i[kRec], r_j[kRec];
  __shared__ double r_bid[kRec];
  __shared__ Top2 cand[CS];  // greedy completion: per-CTA candidates (rank 0's copy is used)

  const bool has_deadline = remaining_ns >= 0;
  unsigned long long deadline_gt = 0;
  if (rank == 0 && tid == 0) deadline_gt = now_ns() + static_cast<unsigned long long>(has_deadline ? remaining_ns : 0);
  if (tid == 0) {
    s_expired = 0;
    s_awards = 0;
  }
  if (sprice)
    for (int32_t x = tid; x < n; x += kNT) sprice[x] = 0.0;
  cluster.sync();  // every CTA's flags are initialised before peers write them
  int32_t* grec_i = a.rec_i + static_cast<int64_t>(rank) * n;
  int32_t* grec_j = a.rec_j + static_cast<int64_t>(rank) * n;
  double* grec_b = a.rec_bid + static_cast<int64_t>(rank) * n;

  int cur = 0;
  bool finished = true;
  int64_t round = 0, bids = 0;
  bool snap = false;
  const int32_t per0 = (n + CS - 1) / CS;
  for (int p = 0; p < a.n_eps && finished; ++p) {
    const double eps = a.eps_list[p];
    // clear_assignment (auction.cpp:23-27); prices persist across phases.
    // Bidder list: CTA r's segment [r*n, r*n + cnt) of the current list.
    int32_t* wl0 = cur ? a.wl[1] : a.wl[0];
    for (int32_t x = gtid; x < n; x += kThreads) a.owner[x] = -1;
    for (int32_t x = tid; x < per0 && rank * per0 + x < n; x += kNT) wl0[static_cast<int64_t>(rank) * n + x] = rank * per0 + x;
    if (tid < CS) s_cnt[cur][tid] = max(0, min(n, (tid + 1) * per0) - tid * per0);
    if (rank == 0 && tid == 0) {
      C->phases += 1;
      if (has_deadline && now_ns() >= deadline_gt)  // dl.expired(), auction.cpp:42
        for (int r = 0; r < CS; ++r) *cluster.map_shared_rank(&s_expired, r) = 1;
    }
    cluster.sync();
    for (;;) {
      if (snap) {  // on_round observer (auction.cpp:76): prices after round `round`
        if (round - 1 < a.round_cap)
          for (int32_t x = gtid; x < n; x += kThreads)
            a.round_prices[(round - 1) * static_cast<int64_t>(n) + x] = ldcg(a.prices + x);
        snap = false;
      }
      if (tid == 0) {
        int acc = 0;
        for (int r = 0; r < CS; ++r) {
          s_pre[r] = acc;
          acc += s_cnt[cur][r];
        }
        s_pre[CS] = acc;
        s_nrec = 0;
        s_push = 0;
      }
      __syncthreads();
      const int32_t cnt = s_pre[CS];
      if (rank == 0 && tid == 0) tl_mark(st.ctrl, st.tl, st.tl_cap, 1);
      if (cnt == 0) break;
      if (s_expired) {
        finished = false;
        break;
      }
      const int32_t* wl = cur ? a.wl[1] : a.wl[0];
      int32_t* next = cur ? a.wl[0] : a.wl[1];

      // ---- bid: scan, then post to the job's slot ----
      const int per_cta = (cnt + CS - 1) / CS;
      int G = 32;
      while (G > 1 && 32 / G < per_cta) G >>= 1;
      const int groups = 32 / G, grp = warp / G, wig = warp % G;
      for (int32_t base = 0; base < cnt; base += CS * groups) {
        const int32_t k = base + rank * groups + grp;
        const bool valid = k < cnt;
        Top2 t = top2_empty();
        int32_t i = -1;
        if (valid) {
          int sg = 0;
          while (s_pre[sg + 1] <= k) ++sg;
          i = ldcg(wl + static_cast<int64_t>(sg) * n + (k - s_pre[sg]));
          // lane-consecutive elements: coalesced row loads, conflict-free
          // price reads (a 16-byte-vector variant measured slower)
          const E* row = A + static_cast<int64_t>(i) * ld;
          if (sprice) {
#pragma unroll 4
            for (int32_t x = wig * 32 + lane; x < n; x += G * 32)
              top2_add(t, __dsub_rn(static_cast<double>(row[x]), sprice[x]), x);
          } else {
#pragma unroll 4
            for (int32_t x = wig * 32 + lane; x < n; x += G * 32)
              top2_add(t, __dsub_rn(static_cast<double>(row[x]), ldcg(a.prices + x)), x);
          }
        }
        t = top2_warp(t);
        if (lane == 0) part[warp] = t;
        __syncthreads();
        if (valid && wig == 0) {  // the group's first warp merges its G partials
          t = top2_warp(lane < G ? part[warp + lane] : top2_empty());
        }
        if (valid && wig == 0 && lane == 0) {
          const double second = n > 1 ? t.b2 : t.b1;
          const double pb = sprice ? sprice[t.i1] : ldcg(a.prices + t.i1);
          const double bid = __dadd_rn(__dadd_rn(pb, __dsub_rn(t.b1, second)), eps);
          post_bid(a.slot + 2 * static_cast<int64_t>(t.i1), bid, i);
          const int r = atomicAdd(&s_nrec, 1);
          if (r < kRec) {
            r_i[r] = i;
            r_j[r] = t.i1;
            r_bid[r] = bid;
          } else {
            grec_i[r] = i;
            grec_j[r] = t.i1;
            grec_b[r] = bid;
          }
        }
        __syncthreads();
      }
      if (rank == 0 && tid == 0) tl_mark(st.ctrl, st.tl, st.tl_cap, 2);
      cluster.sync();
      if (rank == 0 && tid == 0) tl_mark(st.ctrl, st.tl, st.tl_cap, 3);

      // ---- award + apply: the slot holds the highest bid / smallest agent ----
      const int nrec = s_nrec;
      const int nxt = cur ^ 1;
      int awards = 0;
      for (int base = tid - lane; base < nrec; base += kNT) {
        const int r = base + lane;
        bool lost = false, displaced = false;
        int32_t i = -1, prev = -1;
        if (r < nrec) {
          int32_t j;
          double bid;
          if (r < kRec) {
            i = r_i[r];
            j = r_j[r];
            bid = r_bid[r];
          } else {
            i = grec_i[r];
            j = grec_j[r];
            bid = grec_b[r];
          }
          unsigned long long* sl = a.slot + 2 * static_cast<int64_t>(j);
          const int32_t w = static_cast<int32_t>(0xFFFFFFFFull - ldcg(sl));
          const int32_t old = ldcg(a.owner + j);
          if (w == i) {
            prev = old;
            displaced = prev >= 0;
            a.owner[j] = i;
            a.prices[j] = bid;
            if (sprice)
              for (int q = 0; q < CS; ++q) *cluster.map_shared_rank(sprice + j, q) = bid;
            sl[0] = 0ull;
            sl[1] = 0ull;
            ++awards;
          } else {
            lost = true;
          }
        }
        // losers and displaced holders bid again next round (this CTA's segment)
        const unsigned ml = __ballot_sync(0xffffffffu, lost), md = __ballot_sync(0xffffffffu, displaced);
        if (ml | md) {
          int b0 = 0;
          if (lane == 0) b0 = atomicAdd(&s_push, __popc(ml) + __popc(md));
          b0 = __shfl_sync(0xffffffffu, b0, 0);
          int32_t* seg = next + static_cast<int64_t>(rank) * n;
          if (lost) seg[b0 + __popc(ml & ((1u << lane) - 1))] = i;
          if (displaced) seg[b0 + __popc(ml) + __popc(md & ((1u << lane) - 1))] = prev;
          // next round's rows start streaming into L2 now (matrices larger than L2)
          if (a.row_prefetch) {
            const uint32_t rb = static_cast<uint32_t>(static_cast<size_t>(n) * sizeof(E) + 15) / 16 * 16;
            if (lost) row_pf(A + static_cast<int64_t>(i) * ld, rb);
            if (displaced) row_pf(A + static_cast<int64_t>(prev) * ld, rb);
          }
        }
      }
      for (int off = 16; off > 0; off >>= 1) awards += __shfl_down_sync(0xffffffffu, awards, off);
      if (lane == 0 && awards) atomicAdd(&s_awards, awards);
      __syncthreads();
      if (tid < CS) *cluster.map_shared_rank(&s_cnt[nxt][rank], tid) = s_push;
      if (rank == 0 && tid == 0 && has_deadline && now_ns() >= deadline_gt)
        for (int r = 0; r < CS; ++r) *cluster.map_shared_rank(&s_expired, r) = 1;
      if (rank == 0 && tid == 0) tl_mark(st.ctrl, st.tl, st.tl_cap, 4);
      bids += cnt;
      ++round;
      snap = true;
      cluster.sync();
      cur = nxt;
    }
  }

  if (!finished) {
    // complete_greedily (auction.cpp:84-106): ascending unassigned agents,
    // each takes its best free job by raw benefit (first job on ties)
    for (int32_t x = gtid; x < n; x += kThreads) a.assigned[x] = -1;
    cluster.sync();
    for (int32_t x = gtid; x < n; x += kThreads) {
      const int32_t o = ldcg(a.owner + x);
      if (o >= 0) a.assigned[o] = x;
    }
    cluster.sync();
    const int32_t j0 = rank * per0, j1 = min(n, j0 + per0);
    for (int32_t i = 0; i < n; ++i) {
      if (ldcg(a.assigned + i) >= 0) continue;
      const E* row = A + static_cast<int64_t>(i) * ld;
      Top2 t = top2_empty();
      for (int32_t j = j0 + tid; j < j1; j += kNT)
        if (ldcg(a.owner + j) < 0) top2_add(t, static_cast<double>(row[j]), j);
      t = top2_warp(t);
      if (lane == 0) part[warp] = t;
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < 32; ++w) t = top2_merge(t, part[w]);
        *cluster.map_shared_rank(&cand[rank], 0) = t;
      }
      cluster.sync();
      if (rank == 0 && tid == 0) {
        Top2 b = cand[0];
        for (int r = 1; r < CS; ++r) b = top2_merge(b, cand[r]);
        a.owner[b.i1] = i;
        a.assigned[i] = b.i1;
      }
      cluster.sync();
    }
  }
  if (tid == 0) {
    if (s_awards) atomicAdd(reinterpret_cast<unsigned long long*>(&C->switches),
                            static_cast<unsigned long long>(s_awards));
    if (rank == 0) {
      C->rounds = round;  // rep.outer_iterations
      C->bids = bids;
      C->finished = finished ? 1 : 0;
      C->greedy = finished ? 0 : 1;
    }
  }
  cluster.sync();
  // sigma = owner (auction.cpp:147-148); the host derives tau and the value
  for (int32_t x = gtid; x < n; x += kThreads) st.sigma[x] = ldcg(a.owner + x);
}

template <class E>
__global__ void minmax_kernel(DevState st, AuctionCtrl* c) {
  const E* A = static_cast<const E*>(st.A);
  const double inf = __longlong_as_double(0x7FF0000000000000ll);
  double lo = inf, hi = -inf;
  for (int64_t r = blockIdx.x; r < st.n; r += gridDim.x) {
    const E* row = A + r * st.ld;
    for (int32_t k = threadIdx.x; k < st.n; k += blockDim.x) {
      const double v = static_cast<double>(row[k]);
      lo = fmin(lo, v);
      hi = fmax(hi, v);
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, off));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, off));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&c->lo_key, okey(lo));
    atomicMax(&c->hi_key, okey(hi));
  }
}

template <class E, int CS>
cudaError_t launch_cs(const DevState& d, const AuctionDev& a, int64_t remaining_ns, cudaStream_t st) {
  auto k = auction_kernel<E, CS>;
  if (CS > 8) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  const size_t dyn = a.local_prices ? sizeof(double) * static_cast<size_t>(d.n) : 0;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS);
  cfg.blockDim = dim3(kNT);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, d, a, remaining_ns);
}

template <int CS>
cudaError_t launch_any(const DevState& d, const AuctionDev& a, int64_t remaining_ns, cudaStream_t st) {
  switch (d.storage) {
    case kI16: return launch_cs<int16_t, CS>(d, a, remaining_ns, st);
    case kI32: return launch_cs<int32_t, CS>(d, a, remaining_ns, st);
    case kF32: return launch_cs<float, CS>(d, a, remaining_ns, st);
    case kF64: return launch_cs<double, CS>(d, a, remaining_ns, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

// Largest n whose price replica fits next to the static shared memory.
int32_t auction_local_price_cap() { return 20480; }

int auction_cluster_size() {
  static int cached = 0;
  if (cached) return cached;
  auto k = auction_kernel<int32_t, 16>;
  int clusters = 0;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(kNT);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 16;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&clusters, k, &cfg) != cudaSuccess) clusters = 0;
  }
  cudaGetLastError();
  cached = clusters > 0 ? 16 : 8;
  return cached;
}

cudaError_t launch_auction(const DevState& d, const AuctionDev& a, int64_t remaining_ns, cudaStream_t st) {
  return auction_cluster_size() == 16 ? launch_any<16>(d, a, remaining_ns, st)
                                      : launch_any<8>(d, a, remaining_ns, st);
}

cudaError_t launch_minmax(const DevState& d, AuctionCtrl* c, cudaStream_t st) {
  const dim3 grid(static_cast<unsigned>(std::min<int64_t>(d.n, 148 * 8))), block(256);
  switch (d.storage) {
    case kI16: minmax_kernel<int16_t><<<grid, block, 0, st>>>(d, c); break;
    case kI32: minmax_kernel<int32_t><<<grid, block, 0, st>>>(d, c); break;
    case kF32: minmax_kernel<float><<<grid, block, 0, st>>>(d, c); break;
    case kF64: minmax_kernel<double><<<grid, block, 0, st>>>(d, c); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

double auction_key_value(unsigned long long key) {
  const unsigned long long b = (key >> 63) ? (key & 0x7FFFFFFFFFFFFFFFull) : ~key;
  double v;
  static_assert(sizeof(v) == sizeof(b), "");
  __builtin_memcpy(&v, &b, sizeof(v));
  return v;
}

}  // namespace lsapgpu
