// scan_big.cuh -- the pair scan for rows too long to double-buffer on one SM
// but short enough to stage once (C4: n = 30000 fp32, 120 KB rows).
//
// Same work item and arithmetic as the other scan kernels (scan_kernel.cuh):
// item = agent i with its job j0 = tau[i]; candidates over i' with
// t = tau[i'], x = AT[j0][i'], g = A[i][t], c = acur[i'] give agent i's record
// ((g - s) + (x - c), tie index t) and job j0's record ((x - s) + (g - c),
// tie index i') -- kernels_scalar.cpp:6-25, solver_state.hpp:78-92.
//
// One item per stage.  The gathered row A[i,:] is staged whole (TMA, one
// buffer: two do not fit), and everything indexed by the position i' --
// AT[j0,:], tau16 and acur -- streams through a ring of position chunks that
// TMA fills ahead of the consumers (one copy per array per chunk, issued by
// three lanes in parallel so small copies keep up).  The streaming kernel
// held those streams in registers one vector step ahead, which left the SM
// waiting on HBM latency (43 % long-scoreboard stalls at C4).  While the last
// chunks of an item are scanned, the next item's row is prefetched into L2,
// so the exposed single-buffer refill is served from L2.
//
// Warps: 14 consumers, warp 14 fills the chunk ring, warp 15 stages A rows.
// Algorithmic HBM bytes: 2 * n * sizeof(elem) per item.
#pragma once

#include "scan_resident.cuh"

namespace lsapgpu {
namespace scan_detail {

constexpr int kBigThreads = 512;
constexpr int kBigWarps = kBigThreads / 32 - 2;  // consumer warps
constexpr int kBigSlots = 2;                      // chunk ring depth
constexpr int kBigEdgeBuf = 256;

// smem: A row [ld] | slots [R] x (AT chunk [C] E, acur chunk [C] E, tau16 chunk [C]) |
//       a_full, a_empty, slot_full[R], slot_empty[R] mbarriers | red[NW][2]
template <class E, int KM>
__global__ void __launch_bounds__(kBigThreads, 1)
    pair_scan_big_kernel(DevState st, int full, int32_t C) {
  using Acc = typename Traits<E>::Acc;
  constexpr int V = 16 / sizeof(E);
  constexpr int NW = kBigWarps;
  constexpr int32_t kBlk = 32 * V;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int32_t n = st.n;
  const int64_t ld = st.ld;
  const E* __restrict__ A = static_cast<const E*>(st.A);
  const E* __restrict__ AT = static_cast<const E*>(st.AT);
  const E* __restrict__ acur_g = static_cast<const E*>(st.acur);
  const uint16_t* __restrict__ tau16_g = st.tau16;
  const int32_t* __restrict__ tau_g = st.tau;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  pdl_trigger();
  pdl_wait();
  if (blockIdx.x == 0 && tid == 0) tl_mark(st.ctrl, st.tl, st.tl_cap, full ? kTlScanFull : kTlScan);

  const size_t row_bytes = static_cast<size_t>(ld) * sizeof(E);
  const size_t cb = static_cast<size_t>(C) * sizeof(E);  // AT / acur chunk bytes
  const size_t tb = static_cast<size_t>(C) * 2;           // tau16 chunk bytes
  const size_t slot_bytes = 2 * cb + tb;
  E* a_s = reinterpret_cast<E*>(smem_raw);
  unsigned char* slots = smem_raw + (row_bytes + 127) / 128 * 128;
  uint64_t* bars = reinterpret_cast<uint64_t*>(slots + kBigSlots * ((slot_bytes + 127) / 128 * 128));
  uint64_t* a_full = bars;
  uint64_t* a_empty = bars + 1;
  uint64_t* slot_full = bars + 2;
  uint64_t* slot_empty = bars + 2 + kBigSlots;
  Track<KM>* red = reinterpret_cast<Track<KM>*>(bars + 2 + 2 * kBigSlots);  // [NW][2]
  const size_t slot_stride = (slot_bytes + 127) / 128 * 128;
  __shared__ ResInfo info_s;
  __shared__ int blk_next[kBigSlots];
  __shared__ int slot_done[kBigSlots];
  __shared__ int item_done;
  __shared__ Prop ebuf[kBigEdgeBuf];
  __shared__ int ebuf_n;

  const int32_t count = full ? n : (st.use_own ? st.ctrl->own_count : st.ctrl->work_count);
  const uint32_t* __restrict__ items = st.use_own ? st.items_own : st.items;
  const int32_t stages = count > static_cast<int32_t>(blockIdx.x)
                             ? (count - static_cast<int32_t>(blockIdx.x) + gridDim.x - 1) / gridDim.x
                             : 0;
  const int32_t nchunks = (n + C - 1) / C;
  const int parity_out = st.ctrl->parity;

  if (tid == 0) {
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    for (int k = 0; k < kBigSlots; ++k) {
      mbar_init(&slot_full[k], 1);
      mbar_init(&slot_empty[k], 1);
      slot_done[k] = 0;
    }
    item_done = 0;
    ebuf_n = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto item_of = [&](int32_t q) -> ResInfo {
    ResInfo it;
    const int32_t idx = static_cast<int32_t>(blockIdx.x) + q * static_cast<int32_t>(gridDim.x);
    const uint32_t w = full ? (static_cast<uint32_t>(idx) | kItemAgent | kItemJob) : items[idx];
    it.agent = static_cast<int32_t>(w & kItemMask);
    it.job = tau_g[it.agent];
    it.flags = w & (kItemAgent | kItemJob);
    it.pad = 0;
    it.sv = static_cast<double>(widen(acur_g[it.agent]));
    return it;
  };

  if (warp == NW + 1) {
    // ---------------- A-row producer ----------------
    if (lane == 0) {
      ResInfo nxt = stages > 0 ? item_of(0) : ResInfo{};
      for (int32_t q = 0; q < stages; ++q) {
        const ResInfo cur = nxt;
        if (q + 1 < stages) nxt = item_of(q + 1);
        if (q >= 1) mbar_wait_backoff(a_empty, static_cast<uint32_t>((q - 1) & 1), 32);
        info_s = cur;
        __threadfence_block();
        mbar_expect_tx(a_full, static_cast<uint32_t>(row_bytes));
        bulk_g2s(a_s, A + static_cast<int64_t>(cur.agent) * ld, static_cast<uint32_t>(row_bytes), a_full);
        if (q + 1 < stages) l2_prefetch(A + static_cast<int64_t>(nxt.agent) * ld, static_cast<uint32_t>(row_bytes));
      }
    }
  } else if (warp == NW) {
    // ---------------- chunk-ring producer ----------------
    ResInfo it{};
    int64_t g = 0;  // global chunk sequence number -> slot g % R, use g / R
    for (int32_t q = 0; q < stages; ++q) {
      if (lane == 0) it = item_of(q);
      const int32_t job = __shfl_sync(0xffffffffu, it.job, 0);
      for (int32_t c = 0; c < nchunks; ++c, ++g) {
        const int s = static_cast<int>(g % kBigSlots);
        if (g >= kBigSlots) mbar_wait_backoff(&slot_empty[s], static_cast<uint32_t>(((g / kBigSlots) - 1) & 1), 32);
        const int32_t p0 = c * C;
        const int32_t len = min(C, static_cast<int32_t>(ld) - p0);
        unsigned char* sb = slots + s * slot_stride;
        if (lane == 0) {
          blk_next[s] = 0;
          __threadfence_block();
          mbar_expect_tx(&slot_full[s], static_cast<uint32_t>(len) * static_cast<uint32_t>(2 * sizeof(E) + 2));
        }
        __syncwarp();
        if (lane == 0)
          bulk_g2s(sb, AT + static_cast<int64_t>(job) * ld + p0, static_cast<uint32_t>(len * sizeof(E)), &slot_full[s]);
        else if (lane == 1)
          bulk_g2s(sb + cb, acur_g + p0, static_cast<uint32_t>(len * sizeof(E)), &slot_full[s]);
        else if (lane == 2)
          bulk_g2s(sb + 2 * cb, tau16_g + p0, static_cast<uint32_t>(len * 2), &slot_full[s]);
        __syncwarp();
      }
    }
  } else {
    // ---------------- consumer warps ----------------
    Track<KM> ta, tj;
    int64_t g = 0;
    for (int32_t q = 0; q < stages; ++q) {
      mbar_wait_backoff(a_full, static_cast<uint32_t>(q & 1), 32);
      const ResInfo im = info_s;
      const Acc s = static_cast<Acc>(im.sv);
      ta.init();
      tj.init();
      for (int32_t c = 0; c < nchunks; ++c, ++g) {
        const int sl = static_cast<int>(g % kBigSlots);
        mbar_wait_backoff(&slot_full[sl], static_cast<uint32_t>((g / kBigSlots) & 1), 32);
        const unsigned char* sb = slots + sl * slot_stride;
        const E* at_c = reinterpret_cast<const E*>(sb);
        const E* ac_c = reinterpret_cast<const E*>(sb + cb);
        const uint16_t* t_c = reinterpret_cast<const uint16_t*>(sb + 2 * cb);
        const int32_t p0 = c * C;
        const int32_t plen = min(C, n - p0);
        const int32_t nblk = (plen + kBlk - 1) / kBlk;
        auto grab = [&]() -> int32_t {
          int32_t k = 0;
          if (lane == 0) k = atomicAdd(&blk_next[sl], 1);
          return __shfl_sync(0xffffffffu, k, 0);
        };
        for (int32_t blk = grab(); blk < nblk;) {
          const int32_t nxt = grab();
          const int32_t li = blk * kBlk + lane * V;  // position within the chunk
          if (li < plen) {
            StreamRegs<E, 1> r;
            lds_tau<E>(t_c + li, r.t);
            r.c = *reinterpret_cast<const uint4*>(ac_c + li);
            r.x[0] = *reinterpret_cast<const uint4*>(at_c + li);
            const Acc sv[1] = {s};
            Track<KM> tav[1] = {ta}, tjv[1] = {tj};
            if (li + V <= plen)
              compute_step<E, 1, KM, false>(r, p0 + li, V, a_s, ld, 0, sv, tav, tjv);
            else
              compute_step<E, 1, KM, false>(r, p0 + li, plen - li, a_s, ld, 0, sv, tav, tjv);
            ta = tav[0];
            tj = tjv[0];
          }
          blk = nxt;
        }
        // the last warp done with this chunk hands the slot back
        __syncwarp();
        int last = 0;
        if (lane == 0) last = atomicAdd(&slot_done[sl], 1) == NW - 1;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          if (lane == 0) {
            slot_done[sl] = 0;
            mbar_arrive(&slot_empty[sl]);
          }
        }
      }
      // item end: warp partials -> last warp -> records, proposal, A release
      ta.warp_reduce();
      tj.warp_reduce();
      if (lane == 0) {
        red[warp * 2] = ta;
        red[warp * 2 + 1] = tj;
      }
      int last = 0;
      if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(&item_done, 1) == NW - 1;
        if (last) item_done = 0;
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (!last) continue;
      __threadfence_block();
      Track<KM> r;
      r.init();
      if (lane < 2)
        for (int w = 0; w < NW; ++w) r.merge(red[w * 2 + lane]);
      const bool ok = lane < 2 && r.valid();
      const double d = ok ? r.delta() : 0.0;
      const int32_t k = ok ? r.index() : -1;
      double acur_a = 0.0;
      if (ok && lane == 0) acur_a = static_cast<double>(a_s[k]);  // A[i][k], before the row is released
      __syncwarp();
      if (lane == 0) mbar_arrive(a_empty);
      const bool active = ok && d > st.eps;
      bool emit = false;
      Prop entry;
      if (lane == 0 && (im.flags & kItemAgent)) {
        st.agent_delta[im.agent] = active ? d : 0.0;
        st.agent_partner[im.agent] = active ? k : -1;
        emit = active && st.emit_edges;
        if (emit) entry = Prop{im.agent, im.agent, -1, k, im.job, 1, d, acur_a, 0.0};
      } else if (lane == 1 && (im.flags & kItemJob)) {
        st.job_delta[im.job] = active ? d : 0.0;
        st.job_partner[im.job] = active ? k : -1;
        emit = active && st.emit_edges;
        if (emit) entry = Prop{n + im.job, k, im.agent, im.job, -1, 2, d, 0.0, 0.0};
      }
      const unsigned mask = __ballot_sync(0xffffffffu, emit);
      if (mask) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&ebuf_n, __popc(mask));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (emit) {
          const int pos = base + __popc(mask & ((1u << lane) - 1));
          if (pos < kBigEdgeBuf) {
            ebuf[pos] = entry;
          } else {
            const int gg = atomicAdd(&st.ctrl->edge_count[parity_out], 1);
            st.edges[parity_out][gg] = finish_prop(entry, st.sigma, tau_g, st.A, st.storage, ld, n);
          }
        }
      }
    }
  }
  __syncthreads();
  const int ne = min(ebuf_n, kBigEdgeBuf);
  __shared__ int gbase;
  if (tid == 0 && ne > 0) gbase = atomicAdd(&st.ctrl->edge_count[parity_out], ne);
  __syncthreads();
  for (int e = tid; e < ne; e += kBigThreads)
    st.edges[parity_out][gbase + e] = finish_prop(ebuf[e], st.sigma, tau_g, st.A, st.storage, ld, n);
}

inline size_t big_smem_bytes(int64_t ld, size_t es, int32_t C) {
  const size_t row = (static_cast<size_t>(ld) * es + 127) / 128 * 128;
  const size_t slot = (static_cast<size_t>(C) * (2 * es + 2) + 127) / 128 * 128;
  return row + kBigSlots * slot + (2 + 2 * kBigSlots) * 8 + kBigWarps * 2 * 16;
}

template <class E, int KM>
cudaError_t launch_big(const DevState& d, const ScanPlan& p, int full, cudaStream_t st) {
  auto k = pair_scan_big_kernel<E, KM>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem));
  if (e != cudaSuccess) return e;
  return launch_pdl(k, dim3(p.ctas), dim3(kBigThreads), p.smem, st, d.pdl, d, full, static_cast<int32_t>(p.chunk));
}

}  // namespace scan_detail

template <class E, int KM>
cudaError_t launch_scan_big_typed(const DevState& d, const ScanPlan& p, int full, cudaStream_t st) {
  return scan_detail::launch_big<E, KM>(d, p, full, st);
}

}  // namespace lsapgpu
