// scan_cluster.cuh -- the pair scan for rows too long to stage on one SM
// (C4: n = 30000 fp32, 120 KB rows; C5: n = 100000, 400 KB rows).
//
// Same work item and arithmetic as the other scan kernels (scan_kernel.cuh):
// item = agent i with its job j0 = tau[i]; candidates over i' with
// t = tau[i'], x = AT[j0][i'], g = A[i][t], c = acur[i'] give agent i's record
// ((g - s) + (x - c), tie index t) and job j0's record ((x - s) + (g - c),
// tie index i') -- kernels_scalar.cpp:6-25, solver_state.hpp:78-92.
//
// Measured result (B200, C4): 4x slower than the streaming kernel -- random
// gathers through distributed shared memory cost ~1 us each under load -- so
// the plan uses it only on request (LSAPGPU_SCAN_CLUSTER=N).
//
// A thread-block cluster of CS CTAs (one per SM) scans ONE item per stage.
// CTA r owns the column slice [r*L, r*L + L) of the item's rows: its stage
// buffer receives A[i][slice] and AT[j0][slice] by TMA, and it scans the
// positions i' of its slice (tau / acur of the slice stay resident for the
// launch).  The gather g = A[i][t] reads the slice of the CTA that owns t
// through distributed shared memory (mapa + ld.shared::cluster).  With the
// row split CS ways every CTA double-buffers its slices, so the next item's
// rows stream in while this one is scanned -- the single-SM kernel could only
// single-buffer a 120 KB row and had to re-scan every position per chunk for
// a 400 KB one.
//
// Cross-CTA protocol (mbarriers, remote arrives; no cluster-wide barrier in
// the steady state):
//   full[b]   local: this CTA's slices of the stage landed (TMA complete_tx)
//   ready[b]  count CS: every CTA's slices of the stage landed (each CTA's
//             warp 0 arrives remotely on all ranks once its full[b] passed)
//   empty[b]  count CS: every CTA finished scanning the stage, so nobody
//             reads this CTA's buffer b any more (producer refills after it)
//   part[b]   rank 0 only, count CS: every CTA's partial records arrived
// Rank 0 merges the CS partials, writes the records and emits the proposal.
//
// Algorithmic HBM bytes: 2 * n * sizeof(elem) per item, as for every scan.
#pragma once

#include "scan_resident.cuh"

namespace lsapgpu {
namespace scan_detail {

constexpr int kClThreads = 512;  // 15 consumer warps + 1 producer warp
constexpr int kClWarps = kClThreads / 32 - 1;
constexpr int kClEdgeBuf = 256;

__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
template <class E>
__device__ __forceinline__ E ld_cluster(uint32_t caddr) {
  if constexpr (sizeof(E) == 2) {
    uint16_t v;
    asm volatile("ld.shared::cluster.u16 %0, [%1];" : "=h"(v) : "r"(caddr));
    return static_cast<E>(static_cast<int16_t>(v));
  } else if constexpr (sizeof(E) == 4) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(caddr));
    E e;
    memcpy(&e, &v, 4);
    return e;
  } else {
    unsigned long long v;
    asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(caddr));
    E e;
    memcpy(&e, &v, 8);
    return e;
  }
}
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* local_bar, uint32_t rank) {
  const uint32_t c = mapa_rank(smem_u32(local_bar), rank);
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "LAB_WAIT_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// One vector step of candidates for the single item of a stage.
template <class E, int KM, class Gather>
__device__ __forceinline__ void cl_step(const int32_t (&t)[16 / sizeof(E)], const uint4& cw, const uint4& xw,
                                        int32_t i0, int nvalid, typename Traits<E>::Acc s, Gather gather,
                                        Track<KM>& ta, Track<KM>& tj) {
  using Acc = typename Traits<E>::Acc;
  constexpr int V = 16 / sizeof(E);
#pragma unroll
  for (int v = 0; v < V; ++v) {
    if (v >= nvalid) break;
    const int32_t ip = i0 + v;
    const Acc c = vget<E>(cw, v);
    const Acc x = vget<E>(xw, v);
    const Acc g = static_cast<Acc>(gather(t[v]));
    if constexpr (KM == kPacked32) {
      const uint32_t u = static_cast<uint32_t>(g + x - s - c + kOff32) * 16384u;
      ta.k = max(ta.k, u + 16383u - static_cast<uint32_t>(t[v]));
      tj.k = max(tj.k, u + 16383u - static_cast<uint32_t>(ip));
    } else if constexpr (KM == kPacked64) {
      const int32_t d = (g - s) + (x - c);
      ta.add(d, t[v]);
      tj.add(d, ip);
    } else {
      ta.add(delta4(g, s, x, c), t[v]);  // agent: (g - s) + (x - c)
      tj.add(delta4(x, s, g, c), ip);    // job:   (x - s) + (g - c)
    }
  }
}

// smem: tau slice (int32, L) | acur slice (L) | stages [2] x (A slice, AT slice) |
//       full[2], ready[2], empty[2], part[2], res mbarriers | red[2][NW][2] | cparts[2][CS][2]
template <class E, int KM, int CS>
__global__ void __launch_bounds__(kClThreads, 1)
    pair_scan_cl_kernel(DevState st, int full, int32_t L, uint32_t magic) {
  using Acc = typename Traits<E>::Acc;
  constexpr int V = 16 / sizeof(E);
  constexpr int NW = kClWarps;
  constexpr int32_t kBlk = 32 * V;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int32_t n = st.n;
  const int64_t ld = st.ld;
  const E* __restrict__ A = static_cast<const E*>(st.A);
  const E* __restrict__ AT = static_cast<const E*>(st.AT);
  const E* __restrict__ acur_g = static_cast<const E*>(st.acur);
  const int32_t* __restrict__ tau_g = st.tau;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  pdl_trigger();
  pdl_wait();
  if (blockIdx.x == 0 && tid == 0) tl_mark(st.ctrl, st.tl, st.tl_cap, full ? kTlScanFull : kTlScan);

  // this CTA's column / position slice
  const int32_t lo = static_cast<int32_t>(rank) * L;
  const int64_t rem = ld - lo;
  const int32_t Lr = rem <= 0 ? 0 : (rem < L ? static_cast<int32_t>(rem) : L);  // elements staged
  const int32_t hi = min(n, lo + L);                                                                   // positions scanned
  const size_t slice_bytes = static_cast<size_t>(L) * sizeof(E);
  const size_t stage_bytes = 2 * ((slice_bytes + 127) / 128 * 128);
  int32_t* tau_s = reinterpret_cast<int32_t*>(smem_raw);
  E* acur_s = reinterpret_cast<E*>(smem_raw + (static_cast<size_t>(L) * 4 + 127) / 128 * 128);
  unsigned char* stage_base = reinterpret_cast<unsigned char*>(acur_s) + (slice_bytes + 127) / 128 * 128;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stage_base + 2 * stage_bytes);
  uint64_t* ready_bar = full_bar + 2;
  uint64_t* empty_bar = full_bar + 4;
  uint64_t* part_bar = full_bar + 6;
  uint64_t* res_bar = full_bar + 8;
  Track<KM>* red = reinterpret_cast<Track<KM>*>(full_bar + 10);  // [2][NW][2]
  Track<KM>* cparts = red + 2 * NW * 2;                          // [2][CS][2] (rank 0)
  __shared__ ResInfo info_s[2];
  __shared__ int arrive_cnt[2];
  __shared__ int blk_next[2];
  __shared__ Prop ebuf[kClEdgeBuf];
  __shared__ int ebuf_n;

  const int32_t count = full ? n : (st.use_own ? st.ctrl->own_count : st.ctrl->work_count);
  const uint32_t* __restrict__ items = st.use_own ? st.items_own : st.items;
  const int32_t nclusters = static_cast<int32_t>(gridDim.x) / CS;
  const int32_t cid = static_cast<int32_t>(blockIdx.x) / CS;
  const int32_t stages = count > cid ? (count - cid + nclusters - 1) / nclusters : 0;
  const int parity_out = st.ctrl->parity;

  if (tid == 0) {
    for (int k = 0; k < 2; ++k) {
      mbar_init(&full_bar[k], 1);
      mbar_init(&ready_bar[k], CS);
      mbar_init(&empty_bar[k], CS);
      mbar_init(&part_bar[k], CS);
      arrive_cnt[k] = 0;
    }
    mbar_init(res_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    ebuf_n = 0;
  }
  cluster_sync_all();  // every CTA's barriers exist before any remote arrive

  if (stages > 0) {
    if (warp == NW) {
      // ---------------- producer warp ----------------
      if (lane == 0) {  // resident tau / acur of this slice
        const uint32_t tb = static_cast<uint32_t>(static_cast<size_t>(Lr) * 4);
        const uint32_t cb = static_cast<uint32_t>(static_cast<size_t>(Lr) * sizeof(E));
        mbar_expect_tx(res_bar, tb + cb);
        bulk_g2s(tau_s, tau_g + lo, tb, res_bar);
        bulk_g2s(acur_s, acur_g + lo, cb, res_bar);
      }
      for (int32_t q = 0; q < stages; ++q) {
        const int b = q & 1;
        if (q >= 2) mbar_wait_cluster(&empty_bar[b], static_cast<uint32_t>(((q >> 1) - 1) & 1));
        if (lane == 0) {
          const int32_t idx = cid + q * nclusters;
          ResInfo it;
          const uint32_t w = full ? (static_cast<uint32_t>(idx) | kItemAgent | kItemJob) : items[idx];
          it.agent = static_cast<int32_t>(w & kItemMask);
          it.job = tau_g[it.agent];
          it.flags = w & (kItemAgent | kItemJob);
          it.pad = 0;
          it.sv = static_cast<double>(widen(acur_g[it.agent]));
          info_s[b] = it;
          blk_next[b] = 0;
          __threadfence_block();
          const uint32_t bytes = static_cast<uint32_t>(static_cast<size_t>(Lr) * sizeof(E));
          mbar_expect_tx(&full_bar[b], 2 * bytes);
          unsigned char* sb = stage_base + b * stage_bytes;
          bulk_g2s(sb, A + static_cast<int64_t>(it.agent) * ld + lo, bytes, &full_bar[b]);
          bulk_g2s(sb + stage_bytes / 2, AT + static_cast<int64_t>(it.job) * ld + lo, bytes, &full_bar[b]);
        }
        __syncwarp();
      }
    } else {
      // ---------------- consumer warps ----------------
      mbar_wait(res_bar, 0);
      Track<KM> ta, tj;
      for (int32_t q = 0; q < stages; ++q) {
        const int b = q & 1;
        const uint32_t ph = static_cast<uint32_t>((q >> 1) & 1);
        if (warp == 0 && lane == 0) {  // my slices landed: tell every CTA of the cluster
          mbar_wait(&full_bar[b], ph);
          for (uint32_t r = 0; r < static_cast<uint32_t>(CS); ++r) mbar_arrive_remote(&ready_bar[b], r);
        }
        mbar_wait_cluster(&ready_bar[b], ph);
        const ResInfo im = info_s[b];
        const Acc s = static_cast<Acc>(im.sv);
        ta.init();
        tj.init();
        const E* sA = reinterpret_cast<const E*>(stage_base + b * stage_bytes);
        const E* sT = reinterpret_cast<const E*>(stage_base + b * stage_bytes + stage_bytes / 2);
        const uint32_t sA_addr = smem_u32(sA);
        auto gather = [&](int32_t t) -> E {
          uint32_t owner = __umulhi(static_cast<uint32_t>(t), magic);
          int32_t off = t - static_cast<int32_t>(owner) * L;
          if (off < 0) {  // magic = ceil(2^32 / L) can round the quotient up by one
            --owner;
            off += L;
          }
          if (owner == rank) return sA[off];
          return ld_cluster<E>(mapa_rank(sA_addr + static_cast<uint32_t>(off) * sizeof(E), owner));
        };
        const int32_t nblk = (hi - lo + kBlk - 1) / kBlk;
        auto grab = [&]() -> int32_t {
          int32_t k = 0;
          if (lane == 0) k = atomicAdd(&blk_next[b], 1);
          return __shfl_sync(0xffffffffu, k, 0);
        };
        for (int32_t blk = nblk > 0 ? grab() : 0; blk < nblk;) {
          const int32_t nxt = grab();
          const int32_t i0 = lo + blk * kBlk + lane * V;  // global position
          if (i0 < hi) {
            const int32_t li = i0 - lo;
            int32_t t[V];
            if constexpr (V == 8) {
              const int4 a0 = *reinterpret_cast<const int4*>(tau_s + li);
              const int4 a1 = *reinterpret_cast<const int4*>(tau_s + li + 4);
              t[0] = a0.x; t[1] = a0.y; t[2] = a0.z; t[3] = a0.w;
              t[4] = a1.x; t[5] = a1.y; t[6] = a1.z; t[7] = a1.w;
            } else if constexpr (V == 4) {
              const int4 a0 = *reinterpret_cast<const int4*>(tau_s + li);
              t[0] = a0.x; t[1] = a0.y; t[2] = a0.z; t[3] = a0.w;
            } else {
              const int2 a0 = *reinterpret_cast<const int2*>(tau_s + li);
              t[0] = a0.x; t[1] = a0.y;
            }
            const uint4 cw = *reinterpret_cast<const uint4*>(acur_s + li);
            const uint4 xw = *reinterpret_cast<const uint4*>(sT + li);
            if (i0 + V <= hi)
              cl_step<E, KM>(t, cw, xw, i0, V, s, gather, ta, tj);
            else
              cl_step<E, KM>(t, cw, xw, i0, hi - i0, s, gather, ta, tj);
          }
          blk = nxt;
        }
        // CTA partials: warp -> last warp of this CTA -> rank 0
        ta.warp_reduce();
        tj.warp_reduce();
        Track<KM>* rq = red + b * NW * 2;
        if (lane == 0) {
          rq[warp * 2] = ta;
          rq[warp * 2 + 1] = tj;
        }
        int last = 0;
        if (lane == 0) {
          __threadfence_block();
          last = atomicAdd(&arrive_cnt[b], 1) == NW - 1;
          if (last) arrive_cnt[b] = 0;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (!last) continue;
        __threadfence_block();
        Track<KM> r;
        r.init();
        if (lane < 2)
          for (int w = 0; w < NW; ++w) r.merge(rq[w * 2 + lane]);
        if (lane < 2) {  // publish to rank 0's cparts[b][rank][side]
          Track<KM>* dst = cparts + (b * CS + static_cast<int>(rank)) * 2 + lane;
          const uint32_t caddr = mapa_rank(smem_u32(dst), 0);
          if constexpr (KM == kFloat) {
            asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(caddr), "d"(r.d) : "memory");
            asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(caddr + 8), "r"(r.i) : "memory");
          } else if constexpr (KM == kPacked64) {
            asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(caddr), "l"(r.k) : "memory");
          } else {
            asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(caddr), "r"(r.k) : "memory");
          }
          asm volatile("fence.acq_rel.cluster;" ::: "memory");
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&part_bar[b], 0);  // release: the stores above are visible
        if (rank != 0) {
          __syncwarp();
          if (lane < CS) mbar_arrive_remote(&empty_bar[b], static_cast<uint32_t>(lane));
          continue;
        }
        // ---- rank 0: merge the CS partials, write the records, emit ----
        mbar_wait_cluster(&part_bar[b], ph);
        Track<KM> c;
        c.init();
        if (lane < 2)
          for (int r2 = 0; r2 < CS; ++r2) c.merge(cparts[(b * CS + r2) * 2 + lane]);
        __syncwarp();
        if (lane < CS) mbar_arrive_remote(&empty_bar[b], static_cast<uint32_t>(lane));  // cparts[b] consumed
        const bool ok = lane < 2 && c.valid();
        const double d = ok ? c.delta() : 0.0;
        const int32_t k = ok ? c.index() : -1;
        const bool active = ok && d > st.eps;
        bool emit = false;
        Prop entry;
        if (lane == 0 && (im.flags & kItemAgent)) {
          st.agent_delta[im.agent] = active ? d : 0.0;
          st.agent_partner[im.agent] = active ? k : -1;
          emit = active && st.emit_edges;
          if (emit) entry = Prop{im.agent, im.agent, -1, k, im.job, 2, d, 0.0, 0.0};
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
            if (pos < kClEdgeBuf) {
              ebuf[pos] = entry;
            } else {
              const int g = atomicAdd(&st.ctrl->edge_count[parity_out], 1);
              st.edges[parity_out][g] = finish_prop(entry, st.sigma, tau_g, st.A, st.storage, ld, n);
            }
          }
        }
      }
    }
  }
  // flush rank 0's buffered proposals; keep every CTA alive until no peer can
  // touch its shared memory
  __syncthreads();
  const int ne = min(ebuf_n, kClEdgeBuf);
  __shared__ int gbase;
  if (tid == 0 && ne > 0) gbase = atomicAdd(&st.ctrl->edge_count[parity_out], ne);
  __syncthreads();
  for (int e = tid; e < ne; e += kClThreads)
    st.edges[parity_out][gbase + e] = finish_prop(ebuf[e], st.sigma, tau_g, st.A, st.storage, ld, n);
  cluster_sync_all();
}

// Dynamic smem of the cluster kernel for a slice of L elements.
inline size_t cl_smem_bytes(int32_t L, size_t es, int CS) {
  const size_t slice = (static_cast<size_t>(L) * es + 127) / 128 * 128;
  const size_t tau = (static_cast<size_t>(L) * 4 + 127) / 128 * 128;
  return tau + slice + 2 * 2 * slice + 10 * 8 + 2 * kClWarps * 2 * 16 + 2 * CS * 2 * 16;
}

template <class E, int KM, int CS>
cudaError_t launch_cl_t(const DevState& d, const ScanPlan& p, int full, cudaStream_t st) {
  auto k = pair_scan_cl_kernel<E, KM, CS>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem));
  if (e != cudaSuccess) return e;
  if (CS > 8) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  const int32_t L = static_cast<int32_t>(p.chunk);
  const uint32_t magic = static_cast<uint32_t>((0x100000000ull + L - 1) / L);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.ctas);
  cfg.blockDim = dim3(kClThreads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = d.pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, k, d, full, L, magic);
}

template <class E, int KM>
cudaError_t launch_cl(const DevState& d, const ScanPlan& p, int full, cudaStream_t st) {
  switch (p.cluster) {
    case 2: return launch_cl_t<E, KM, 2>(d, p, full, st);
    case 4: return launch_cl_t<E, KM, 4>(d, p, full, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace scan_detail

template <class E, int KM>
cudaError_t launch_scan_cl_typed(const DevState& d, const ScanPlan& p, int full, cudaStream_t st) {
  return scan_detail::launch_cl<E, KM>(d, p, full, st);
}

}  // namespace lsapgpu
