#pragma once
// scan_filter.cuh -- the pair scan for long rows (n beyond what the resident
// kernel holds on chip: C4 n = 30000, C5 n = 100000), computing the same
// records as every other scan kernel (kernels_scalar.cpp:6-25,
// kernels_avx2.cpp:40-92, solver_state.hpp:78-104) with a quantized filter
// and an exact verification step.
//
// Work item: agent i with its job j0 = tau[i]; over every position p with
// t = tau[p], g = A[i][t], x = AT[j0][p], c = acur[p], s = acur[i]:
//   agent candidate (g - s) + (x - c), tie index t
//   job   candidate (x - s) + (g - c), tie index p
// in fp64, maximum with the smallest index on ties, active iff > eps.
//
// Filter.  Both candidates are roundings of the same real D = g + x - c - s.
// With a power-of-two scale S (max |a| * S <= 16383 for 16-bit, 127 for
// 8-bit) the layout keeps Q = ceil(A * S) and QT = ceil(AT * S), and the
// per-launch position array aux[p] = tau[p] sizeof(Q) | (floor(acur[p] * S) + 2^14) << 17.
// U = Q[i][t] + QT[j0][p] - floor(c * S) is an integer with
//   (g + x - c) S  <=  U  <  (g + x - c) S + 3.
// A position can be discarded without changing either record when
//   * U < floor((s + eps) S) - 1: then D < eps - 1/S, so neither candidate
//     is active (the fp64 rounding of D is far below 1/S), or
//   * U < U_r - 4 for another position r: then D_r - D_p > 2/S, so r beats p
//     strictly on both sides (no tie either).
// Everything else goes to a per-item queue and is evaluated EXACTLY (fp64,
// the reference's operation order) from the fp32 A / AT / acur in HBM, so
// the records are bit-identical to the unfiltered scans'.  On uniform data
// a few dozen of n positions survive per item; a queue overflow (adversarial
// ties) falls back to an exact scan of the whole item.
//
// Data movement per item: the Q row (gathered at random t: staged in shared
// memory by TMA) and the QT row (streamed through a ring of TMA chunk slots)
// -- 2 n sizeof(Q) bytes of HBM instead of 2 n sizeof(float) -- plus aux[]
// (4 n bytes, shared by every item of the launch), which each CTA copies
// into its tensor memory once per launch (the first 16 chunks; the rest, for
// n > 65536, is loaded from L2 straight into registers: through shared
// memory it cost as much smem bandwidth as the gather).  Row buffers are
// double-buffered where two fit.
//
// Warps: 16 consumers (each takes one 256-position block of every chunk),
// one row producer, one chunk producer, one verifier that evaluates item q's
// queue while the consumers scan item q + 1.
#include "scan_resident.cuh"

namespace lsapgpu {
namespace scan_detail {

constexpr int kFW = 16;                     // consumer warps
constexpr int kFV = 8;                      // positions per lane per block
constexpr int kFBlk = 32 * kFV;             // 256 positions per warp block
constexpr int32_t kFChunk = kFW * kFBlk;    // 4096 positions per chunk (one block per consumer warp)
constexpr int kFThreads = 32 * (kFW + 3);   // + row producer, chunk producer, verifier
constexpr int kFQueueMax = 1024;            // candidates per item (two item parities) at most
constexpr int kFMaxSlots = 8;
constexpr int kFEdgeBuf = 128;
constexpr int32_t kAuxBias = 16384;         // bias of the 15-bit floor(c S) field
constexpr int32_t kFNeg = -(1 << 24);       // below every U

struct FInfo {
  int32_t agent;
  int32_t job;
  uint32_t flags;
  int32_t t0;  // eps gate in biased U units
  double sv;   // acur[agent]
};

template <class Q>
__device__ __forceinline__ int32_t q_elem(const uint4& w, int v) {
  if constexpr (sizeof(Q) == 2) {
    const uint32_t x = (&w.x)[v >> 1];
    return (v & 1) ? (static_cast<int32_t>(x) >> 16) : static_cast<int32_t>(static_cast<int16_t>(x & 0xFFFFu));
  } else {
    const uint32_t x = (&w.x)[v >> 2];
    return static_cast<int32_t>(x << (24 - 8 * (v & 3))) >> 24;
  }
}

// mbarrier arrive that cannot be issued before `dep` is computed (the value
// is an asm operand): used to release a buffer only after loads from it have
// been consumed.
__device__ __forceinline__ void mbar_arrive_after(uint64_t* bar, uint32_t dep) {
  asm volatile(
      "{\n .reg .b32 d;\n mov.b32 d, %1;\n mbarrier.arrive.shared::cta.b64 _, [%0];\n}" ::"r"(smem_u32(bar)),
      "r"(dep)
      : "memory");
}

// Tensor memory (TMEM) holding the launch's aux[] words: consumer warp w
// keeps the words of its positions in TMEM lane quarter w % 4, columns
// (w / 4) * ntm * V + c * V .. + V - 1 for chunk c < ntm = min(chunks, 16)
// (512 columns), and reads a chunk's V words with one 32x32b load instead of
// V / 4 L2 loads per item; chunks beyond the first 16 (n > 65536) still come
// from L2.
__device__ __forceinline__ void tmem_alloc512(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(dst_smem))
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc512(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&w)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&w)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ int32_t eps_gate(double sv, double eps, double S) {
  const double r = floor((sv + eps) * S);
  if (!(r < 1e9)) return 1 << 24;  // (also NaN-safe) nothing can be active
  if (r < -1e9) return kFNeg;
  return static_cast<int32_t>(r) - 1 - kAuxBias;
}

// smem: rows [RB][ld] Q | slots [NS] x QT chunk [C] Q | queue [2][qcap] u64 |
//       row_full[RB], slot_full[NS], slot_empty[NS], item_done[2], queue_free[2] mbarriers
// W consumer warps of V positions per lane: a chunk is W * 32 * V positions.
template <int V>
struct AuxW {
  uint32_t w[V];
};
template <int V>
__device__ __forceinline__ void ld_aux(AuxW<V>& a, const uint32_t* p, bool ok) {
#pragma unroll
  for (int k = 0; k < V / 4; ++k) {
    const uint4 x = ok ? __ldcg(reinterpret_cast<const uint4*>(p) + k) : make_uint4(0u, 0u, 0u, 0u);
    a.w[4 * k] = x.x;
    a.w[4 * k + 1] = x.y;
    a.w[4 * k + 2] = x.z;
    a.w[4 * k + 3] = x.w;
  }
}
// V consecutive Q elements of a staged QT chunk, as the first V*sizeof(Q) bytes of a uint4
template <class Q, int V>
__device__ __forceinline__ uint4 lds_q(const unsigned char* p) {
  constexpr int kBytes = V * static_cast<int>(sizeof(Q));
  if constexpr (kBytes == 16) {
    return *reinterpret_cast<const uint4*>(p);
  } else if constexpr (kBytes == 8) {
    const uint2 h = *reinterpret_cast<const uint2*>(p);
    return make_uint4(h.x, h.y, 0u, 0u);
  } else {
    return make_uint4(*reinterpret_cast<const uint32_t*>(p), 0u, 0u, 0u);
  }
}

// kAux: 0 = aux[] from L2, 1 = the first 16 chunks from TMEM and the rest
// from L2, 2 = every chunk from TMEM (n <= 65536: no L2 lookahead code at all)
template <class E, class Q, int RB, int W, int V, int kAux>
__global__ void __launch_bounds__(32 * (W + 3), 1)
    pair_scan_filter_kernel(DevState st, int full, int NS, int qcap) {
  constexpr bool kTM = kAux > 0, kAllTM = kAux == 2;
  static_assert(!kTM || V == 8, "TMEM aux: 8 words per lane per chunk");
  // the geometry of this instantiation (shadowing the default constants)
  constexpr int kFW = W;
  constexpr int kFV = V;
  constexpr int kFBlk = 32 * V;
  constexpr int32_t kFChunk = W * 32 * V;
  constexpr int kFThreads = 32 * (W + 3);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int32_t n = st.n;
  const int64_t ld = st.ld;
  // this rank's row blocks of Q and A (row-block placement; single GPU: all rows)
  const Q* __restrict__ Qg = static_cast<const Q*>(st.Q) - static_cast<int64_t>(st.a_row0) * st.ld;
  const Q* __restrict__ QTg = static_cast<const Q*>(st.QT);
  const uint32_t* __restrict__ aux_g = st.aux;
  const E* __restrict__ A = static_cast<const E*>(st.A) - static_cast<int64_t>(st.a_row0) * st.ld;
  const E* __restrict__ AT = static_cast<const E*>(st.AT);
  const E* __restrict__ acur_g = static_cast<const E*>(st.acur);
  const int32_t* __restrict__ tau_g = st.tau;
  const double S = st.qscale;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  pdl_trigger();
  pdl_wait();  // the aux build (and the commit / apply before it) wrote what this scan reads
  if (blockIdx.x == 0 && tid == 0) tl_mark(st.ctrl, st.tl, st.tl_cap, full ? kTlScanFull : kTlScan);

  const int32_t count = full ? n : (st.use_own ? st.ctrl->own_count : st.ctrl->work_count);
  const uint32_t* __restrict__ items = st.use_own ? st.items_own : st.items;
  const int32_t stages = count > static_cast<int32_t>(blockIdx.x)
                             ? (count - static_cast<int32_t>(blockIdx.x) + gridDim.x - 1) / gridDim.x
                             : 0;
  if (stages == 0) return;
  const int32_t nch = static_cast<int32_t>((n + kFChunk - 1) / kFChunk);
  const int parity_out = st.ctrl->parity;

  const size_t row_bytes = (static_cast<size_t>(ld) * sizeof(Q) + 127) / 128 * 128;
  constexpr size_t kSlotBytes = static_cast<size_t>(kFChunk) * sizeof(Q);
  Q* rows = reinterpret_cast<Q*>(smem_raw);
  unsigned char* slots = smem_raw + RB * row_bytes;
  unsigned long long* queue = reinterpret_cast<unsigned long long*>(slots + NS * kSlotBytes);  // [2][qcap]
  uint64_t* bars = reinterpret_cast<uint64_t*>(queue + 2 * qcap);
  uint64_t* row_full = bars;
  uint64_t* slot_full = bars + RB;
  uint64_t* slot_empty = slot_full + kFMaxSlots;
  uint64_t* item_done = slot_empty + kFMaxSlots;
  uint64_t* queue_free = item_done + 2;
  __shared__ FInfo info_s[RB];
  __shared__ FInfo vinfo[4];  // the verifier's copy (item q in q & 3)
  __shared__ int qn[2];
  __shared__ int tmax[2];
  __shared__ Prop ebuf[kFEdgeBuf];
  __shared__ int ebuf_n;

  if (tid == 0) {
    for (int k = 0; k < RB; ++k) mbar_init(&row_full[k], 1);
    for (int k = 0; k < NS; ++k) {
      mbar_init(&slot_full[k], 1);
      mbar_init(&slot_empty[k], kFW);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&item_done[k], kFW * 32);  // every consumer lane arrives (its own queue stores released)
      mbar_init(&queue_free[k], 1);
      qn[k] = 0;
      tmax[k] = kFNeg;
    }
    ebuf_n = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __shared__ uint32_t tmem_base_s;
  if constexpr (kTM) {
    if (warp == 0) tmem_alloc512(&tmem_base_s);  // one CTA per SM: the whole TMEM
    tmem_fence_before();
  }
  __syncthreads();
  uint32_t tmem_base = 0;
  const int32_t ntm = kTM ? min(nch, 512 / (4 * kFV)) : 0;  // chunks whose aux lives in TMEM
  if constexpr (kTM) {
    tmem_fence_after();
    tmem_base = tmem_base_s;
    if (warp < kFW) {  // each consumer warp stores the aux words of its own positions, every chunk
      const int32_t lo0 = warp * kFBlk + lane * kFV;
      const uint32_t tw = tmem_base + (static_cast<uint32_t>(32 * (warp & 3)) << 16) +
                          static_cast<uint32_t>((warp >> 2) * ntm * kFV);
      for (int32_t c = 0; c < ntm; ++c) {
        const int64_t p = static_cast<int64_t>(c) * kFChunk + lo0;
        AuxW<kFV> x;
        ld_aux<kFV>(x, aux_g + p, p < n);
        tmem_st8(tw + static_cast<uint32_t>(c * kFV), x.w);
      }
      tmem_wait_st();
    }
  }

  auto item_of = [&](int32_t q) -> FInfo {
    FInfo it;
    const int32_t idx = static_cast<int32_t>(blockIdx.x) + q * static_cast<int32_t>(gridDim.x);
    const uint32_t w = full ? (static_cast<uint32_t>(idx) | kItemAgent | kItemJob) : items[idx];
    it.agent = static_cast<int32_t>(w & kItemMask);
    it.job = tau_g[it.agent];
    it.flags = w & (kItemAgent | kItemJob);
    it.sv = static_cast<double>(acur_g[it.agent]);
    it.t0 = eps_gate(it.sv, st.eps, S);
    return it;
  };

  if (warp == kFW) {
    // ---------------- row producer: Q[i,:] of item q into row buffer q % RB ----------------
    // (8 KB pieces, one per lane: a lane issues its bulk copies one after another
    // at ~0.2 us each, so several lanes keep a row's copies in flight together;
    // B200 TMA from HBM: 3.1 TB/s issued from one lane, 6.8 TB/s from four)
    FInfo nxt = item_of(0);
    const uint32_t rbytes = static_cast<uint32_t>(ld * sizeof(Q));
    constexpr uint32_t kPiece = 8192;
    const int pieces = static_cast<int>((rbytes + kPiece - 1) / kPiece);
    for (int32_t q = 0; q < stages; ++q) {
      const FInfo cur = nxt;
      const int rb = q % RB;
      if (q >= RB) mbar_wait_backoff(&item_done[(q - RB) & 1], static_cast<uint32_t>(((q - RB) >> 1) & 1), 64);
      if (lane == 0) {
        info_s[rb] = cur;
        vinfo[q & 3] = cur;
        mbar_expect_tx(&row_full[rb], rbytes);
      }
      __syncwarp();
      for (int pc = lane; pc < pieces; pc += 32) {
        const uint32_t off = static_cast<uint32_t>(pc) * kPiece;
        const uint32_t sz = (rbytes - off) < kPiece ? (rbytes - off) : kPiece;
        bulk_g2s(reinterpret_cast<unsigned char*>(rows) + rb * row_bytes + off,
                 reinterpret_cast<const unsigned char*>(Qg + static_cast<int64_t>(cur.agent) * ld) + off, sz,
                 &row_full[rb]);
      }
      if (q + 1 < stages) {
        nxt = item_of(q + 1);
        // one row buffer: pull the next row into L2 now, so its (exposed)
        // staging copy after this item streams from L2 rather than HBM
        if (RB == 1)
          for (int pc = lane; pc < pieces; pc += 32) {
            const uint32_t off = static_cast<uint32_t>(pc) * kPiece;
            l2_prefetch(reinterpret_cast<const unsigned char*>(Qg + static_cast<int64_t>(nxt.agent) * ld) + off,
                        (rbytes - off) < kPiece ? (rbytes - off) : kPiece);
          }
      }
    }
  } else if (warp == kFW + 1) {
    // ---------------- chunk producer: QT chunk c of item q into the slot ring ----------------
    int s = 0;
    uint32_t eph = 0;   // parity of the slot_empty phase to wait for
    bool wrapped = false;
    int32_t job_next = item_of(0).job;
    for (int32_t q = 0; q < stages; ++q) {
      const int32_t job = job_next;
      if (q + 1 < stages) job_next = item_of(q + 1).job;
      for (int32_t c = 0; c < nch; ++c) {
        if (wrapped) mbar_wait_backoff(&slot_empty[s], eph, 32);
        const int64_t p0 = static_cast<int64_t>(c) * kFChunk;
        const uint32_t len = static_cast<uint32_t>((ld - p0) < kFChunk ? (ld - p0) : kFChunk);
        const uint32_t qbytes = len * static_cast<uint32_t>(sizeof(Q));
        constexpr uint32_t kP = 4096;
        const uint32_t nq = (qbytes + kP - 1) / kP;
        if (lane == 0) mbar_expect_tx(&slot_full[s], qbytes);
        __syncwarp();
        if (static_cast<uint32_t>(lane) < nq) {
          const uint32_t off = lane * kP;
          bulk_g2s(slots + s * kSlotBytes + off,
                   reinterpret_cast<const unsigned char*>(QTg + static_cast<int64_t>(job) * ld + p0) + off,
                   min(kP, qbytes - off), &slot_full[s]);
        }
        __syncwarp();
        if (++s == NS) {
          s = 0;
          if (wrapped) eph ^= 1u;
          wrapped = true;
        }
      }
    }
  } else if (warp == kFW + 2) {
    // ---------------- verifier: exact records of item q from its queue ----------------
    long long kept = 0, overflows = 0;
    for (int32_t q = 0; q < stages; ++q) {
      const int par = q & 1;
      mbar_wait_backoff(&item_done[par], static_cast<uint32_t>((q >> 1) & 1), 64);
      const FInfo im = vinfo[q & 3];
      const int cnt = qn[par];
      kept += cnt;
      const double s = im.sv;
      const E* arow = A + static_cast<int64_t>(im.agent) * ld;
      const E* xrow = AT + static_cast<int64_t>(im.job) * ld;
      Track<kFloat> ta, tj;
      ta.init();
      tj.init();
      if (cnt <= qcap) {
        // four entries per lane per round, every global load of a round in
        // flight together (the entries are random positions: one HBM round
        // trip per round instead of one per entry)
        for (int e0 = 0; e0 < cnt; e0 += 128) {
          int32_t pp[4], tt[4];
          E gg[4], xx[4], cc[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * 32 + lane;
            const unsigned long long ent = e < cnt ? queue[par * qcap + e] : 0ull;
            pp[u] = static_cast<int32_t>(ent & 0xFFFFFFFFull);
            tt[u] = e < cnt ? static_cast<int32_t>(ent >> 32) : -1;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const bool ok = tt[u] >= 0;
            gg[u] = ok ? arow[tt[u]] : E(0);
            xx[u] = ok ? xrow[pp[u]] : E(0);
            cc[u] = ok ? acur_g[pp[u]] : E(0);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (tt[u] < 0) continue;
            const double gv = static_cast<double>(gg[u]), xv = static_cast<double>(xx[u]),
                         cv = static_cast<double>(cc[u]);
            ta.add(delta4(gv, s, xv, cv), tt[u]);
            tj.add(delta4(xv, s, gv, cv), pp[u]);
          }
        }
      } else {  // queue overflow (heavy ties): exact scan of the whole item
        ++overflows;
        for (int32_t p = lane; p < n; p += 32) {
          const int32_t t = tau_g[p];
          const double gv = static_cast<double>(arow[t]);
          const double xv = static_cast<double>(xrow[p]);
          const double cv = static_cast<double>(acur_g[p]);
          ta.add(delta4(gv, s, xv, cv), t);
          tj.add(delta4(xv, s, gv, cv), p);
        }
      }
      ta.warp_reduce();
      tj.warp_reduce();
      if (st.filter_check > 0 && (q % st.filter_check) == 0) {
        // diagnostics: the same item unfiltered; any difference is recorded
        Track<kFloat> ua, uj;
        ua.init();
        uj.init();
        for (int32_t p = lane; p < n; p += 32) {
          const int32_t t = tau_g[p];
          const double gv = static_cast<double>(arow[t]);
          const double xv = static_cast<double>(xrow[p]);
          const double cv = static_cast<double>(acur_g[p]);
          ua.add(delta4(gv, s, xv, cv), t);
          uj.add(delta4(xv, s, gv, cv), p);
        }
        ua.warp_reduce();
        uj.warp_reduce();
        if (lane == 0) {
          for (int side = 0; side < 2; ++side) {
            const Track<kFloat>& w = side ? uj : ua;
            const Track<kFloat>& f = side ? tj : ta;
            const bool wa = w.valid() && w.delta() > st.eps, fa = f.valid() && f.delta() > st.eps;
            const bool same = wa == fa && (!wa || (w.delta() == f.delta() && w.index() == f.index()));
            if (!same && atomicAdd(&st.ctrl->fchk_mismatch, 1) == 0) {
              st.ctrl->fchk_item = side ? im.job : im.agent;
              st.ctrl->fchk_cnt = cnt;
              st.ctrl->fchk_side = side;
              st.ctrl->fchk_want_d = wa ? w.delta() : 0.0;
              st.ctrl->fchk_want_k = wa ? w.index() : -1;
              st.ctrl->fchk_got_d = fa ? f.delta() : 0.0;
              st.ctrl->fchk_got_k = fa ? f.index() : -1;
              // the wanted candidate's filter value from the copies in HBM,
              // and what it was compared with
              const int32_t wp = !wa ? -1 : (side ? w.index() : st.sigma[w.index()]);
              if (wp >= 0) {
                const int32_t wt = tau_g[wp];
                const uint32_t a = aux_g[wp];
                st.ctrl->fchk_p = wp;
                st.ctrl->fchk_aux_ok = (a & 0x1FFFFu) == static_cast<uint32_t>(wt) * sizeof(Q) &&
                                       static_cast<int32_t>(a >> 17) ==
                                           static_cast<int32_t>(floor(static_cast<double>(acur_g[wp]) * S)) + kAuxBias;
                st.ctrl->fchk_u = static_cast<int32_t>(Qg[static_cast<int64_t>(im.agent) * ld + wt]) +
                                  static_cast<int32_t>(QTg[static_cast<int64_t>(im.job) * ld + wp]) -
                                  static_cast<int32_t>(a >> 17);
              }
              st.ctrl->fchk_t0 = im.t0;
              st.ctrl->fchk_tmax = tmax[par];
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        qn[par] = 0;
        tmax[par] = kFNeg;
        // (the reduced tracks depend on every lane's queue reads)
        mbar_arrive_after(&queue_free[par], static_cast<uint32_t>(ta.i ^ tj.i));
      }
      // records + proposals (entries filled in at the flush: finish_prop pad 2)
      bool emit = false;
      Prop entry;
      if (lane < 2) {
        const Track<kFloat>& r = lane == 0 ? ta : tj;
        const bool ok = r.valid();
        const double d = ok ? r.delta() : 0.0;
        const int32_t k = ok ? r.index() : -1;
        const bool active = ok && d > st.eps;
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
      }
      const unsigned mask = __ballot_sync(0xffffffffu, emit);
      if (mask) {
        const int base = ebuf_n;  // this warp is the only writer
        if (emit) {
          const int pos = base + __popc(mask & ((1u << lane) - 1));
          if (pos < kFEdgeBuf) {
            ebuf[pos] = entry;
          } else {
            const int gg = atomicAdd(&st.ctrl->edge_count[parity_out], 1);
            st.edges[parity_out][gg] = finish_prop(entry, st.sigma, tau_g, st.AT, st.storage, ld, n);
          }
        }
        __syncwarp();
        if (lane == 0) ebuf_n = base + __popc(mask);
        __syncwarp();
      }
    }
    if (lane == 0) {  // instrumentation: candidates verified, whole-item fallbacks
      atomicAdd(reinterpret_cast<unsigned long long*>(&st.ctrl->filter_kept), static_cast<unsigned long long>(kept));
      if (overflows)
        atomicAdd(reinterpret_cast<unsigned long long*>(&st.ctrl->filter_overflows),
                  static_cast<unsigned long long>(overflows));
    }
  } else {
    // ---------------- consumers: block `warp` of every chunk ----------------
    // The 8 aux words of a lane's positions come from tensor memory (or, past
    // the first 16 chunks, from L2 two chunks ahead in registers); only the
    // QT chunk and the gathered Q row go through shared memory.
    const int32_t lo = warp * kFBlk + lane * kFV;  // position offset within a chunk
    int s = 0;
    uint32_t fph = 0;  // slot_full phase parity
    auto load_aux = [&](int32_t c, AuxW<kFV>& x) {
      const int64_t p = static_cast<int64_t>(c) * kFChunk + lo;
      ld_aux<kFV>(x, aux_g + p, p < n);
    };
    // two chunks of aux in flight: L2 latency under this load exceeds one
    // chunk's compute (long-scoreboard stalls with a one-chunk lead)
    AuxW<kFV> nx, fx;
    int32_t cnext = nch > 1 ? 1 : 0;  // chunk held in fx
    // (chunks >= ntm rotate through nx / fx, two chunks ahead)
    if constexpr (!kAllTM) {
      if (0 >= ntm) load_aux(0, nx);
      if (cnext >= ntm) load_aux(cnext, fx);
    }
    const uint32_t tw = tmem_base + (static_cast<uint32_t>(32 * (warp & 3)) << 16) +
                        static_cast<uint32_t>((warp >> 2) * ntm * kFV);
    for (int32_t q = 0; q < stages; ++q) {
      const int rb = q % RB;
      const int par = q & 1;
      mbar_wait_backoff(&row_full[rb], static_cast<uint32_t>((q / RB) & 1), 32);
      if (q >= 2) mbar_wait_backoff(&queue_free[par], static_cast<uint32_t>(((q - 2) >> 1) & 1), 32);
      const int32_t t0 = info_s[rb].t0;
      const unsigned char* rowb = reinterpret_cast<const unsigned char*>(rows) + static_cast<size_t>(rb) * row_bytes;
      int32_t T = t0;
      int32_t tshare = kFNeg;  // last read of tmax[par]
      for (int32_t c = 0; c < nch; ++c) {
        AuxW<kFV> ax;
        const bool in_tm = kAllTM || c < ntm;  // (warp-uniform)
        if (in_tm)
          tmem_ld8(tw + static_cast<uint32_t>(c * kFV), ax.w);  // completes behind the slot wait
        else
          ax = nx;
        if constexpr (!kAllTM) {
          nx = fx;
          cnext = cnext + 1 < nch ? cnext + 1 : 0;  // chunk c + 2 (wrapping into the next item)
          if (cnext >= ntm) load_aux(cnext, fx);
        }
        mbar_wait_backoff(&slot_full[s], fph, 20);
        if (in_tm) tmem_wait_ld();
        const unsigned char* sb = slots + s * kSlotBytes;
        const uint4 qv = lds_q<Q, kFV>(sb + lo * static_cast<int>(sizeof(Q)));
        const uint32_t(&aw)[kFV] = ax.w;
        const int32_t p0 = c * kFChunk + lo;
        // aux low 17 bits = the BYTE offset of Q[i][t] in the staged row, so a
        // gather is one LOP3 + one LDS [reg + uniform base]
        int32_t U[kFV];
#pragma unroll
        for (int v = 0; v < kFV; ++v) {
          const uint32_t off = aw[v] & 0x1FFFFu;
          const int32_t cb = static_cast<int32_t>(aw[v] >> 17);
          U[v] = static_cast<int32_t>(*reinterpret_cast<const Q*>(rowb + off)) + q_elem<Q>(qv, v) - cb;
        }
        if (c == nch - 1) {  // the ragged last chunk: positions past n (aux word 0) never count
#pragma unroll
          for (int v = 0; v < kFV; ++v) U[v] = (p0 + v < n) ? U[v] : kFNeg;
        }
        int32_t m = U[0];
#pragma unroll
        for (int v = 1; v < kFV; ++v) m = max(m, U[v]);
        // the CTA's best bound, read (plain LDS) one chunk late: a stale,
        // lower T only keeps more candidates, never drops one
        T = max(T, tshare - 4);
        // Common path: no lane reaches T (once an item's maximum is known,
        // almost every block), one vote and nothing else.  A block that
        // reaches T raises T to its own max - 4, tests its positions one by
        // one and publishes the max for the other warps.
        const bool hit = __any_sync(0xffffffffu, m >= T);
        // Release the QT slot only after the vote: it consumed every lane's
        // loads, and the arrive takes it as an operand, so no lane's LDS can
        // still be in flight when the TMA refills the slot.  (An arrive right
        // after the LDS did exactly that on a 3-slot ring: the self-check
        // LSAPGPU_FILTER_CHECK caught dropped maxima at C5.)
        if (lane == 0) mbar_arrive_after(&slot_empty[s], hit ? 1u : 0u);
        if (++s == NS) {
          s = 0;
          fph ^= 1u;
        }
        if (hit) {
          const int32_t wm = __reduce_max_sync(0xffffffffu, m);
          T = max(T, wm - 4);
          if (lane == 0) atomicMax(&tmax[par], wm);
          uint32_t bits = 0;
#pragma unroll
          for (int v = 0; v < kFV; ++v) bits |= (U[v] >= T ? 1u : 0u) << v;
          if (bits) {
            int pos = atomicAdd(&qn[par], __popc(bits));
#pragma unroll
            for (int v = 0; v < kFV; ++v)
              if ((bits >> v) & 1u) {
                if (pos < qcap)
                  queue[par * qcap + pos] = static_cast<unsigned long long>(static_cast<uint32_t>(p0 + v)) |
                                            (static_cast<unsigned long long>((aw[v] & 0x1FFFFu) / sizeof(Q)) << 32);
                ++pos;
              }
          }
        }
        tshare = *reinterpret_cast<volatile int*>(&tmax[par]);  // used at the next chunk
      }
      // every lane arrives after its last use of row buffer rb and its own
      // queue stores: releases the row and hands the queue to the verifier
      mbar_arrive_after(&item_done[par], static_cast<uint32_t>(tshare));
    }
  }
  if constexpr (kTM) tmem_fence_before();
  __syncthreads();
  if constexpr (kTM) {
    tmem_fence_after();
    if (warp == 0) tmem_dealloc512(tmem_base);
  }
  const int ne = min(ebuf_n, kFEdgeBuf);
  __shared__ int gbase;
  if (tid == 0 && ne > 0) gbase = atomicAdd(&st.ctrl->edge_count[parity_out], ne);
  __syncthreads();
  for (int e = tid; e < ne; e += kFThreads)
    st.edges[parity_out][gbase + e] = finish_prop(ebuf[e], st.sigma, tau_g, st.AT, st.storage, ld, n);
}

// Per-launch position array: aux[p] = tau[p] * sizeof(Q) | (floor(acur[p] * S) + 2^14) << 17
// (the byte offset of the gathered element in a staged Q row: < 2^17 for
// every plan, int16 copies are only chosen when two rows fit on chip).
template <class E, class Q>
__global__ void filter_aux_kernel(DevState st) {
  pdl_trigger();
  pdl_wait();
  const E* acur = static_cast<const E*>(st.acur);
  const double S = st.qscale;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < st.ld;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t w = 0;
    if (p < st.n) {
      const int32_t cq = static_cast<int32_t>(floor(static_cast<double>(acur[p]) * S)) + kAuxBias;
      w = static_cast<uint32_t>(st.tau[p]) * static_cast<uint32_t>(sizeof(Q)) | (static_cast<uint32_t>(cq) << 17);
    }
    st.aux[p] = w;
  }
}

template <class E, class Q, int RB, int W, int V, int kAux>
cudaError_t launch_filter_t(const DevState& d, const ScanPlan& p, int full, cudaStream_t st) {
  cudaError_t e = launch_pdl(filter_aux_kernel<E, Q>, dim3(p.ctas), dim3(256), 0, st, d.pdl, d);
  if (e != cudaSuccess) return e;
  auto k = pair_scan_filter_kernel<E, Q, RB, W, V, kAux>;
  e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem));
  if (e != cudaSuccess) return e;
  return launch_pdl(k, dim3(p.ctas), dim3(32 * (W + 3)), p.smem, st, d.pdl, d, full, p.bufs, p.filter_queue);
}

// consumer geometry: 16 warps x 8 positions per lane (24 x 4 measured no
// faster at C4 / C5: the kernel is not short of warps; 16 x 16 for int8
// copies measured 28% slower at C5, and three rotating aux register sets
// instead of the copy per chunk 6-17% slower: a later aux load issue)
template <class E, class Q, int RB>
cudaError_t launch_filter_g(const DevState& d, const ScanPlan& p, int full, cudaStream_t st) {
  if (p.filter_tmem && (d.n + 4095) / 4096 <= 16) return launch_filter_t<E, Q, RB, 16, 8, 2>(d, p, full, st);
  if (p.filter_tmem) return launch_filter_t<E, Q, RB, 16, 8, 1>(d, p, full, st);
  return launch_filter_t<E, Q, RB, 16, 8, 0>(d, p, full, st);
}

}  // namespace scan_detail

template <class E>
cudaError_t launch_scan_filter_typed(const DevState& d, const ScanPlan& p, int full, cudaStream_t st) {
  if (p.filter == 16)
    return p.m == 2 ? scan_detail::launch_filter_g<E, int16_t, 2>(d, p, full, st)
                    : scan_detail::launch_filter_g<E, int16_t, 1>(d, p, full, st);
  return p.m == 2 ? scan_detail::launch_filter_g<E, int8_t, 2>(d, p, full, st)
                  : scan_detail::launch_filter_g<E, int8_t, 1>(d, p, full, st);
}

}  // namespace lsapgpu
