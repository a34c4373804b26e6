// commit_cluster.cu -- the production commit kernel: one inner iteration of
// the reference's batch loop (proj/src/parallel.cpp:264-335) minus the scans,
// run by ONE thread-block cluster (16 CTAs x 1024 threads where the part
// allows non-portable clusters, else 8) that keeps the whole conflict-check
// state in distributed shared memory.
//
//   P0  control: abort tests (no active record -> inner loop done and the
//       graph's WHILE condition is cleared; deadline; full delta log)
//   P1  proposals -> edges (agent endpoints from the frozen sigma), chunked
//       over the cluster's CTAs; vertex keys zeroed (keys of vertex v live in
//       CTA v % CS at index v / CS)
//   P2  LFMM rounds (see commit.cu for why they equal the reference's
//       sequential reservation walk, parallel.cpp:35-76): phase A posts the
//       edge's epoch-tagged inverted priority to both endpoint keys with
//       DSMEM atomicMax (or rejects it when an endpoint is matched), phase B
//       accepts the edges that hold both keys and marks the endpoints
//       matched; a cluster barrier (~0.3 us) separates the phases
//   P3  select: accepted records are zeroed and their improvement recomputed
//       on the frozen assignment (solver_state.hpp:106-122), committed iff > eps
//   P4  apply + delta log + touched work items, disjointness asserted
//       (parallel.cpp:296-310)
//   P5  conflicted work items (touched_and_conflicted) or carried edges
//       (touched_only), parallel.cpp:312-330
#include <cooperative_groups.h>

#include <climits>

#include "state.h"

namespace cg = cooperative_groups;

namespace lsapgpu {
namespace {

constexpr uint8_t kEdgeCommitted = 4;
constexpr uint32_t kMatched = 0xFFFFFFFFu;
constexpr uint32_t kKeyShift = 18;  // priorities (slots) < 2^18
constexpr uint32_t kRoundLimit = (1u << 14) - 2;
constexpr int kNT = 1024;

__device__ __forceinline__ uint32_t make_key(uint32_t round, int32_t slot) {
  return (round << kKeyShift) | (0x3FFFFu - static_cast<uint32_t>(slot));
}

// warp-aggregated append of `want` (0/1) entries to a global counter
__device__ __forceinline__ int warp_append(int* counter, bool want) {
  const unsigned mask = __ballot_sync(0xffffffffu, want);
  if (!mask) return -1;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(mask) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  return want ? base + __popc(mask & ((1u << lane) - 1)) : -1;
}
__device__ __forceinline__ long long warp_append64(long long* counter, bool want) {
  const unsigned mask = __ballot_sync(0xffffffffu, want);
  if (!mask) return -1;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(mask) - 1;
  unsigned long long base = 0;
  if (lane == leader)
    base = atomicAdd(reinterpret_cast<unsigned long long*>(counter), static_cast<unsigned long long>(__popc(mask)));
  base = __shfl_sync(0xffffffffu, base, leader);
  return want ? static_cast<long long>(base) + __popc(mask & ((1u << lane) - 1)) : -1;
}

__device__ __forceinline__ int block_sum(int v, int* s) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(s, v);
  return v;
}

struct CommitScratch {  // per-CTA shared scalars
  int abort;
  int count[2];
  int committed, ascans, jscans, items;
  int total;
};

template <class E, int CS>
__global__ void __launch_bounds__(kNT, 1)
    commit_cluster_kernel(DevState st, int mode, cudaGraphConditionalHandle cond, int use_cond,
                          int edge_cap) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const int tid = threadIdx.x;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ CommitScratch sc;
  __shared__ uint32_t* kbase[CS];

  Ctrl* C = st.ctrl;
  const int32_t n = st.n;
  const E* A = static_cast<const E*>(st.A);
  E* acur = static_cast<E*>(st.acur);
  const int64_t ld = st.ld;
  const int P = C->parity;
  const int32_t m = C->edge_count[P];
  const int4* edges = st.edges[P];

  // ---- P0: control (rank 0 decides, everyone reads its verdict) ----
  if (tid == 0) {
    sc.abort = 0;
    sc.count[0] = sc.count[1] = 0;
    sc.committed = sc.ascans = sc.jscans = sc.items = 0;
    if (rank == 0 && mode == kCommitSolve) {
      if (C->expired || C->drain || C->error || C->inner_done)
        sc.abort = 1;
      else if (m == 0)
        sc.abort = 2;
      else if (C->deadline_gt != 0 && globaltimer() >= C->deadline_gt)
        sc.abort = 3;
      else if (C->log_count + m > st.log_cap)
        sc.abort = 4;
    }
  }
  if (tid < CS) kbase[tid] = cluster.map_shared_rank(reinterpret_cast<uint32_t*>(smem), tid);
  cluster.sync();
  const int abort = *cluster.map_shared_rank(&sc.abort, 0);
  cluster.sync();  // rank 0's shared memory must outlive every peer read
  if (abort) {
    if (rank == 0 && tid == 0) {
      if (abort == 2) C->inner_done = 1;
      if (abort == 3) C->expired = 1;
      if (abort == 4) C->drain = 1;
      C->work_count = 0;
      if (use_cond) cudaGraphSetConditional(cond, 0);
    }
    return;
  }
  const int32_t iter = C->iter + 1;
  if (rank == 0 && tid == 0) C->work_count = 0;  // nobody appends before the next cluster barrier

  // ---- P1: keys and this CTA's edges ----
  const int32_t kslice = (n + CS - 1) / CS;
  uint32_t* mykeys = reinterpret_cast<uint32_t*>(smem);
  for (int32_t x = tid; x < kslice; x += kNT) mykeys[x] = 0u;
  const int32_t per = (m + CS - 1) / CS;
  const int32_t e0 = rank * per;
  const int32_t cnt = max(0, min(m, e0 + per) - e0);
  int32_t *Eu, *Ev, *Ejold, *Ejnew;
  uint8_t* Est;
  double* Edel;
  if (per <= edge_cap) {
    unsigned char* q = smem + ((static_cast<size_t>(kslice) * 4 + 15) / 16) * 16;
    Edel = reinterpret_cast<double*>(q);
    q += static_cast<size_t>(edge_cap) * 8;
    Eu = reinterpret_cast<int32_t*>(q);
    q += static_cast<size_t>(edge_cap) * 4;
    Ev = reinterpret_cast<int32_t*>(q);
    q += static_cast<size_t>(edge_cap) * 4;
    Ejold = reinterpret_cast<int32_t*>(q);
    q += static_cast<size_t>(edge_cap) * 4;
    Ejnew = reinterpret_cast<int32_t*>(q);
    q += static_cast<size_t>(edge_cap) * 4;
    Est = q;
  } else {  // too many proposals for DSMEM: same layout in global scratch
    Eu = st.eu + e0;
    Ev = st.ev + e0;
    Ejold = st.eprop + e0;
    Ejnew = st.c_jnew + e0;
    Est = st.estate + e0;
    Edel = st.c_delta + e0;
  }
  for (int32_t l = tid; l < cnt; l += kNT) {
    // proposals carry {slot, proposer, partner, job}: one dependent load left
    const int4 en = edges[e0 + l];
    Eu[l] = en.y;  // proposer: the agent, or the job's current holder (frozen)
    if (en.x < n) {
      Ev[l] = st.sigma[en.z];  // the displaced holder of the proposed job
    } else {
      Ev[l] = en.z;                 // the proposed agent
      Ejold[l] = st.tau[en.z];      // ... and its current job
    }
    Est[l] = kEdgeUndecided;
  }
  cluster.sync();

  // ---- P2: LFMM rounds ----
  uint32_t R = 1;
  int rounds = 0;
  for (;;) {
    if (R >= kRoundLimit) {
      for (int32_t x = tid; x < kslice; x += kNT)
        if (mykeys[x] != kMatched) mykeys[x] = 0u;
      R = 1;
      cluster.sync();
    }
    int local = 0;
    for (int32_t l = tid; l < cnt; l += kNT) {
      if (Est[l] != kEdgeUndecided) continue;
      const int32_t u = Eu[l], v = Ev[l];
      uint32_t* ku = kbase[u % CS] + u / CS;
      uint32_t* kv = kbase[v % CS] + v / CS;
      if (*ku == kMatched || *kv == kMatched) {
        Est[l] = kEdgeRejected;
      } else {
        const uint32_t k = make_key(R, edges[e0 + l].x);
        atomicMax(ku, k);
        atomicMax(kv, k);
        ++local;
      }
    }
    block_sum(local, &sc.count[rounds & 1]);
    cluster.sync();
    if (tid == 0) {
      int tot = 0;
      for (int r = 0; r < CS; ++r) tot += *cluster.map_shared_rank(&sc.count[rounds & 1], r);
      sc.total = tot;
    }
    __syncthreads();
    const int total = sc.total;
    if (tid == 0) sc.count[(rounds + 1) & 1] = 0;  // read by peers only after the next barrier
    if (total == 0) break;
    for (int32_t l = tid; l < cnt; l += kNT) {
      if (Est[l] != kEdgeUndecided) continue;
      const int32_t u = Eu[l], v = Ev[l];
      uint32_t* ku = kbase[u % CS] + u / CS;
      uint32_t* kv = kbase[v % CS] + v / CS;
      const uint32_t k = make_key(R, edges[e0 + l].x);
      if (*ku == k && *kv == k) {
        Est[l] = kEdgeAccepted;
        *ku = kMatched;
        *kv = kMatched;
      }
    }
    cluster.sync();
    ++R;
    ++rounds;
  }

  if (mode == kCommitCheckOnly) {
    if (per <= edge_cap)
      for (int32_t l = tid; l < cnt; l += kNT) {
        st.estate[e0 + l] = Est[l];
        st.eu[e0 + l] = Eu[l];
        st.ev[e0 + l] = Ev[l];
      }
    if (rank == 0 && tid == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&C->lfmm_rounds),
                                         static_cast<unsigned long long>(rounds));
    cluster.sync();  // keep peer smem alive until everyone is done
    return;
  }

  // ---- P3: select (frozen reads) ----
  const double eps = st.eps;
  for (int32_t l = tid; l < cnt; l += kNT) {
    if (Est[l] != kEdgeAccepted) continue;
    const int4 en = edges[e0 + l];
    int32_t agent, j_new, j_old, disp;
    typename Traits<E>::Acc actual;
    if (en.x < n) {  // agent_proposal_delta, solver_state.hpp:106-113
      agent = en.y;
      j_new = en.z;
      j_old = en.w;
      disp = Ev[l];
      st.agent_delta[agent] = 0.0;
      st.agent_partner[agent] = -1;
      const int64_t ra = static_cast<int64_t>(agent) * ld, rd = static_cast<int64_t>(disp) * ld;
      actual = delta4(widen(A[ra + j_new]), widen(A[ra + j_old]), widen(A[rd + j_old]),
                      widen(A[rd + j_new]));
    } else {  // job_proposal_delta, solver_state.hpp:115-122
      agent = en.z;
      j_new = en.w;
      disp = en.y;
      j_old = Ejold[l];
      st.job_delta[j_new] = 0.0;
      st.job_partner[j_new] = -1;
      const int64_t ri = static_cast<int64_t>(agent) * ld, rh = static_cast<int64_t>(disp) * ld;
      actual = delta4(widen(A[ri + j_new]), widen(A[rh + j_new]), widen(A[rh + j_old]),
                      widen(A[ri + j_old]));
    }
    const double dact = static_cast<double>(actual);
    if (dact > eps) {
      Est[l] = kEdgeCommitted;
      Eu[l] = agent;
      Ev[l] = disp;
      Ejold[l] = j_old;
      Ejnew[l] = j_new;
      Edel[l] = dact;
    }
  }
  cluster.sync();

  // ---- P4: apply, log, touched work items ----
  int committed = 0;
  for (int32_t base = 0; base < cnt; base += kNT) {  // warp-uniform trip count for the appends
    const int32_t l = base + tid;
    const bool mine = l < cnt && Est[l] == kEdgeCommitted;
    int32_t agent = 0, disp = 0;
    if (mine) {
      agent = Eu[l];
      disp = Ev[l];
      const int32_t j_old = Ejold[l], j_new = Ejnew[l];
      if (atomicExch(&st.touched_stamp[agent], iter) == iter ||
          atomicExch(&st.touched_stamp[disp], iter) == iter)
        atomicExch(&C->error, 1);
      st.sigma[j_new] = agent;
      st.sigma[j_old] = disp;
      st.tau[agent] = j_new;
      st.tau[disp] = j_old;
      acur[agent] = A[static_cast<int64_t>(agent) * ld + j_new];
      acur[disp] = A[static_cast<int64_t>(disp) * ld + j_old];
      ++committed;
    }
    const long long pos = warp_append64(reinterpret_cast<long long*>(&C->log_count), mine);
    if (mine) st.log[pos] = LogEntry{iter, edges[e0 + l].x, Edel[l]};
    const unsigned mask = __ballot_sync(0xffffffffu, mine);
    if (mask) {
      const int lane = tid & 31;
      const int leader = __ffs(mask) - 1;
      int w = 0;
      if (lane == leader) w = atomicAdd(&C->work_count, 2 * __popc(mask));
      w = __shfl_sync(0xffffffffu, w, leader);
      if (mine) {
        const int o = w + 2 * __popc(mask & ((1u << lane) - 1));
        st.items[o] = static_cast<uint32_t>(agent) | kItemAgent | kItemJob;
        st.items[o + 1] = static_cast<uint32_t>(disp) | kItemAgent | kItemJob;
      }
    }
  }
  block_sum(committed, &sc.committed);
  for (int32_t l = tid; l < cnt; l += kNT)
    if (Est[l] == kEdgeRejected) st.rej_stamp[edges[e0 + l].x] = iter;
  cluster.sync();

  // ---- P5: conflicted re-evaluation / carried edges ----
  int la = 0, lj = 0;
  for (int32_t base = 0; base < cnt; base += kNT) {
    const int32_t l = base + tid;
    bool emit = false, jflag = false;
    int32_t p = 0;
    if (l < cnt && Est[l] == kEdgeRejected) {
      const int4 en = edges[e0 + l];
      p = en.y;  // the proposer (frozen holder for job-side proposals)
      if (st.policy == 0) {
        if (st.touched_stamp[p] != iter && atomicExch(&st.conf_stamp[p], iter) != iter) {
          // p is untouched, so its job is still the proposal's job (en.w for
          // job records, tau[p] = en.w for agent records as well)
          jflag = st.rej_stamp[n + en.w] == iter;
          emit = true;
          ++la;
          if (jflag) ++lj;
        }
      } else if (st.touched_stamp[p] != iter) {
        // touched_only: an untouched proposer keeps its stale record -> carry it
        const int pos = atomicAdd(&C->edge_count[1 - P], 1);
        st.edges[1 - P][pos] = en;
      }
    }
    const int w = warp_append(&C->work_count, emit);
    if (emit) st.items[w] = static_cast<uint32_t>(p) | kItemAgent | (jflag ? kItemJob : 0u);
  }
  block_sum(la, &sc.ascans);
  block_sum(lj, &sc.jscans);
  __syncthreads();
  if (tid == 0) {
    const long long touched = 2ll * sc.committed;
    atomicAdd(reinterpret_cast<unsigned long long*>(&C->switches), static_cast<unsigned long long>(sc.committed));
    atomicAdd(reinterpret_cast<unsigned long long*>(&C->agent_scans),
              static_cast<unsigned long long>(touched + sc.ascans));
    atomicAdd(reinterpret_cast<unsigned long long*>(&C->job_scans),
              static_cast<unsigned long long>(touched + sc.jscans));
    atomicAdd(reinterpret_cast<unsigned long long*>(&C->pair_items),
              static_cast<unsigned long long>(touched + sc.ascans));
  }
  cluster.sync();  // all appends done, peer smem no longer referenced
  if (rank == 0 && tid == 0) {
    C->iter = iter;
    C->round = 1;
    C->parity = 1 - P;
    C->edge_count[P] = 0;
    C->lfmm_rounds += rounds;
    C->inner_iterations += 1;
  }
}

template <class E, int CS>
cudaError_t launch_cs(const DevState& d, const CommitPlan& p, int mode, cudaGraphConditionalHandle cond,
                      int use_cond, cudaStream_t st) {
  auto k = commit_cluster_kernel<E, CS>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(p.cluster_smem));
  if (e != cudaSuccess) return e;
  if (CS > 8) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS);
  cfg.blockDim = dim3(kNT);
  cfg.dynamicSmemBytes = p.cluster_smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, d, mode, cond, use_cond, p.edge_cap);
}

template <int CS>
cudaError_t launch_any(const DevState& d, const CommitPlan& p, int mode, cudaGraphConditionalHandle cond,
                       int use_cond, cudaStream_t st) {
  switch (d.storage) {
    case kI16: return launch_cs<int16_t, CS>(d, p, mode, cond, use_cond, st);
    case kI32: return launch_cs<int32_t, CS>(d, p, mode, cond, use_cond, st);
    case kF32: return launch_cs<float, CS>(d, p, mode, cond, use_cond, st);
    case kF64: return launch_cs<double, CS>(d, p, mode, cond, use_cond, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

// Cluster size: 16 when the device can co-schedule a non-portable 16-CTA
// cluster of this kernel, else the portable 8.
int commit_cluster_size(const DevState& d, size_t smem) {
  static int cached = 0;
  if (cached) return cached;
  auto k = commit_cluster_kernel<int32_t, 16>;
  int clusters = 0;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) ==
          cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(kNT);
    cfg.dynamicSmemBytes = smem;
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
  (void)d;
  cached = clusters > 0 ? 16 : 8;
  return cached;
}

cudaError_t launch_commit_cluster(const DevState& d, const CommitPlan& p, int mode,
                                  cudaGraphConditionalHandle cond, int use_cond, cudaStream_t st) {
  return p.cluster == 16 ? launch_any<16>(d, p, mode, cond, use_cond, st)
                         : launch_any<8>(d, p, mode, cond, use_cond, st);
}

}  // namespace lsapgpu
