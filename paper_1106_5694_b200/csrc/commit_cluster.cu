// commit_cluster.cu -- the production commit kernel: one inner iteration of
// the reference's batch loop (proj/src/parallel.cpp:264-335) minus the scans,
// run by ONE thread-block cluster (16 CTAs x 1024 threads where the part
// allows non-portable clusters, else 8) that keeps every per-vertex structure
// of the conflict check in distributed shared memory.  Vertex v (agent or job
// index) lives in CTA v % CS at slot v / CS: its LFMM key and a flag word
// (bit 0 agent touched by a committed exchange, bit 1 agent already queued as
// conflicted, bit 2 job's own proposal rejected).  The proposals are split in
// contiguous chunks over the CTAs.
//
//   P0  control, decided identically by every CTA from values the previous
//       kernel wrote (no barrier): no active proposal -> inner loop done and
//       the graph's WHILE condition cleared; full delta log -> host drain;
//       deadline flag (checked at the end of the previous commit)
//   P1  proposal endpoints (agents) from the frozen sigma/tau
//   P2  LFMM rounds (see commit.cu for why they equal the sequential
//       reservation walk of check_conflicts_impl, parallel.cpp:35-76):
//       phase A posts the epoch-tagged inverted priority to both endpoint
//       keys with DSMEM atomicMax (or rejects the edge when an endpoint is
//       matched), phase B accepts edges that hold both keys
//   P3  select: accepted records are zeroed and their improvement recomputed
//       on the frozen assignment (solver_state.hpp:106-122), committed iff
//       > eps; committed exchanges mark their agents touched in DSMEM (a
//       second mark is the reference's overlap assertion, parallel.cpp:296-302)
//   P4  apply (sigma/tau/acur), delta log, re-evaluation work items: touched
//       pairs and, under touched_and_conflicted, every untouched conflicted
//       proposer (parallel.cpp:312-330); each CTA reserves its log / item
//       ranges with one global atomic
#include <cooperative_groups.h>

#include <climits>

#include "commit_apply.cuh"
#include "commit_single.cuh"
#include "state.h"

namespace cg = cooperative_groups;

namespace lsapgpu {
namespace {

constexpr uint8_t kEdgeCommitted = 4;
constexpr uint32_t kKeyShift = 18;  // priorities (slots) < 2^18
constexpr int kNT = 1024;
constexpr uint32_t kTouched = 1u, kQueued = 2u, kJobRejected = 4u;
constexpr int32_t kNoEmit = -1;
constexpr int32_t kJobFlagBit = 1 << 30;
constexpr int32_t kSingleLoad = 2048;  // proposals rank 0 of the split commit loads alone

__device__ __forceinline__ uint32_t make_key(uint32_t round, int32_t slot) {
  return (round << kKeyShift) | (0x3FFFFu - static_cast<uint32_t>(slot));
}

// LFMM vertex keys (32 bit).  Narrow (n < 2^17): {14-bit round, 18-bit
// inverted slot}, so keys of earlier rounds lose without clearing.  Wide (any
// larger n; the reference has no size limit): the inverted slot alone, and
// every CTA clears its unmatched keys before each round (one more cluster
// barrier per round).  64-bit keys would need a 64-bit atomic max on
// distributed shared memory, which the hardware emulates with a CAS loop on
// the CTA's OWN shared memory (wrong for a peer's slice).
template <bool kWide>
struct LfmmKey;
template <>
struct LfmmKey<false> {
  static constexpr uint32_t kMatched = 0xFFFFFFFFu;
  static constexpr uint32_t kRoundLimit = (1u << 14) - 2;
  __device__ static uint32_t make(uint32_t round, int32_t slot) { return make_key(round, slot); }
};
template <>
struct LfmmKey<true> {
  static constexpr uint32_t kMatched = 0xFFFFFFFFu;
  static constexpr uint32_t kRoundLimit = 1;  // R >= 1 always: clear before every round
  __device__ static uint32_t make(uint32_t, int32_t slot) { return 0xFFFFFFFEu - static_cast<uint32_t>(slot); }
};

__device__ __forceinline__ void block_add(int v, int* s) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(s, v);
}

struct CommitScratch {  // per-CTA shared scalars
  int count[2];
  int total;
  int nlog, nconf, nconf_j;
  unsigned long long base_log;
  int base_items;
  int base_conf;
};

// Per-proposal working set of this CTA (shared memory, or global scratch
// when the chunk does not fit).
struct EdgeArrays {
  int32_t *u, *v, *jold, *rank, *slot;
  uint8_t* st;
  double *del, *acur_a, *acur_d;
};

template <class E, int CS, bool kWide>
__global__ void __launch_bounds__(kNT, 1)
    commit_cluster_kernel(DevState st, int mode, cudaGraphConditionalHandle cond, int use_cond,
                          int edge_cap, int cta_cap, int var) {
  using KK = LfmmKey<kWide>;
  using K = uint32_t;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const int tid = threadIdx.x;
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ CommitScratch sc;
  __shared__ K* kbase[CS];
  __shared__ uint32_t* fbase[CS];

  Ctrl* C = st.ctrl;
  const int32_t n = st.n;
  const E* AT = static_cast<const E*>(st.AT);  // A[i][j] = AT[j][i]: AT is whole on every rank
  E* acur = static_cast<E*>(st.acur);
  const int64_t ld = st.ld;
  // every control field in one round trip (independent loads: no dependent
  // edge_count[parity] load, no short-circuit chain)
  const int P = C->parity;
  const int32_t ec0 = C->edge_count[0], ec1 = C->edge_count[1];
  const int f_stop = C->expired | C->drain | C->error | C->inner_done;
  const int64_t log_count = C->log_count;
  const int32_t m = P ? ec1 : ec0;
  const Prop* edges = st.edges[P];

  if (rank == 0 && tid == 0) tl_mark(C, st.tl, st.tl_cap, kTlCommit);
  // ---- P0: control ----
  if (mode == kCommitSolve) {
    int abort = 0;
    if (f_stop)
      abort = 1;
    else if (m == 0)
      abort = 2;
    else if (log_count + m > st.log_cap)
      abort = 4;
    if (abort) {
      if (rank == 0 && tid == 0) {
        if (abort == 2) C->inner_done = 1;
        if (abort == 4) C->drain = 1;
        C->work_count = 0;
        C->k2_nlog = C->k2_nconf = 0;
        if (use_cond) cudaGraphSetConditional(cond, 0);
      }
      return;
    }
    if (rank == 0 && tid == 0) {
      C->work_count = 0;  // appends start after two cluster barriers
      C->k2_nlog = C->k2_nconf = 0;
    }
  }
  // Default policy and a batch whose vertex state fits one SM: the conflict
  // check runs on one CTA with CTA barriers and local shared-memory atomics,
  // and the scattered writes follow grid-wide in commit_apply_kernel
  // (commit_single.cuh).  Otherwise the whole cluster runs the iteration.
  if (m <= cta_cap && (st.policy == 0 || mode == kCommitCheckOnly)) {
    if (m <= kSingleLoad) {  // few proposals: rank 0 loads them itself
      if (rank == 0) single::commit_single(st, mode, cta_cap, smem, false, !(var & 2));
    } else {  // many: every rank loads a share straight into rank 0's shared memory
      unsigned char* dst = cluster.map_shared_rank(smem, 0);
      const int32_t per = (m + CS - 1) / CS;
      single::load_share(st, cta_cap, dst, min(m, rank * per), min(m, (rank + 1) * per));
      cluster.sync();
      if (rank == 0) single::commit_single(st, mode, cta_cap, smem, true, !(var & 2));
    }
    return;
  }
  const int32_t iter = C->iter + 1;

  // ---- P1: vertex slices, proposal endpoints ----
  const int32_t kslice = (n + CS - 1) / CS;
  const size_t kbytes = ((static_cast<size_t>(kslice) * sizeof(K) + 15) / 16) * 16;
  const size_t fbytes = ((static_cast<size_t>(kslice) * 4 + 15) / 16) * 16;
  // (the keys live in DSMEM: the same LFMM on global-memory keys, L2
  // atomics, measured 8% slower over a C3 solve's commits)
  K* mykeys = reinterpret_cast<K*>(smem);
  uint32_t* myflags = reinterpret_cast<uint32_t*>(smem + kbytes);
  if (tid < CS) {
    kbase[tid] = cluster.map_shared_rank(mykeys, tid);
    fbase[tid] = cluster.map_shared_rank(myflags, tid);
  }
  if (tid == 0) {
    sc.count[0] = sc.count[1] = 0;
    sc.nlog = sc.nconf = sc.nconf_j = 0;
  }
  for (int32_t x = tid; x < kslice; x += kNT) {
    mykeys[x] = 0;
    myflags[x] = 0u;
  }
  if (mode == kCommitSolve && st.policy == 0) {  // this CTA's slice of the rejected-job bitmap
    const int32_t words = (n + 31) / 32, wper = (words + CS - 1) / CS;
    for (int32_t x = rank * wper + tid; x < min(words, (rank + 1) * wper); x += kNT) st.jbits[x] = 0u;
  }
  const int32_t per = (m + CS - 1) / CS;
  const int32_t e0 = rank * per;
  const int32_t cnt = max(0, min(m, e0 + per) - e0);
  EdgeArrays Ea;
  if (per <= edge_cap) {
    unsigned char* q = smem + kbytes + fbytes;
    Ea.del = reinterpret_cast<double*>(q);
    q += static_cast<size_t>(edge_cap) * 8;
    Ea.acur_a = reinterpret_cast<double*>(q);
    q += static_cast<size_t>(edge_cap) * 8;
    Ea.acur_d = reinterpret_cast<double*>(q);
    q += static_cast<size_t>(edge_cap) * 8;
    Ea.u = reinterpret_cast<int32_t*>(q);
    q += static_cast<size_t>(edge_cap) * 4;
    Ea.v = reinterpret_cast<int32_t*>(q);
    q += static_cast<size_t>(edge_cap) * 4;
    Ea.jold = reinterpret_cast<int32_t*>(q);
    q += static_cast<size_t>(edge_cap) * 4;
    Ea.rank = reinterpret_cast<int32_t*>(q);
    q += static_cast<size_t>(edge_cap) * 4;
    Ea.slot = reinterpret_cast<int32_t*>(q);
    q += static_cast<size_t>(edge_cap) * 4;
    Ea.st = q;
  } else {  // too many proposals for shared memory: same arrays in global scratch
    Ea.del = st.c_delta + e0;
    Ea.acur_a = st.c_acur + e0;
    Ea.acur_d = st.c_acur + 2 * static_cast<int64_t>(n) + e0;
    Ea.u = st.eu + e0;
    Ea.v = st.ev + e0;
    Ea.jold = st.eprop + e0;
    Ea.rank = st.c_rank + e0;
    Ea.slot = st.c_jnew + e0;
    Ea.st = st.estate + e0;
  }
  if (st.policy == 0) {
    // default policy: every proposal was written by this batch's scan on the
    // frozen state, so it carries both endpoints (commit_single.cuh header)
    for (int32_t l = tid; l < cnt; l += kNT) {
      const Prop* pe = edges + e0 + l;
      const int4 h = *reinterpret_cast<const int4*>(pe);  // slot, a, d, j_new
      const bool agent_rec = h.x < n;
      Ea.u[l] = agent_rec ? h.y : h.z;  // proposer: the agent, or the job's holder
      Ea.v[l] = agent_rec ? h.z : h.y;  // the displaced holder / the proposed agent
      Ea.jold[l] = pe->j_old;
      Ea.st[l] = kEdgeUndecided;
      Ea.rank[l] = kNoEmit;
      Ea.slot[l] = h.x;
    }
  } else {
    // touched_only: records may predate this batch; endpoints from the
    // current assignment, as check_conflicts reads them (parallel.cpp:35-76)
    for (int32_t l = tid; l < cnt; l += kNT) {
      const int4 en = prop_key(edges[e0 + l], n);
      Ea.u[l] = en.y;  // proposer: the agent, or the job's current holder (frozen)
      if (en.x < n) {
        Ea.v[l] = st.sigma[en.z];  // the displaced holder of the proposed job
        Ea.jold[l] = en.w;         // the proposer's current job
      } else {
        Ea.v[l] = en.z;             // the proposed agent
        Ea.jold[l] = st.tau[en.z];  // ... and its current job
      }
      Ea.st[l] = kEdgeUndecided;
      Ea.rank[l] = kNoEmit;
      Ea.slot[l] = en.x;
    }
  }
  cluster.sync();
  if (rank == 0 && tid == 0) tl_mark(C, st.tl, st.tl_cap, 11);

  // ---- P2: LFMM rounds ----
  uint32_t R = 1;
  int rounds = 0;
  for (;;) {
    if (R >= KK::kRoundLimit) {
      for (int32_t x = tid; x < kslice; x += kNT)
        if (mykeys[x] != KK::kMatched) mykeys[x] = 0;
      R = 1;
      cluster.sync();
    }
    int local = 0;
    for (int32_t l = tid; l < cnt; l += kNT) {
      if (Ea.st[l] != kEdgeUndecided) continue;
      const int32_t u = Ea.u[l], v = Ea.v[l];
      K* ku = kbase[u % CS] + u / CS;
      K* kv = kbase[v % CS] + v / CS;
      const bool pre = rounds > 0 || (var & 1);  // nothing is matched in round 1
      const K cu = pre ? *ku : K(0), cv = pre ? *kv : K(0);
      if (cu == KK::kMatched || cv == KK::kMatched) {
        Ea.st[l] = kEdgeRejected;
      } else {
        // keys only grow within a round: skip the (serialising, remote)
        // atomic when a higher priority is already posted
        const K k = KK::make(R, Ea.slot[l]);
        if (cu < k) atomicMax(ku, k);
        if (cv < k) atomicMax(kv, k);
        ++local;
      }
    }
    block_add(local, &sc.count[rounds & 1]);
    cluster.sync();
    if (rank == 0 && tid == 0) tl_mark(C, st.tl, st.tl_cap, 13);
    if (tid == 0) {
      int tot = 0;
#pragma unroll
      for (int r = 0; r < CS; ++r) tot += *cluster.map_shared_rank(&sc.count[rounds & 1], r);
      sc.total = tot;
      sc.count[(rounds + 1) & 1] = 0;  // peers read it only after the next cluster barrier
    }
    __syncthreads();
    if (sc.total == 0) break;
    for (int32_t l = tid; l < cnt; l += kNT) {
      if (Ea.st[l] != kEdgeUndecided) continue;
      const int32_t u = Ea.u[l], v = Ea.v[l];
      K* ku = kbase[u % CS] + u / CS;
      K* kv = kbase[v % CS] + v / CS;
      const K k = KK::make(R, Ea.slot[l]);
      if (*ku == k && *kv == k) {
        Ea.st[l] = kEdgeAccepted;
        *ku = KK::kMatched;
        *kv = KK::kMatched;
      }
    }
    cluster.sync();
    if (rank == 0 && tid == 0) tl_mark(C, st.tl, st.tl_cap, 12);
    ++R;
    ++rounds;
  }

  if (mode == kCommitCheckOnly) {
    if (per <= edge_cap)
      for (int32_t l = tid; l < cnt; l += kNT) {
        st.estate[e0 + l] = Ea.st[l];
        st.eu[e0 + l] = Ea.u[l];
        st.ev[e0 + l] = Ea.v[l];
      }
    if (rank == 0 && tid == 0) C->lfmm_rounds += rounds;
    cluster.sync();  // peers may still read our counters
    return;
  }

  if (st.policy == 0) {
    // Default policy: every proposal is fresh (commit_single.cuh), so
    // committed == accepted and touched == matched; classify here and let
    // commit_apply_kernel do the scattered writes grid-wide.
    // Each CTA ranks its edges in shared memory and reserves its range of
    // the committed / queued lists with ONE global atomic (per-warp global
    // atomics on the two counters serialised ~600 deep at L2).
    const int lane = tid & 31;
    for (int32_t base = tid - lane; base < cnt; base += kNT) {
      const int32_t l = base + lane;
      const uint8_t s = l < cnt ? Ea.st[l] : kEdgeUndecided;
      const bool acc = s == kEdgeAccepted;
      const unsigned am = __ballot_sync(0xffffffffu, acc);
      if (am) {
        int r0 = 0;
        if (lane == 0) r0 = atomicAdd(&sc.nlog, __popc(am));
        r0 = __shfl_sync(0xffffffffu, r0, 0);
        if (acc) Ea.rank[l] = r0 + __popc(am & ((1u << lane) - 1));
      }
      if (s == kEdgeRejected && Ea.slot[l] >= n) {
        const int32_t j = Ea.slot[l] - n;
        atomicOr(&st.jbits[j >> 5], 1u << (j & 31));
      }
    }
    __syncthreads();
    if (tid == 0) sc.base_items = sc.nlog ? atomicAdd(&C->k2_nlog, sc.nlog) : 0;
    __syncthreads();
    for (int32_t l = tid; l < cnt; l += kNT)
      if (Ea.st[l] == kEdgeAccepted) st.clist[sc.base_items + Ea.rank[l]] = e0 + l;
    if (rank == 0 && tid == 0) tl_mark(C, st.tl, st.tl_cap, 14);
    // conflicted proposers: unmatched owners of rejected records, queued once
    // (the matched keys are final since the last LFMM barrier)
    for (int32_t base = tid - lane; base < cnt; base += kNT) {
      const int32_t l = base + lane;
      bool q = false;
      if (l < cnt && Ea.st[l] == kEdgeRejected) {
        const int32_t p = Ea.u[l];  // the proposer (the record's owner)
        q = kbase[p % CS][p / CS] != KK::kMatched && !(atomicOr(fbase[p % CS] + p / CS, kQueued) & kQueued);
      }
      const unsigned qm = __ballot_sync(0xffffffffu, q);
      if (qm) {
        int r0 = 0;
        if (lane == 0) r0 = atomicAdd(&sc.nconf, __popc(qm));
        r0 = __shfl_sync(0xffffffffu, r0, 0);
        if (q) Ea.rank[l] = r0 + __popc(qm & ((1u << lane) - 1));
        else if (l < cnt && Ea.st[l] == kEdgeRejected) Ea.rank[l] = kNoEmit;
      } else if (l < cnt && Ea.st[l] == kEdgeRejected) {
        Ea.rank[l] = kNoEmit;
      }
    }
    __syncthreads();
    if (tid == 0) sc.base_conf = sc.nconf ? atomicAdd(&C->k2_nconf, sc.nconf) : 0;
    __syncthreads();
    for (int32_t l = tid; l < cnt; l += kNT)
      if (Ea.st[l] == kEdgeRejected && Ea.rank[l] != kNoEmit) st.qlist[sc.base_conf + Ea.rank[l]] = e0 + l;
    cluster.sync();  // counts final; peers done with this CTA's shared memory
    if (rank == 0 && tid == 0) {
      const int nlog = __ldcg(&C->k2_nlog), nconf = __ldcg(&C->k2_nconf), nitems = 2 * nlog + nconf;
      C->k2_parity = P;
      C->k2_iter = iter;
      C->k2_log_base = C->log_count;
      C->log_count += nlog;
      C->work_count = nitems;
      C->switches += nlog;
      C->pair_items += nitems;
      C->agent_scans += nitems;
      C->job_scans += 2 * nlog;  // + queued proposers with a rejected job record (apply kernel)
      C->iter = iter;
      C->parity = 1 - P;
      C->edge_count[P] = 0;
      C->lfmm_rounds += rounds;
      C->inner_iterations += 1;
      if (!st.dist_vote && C->deadline_gt != 0 && globaltimer() >= C->deadline_gt) C->expired = 1;
      tl_mark(C, st.tl, st.tl_cap, kTlCommitEnd);
    }
    return;
  }

  // ---- P3: select on the frozen assignment; mark touched / rejected ----
  const double eps = st.eps;
  int overlap = 0;
  for (int32_t l = tid; l < cnt; l += kNT) {
    const uint8_t s = Ea.st[l];
    if (s == kEdgeRejected) {
      const int4 en = prop_key(edges[e0 + l], n);
      if (en.x >= n) atomicOr(fbase[en.w % CS] + en.w / CS, kJobRejected);
      continue;
    }
    if (s != kEdgeAccepted) continue;
    const int4 en = prop_key(edges[e0 + l], n);
    int32_t agent, j_new, disp;
    const int32_t j_old = Ea.jold[l];
    if (en.x < n) {  // agent_proposal_delta, solver_state.hpp:106-113
      agent = en.y;
      j_new = en.z;
      disp = Ea.v[l];
      st.agent_delta[agent] = 0.0;
      st.agent_partner[agent] = -1;
    } else {  // job_proposal_delta, solver_state.hpp:115-122 (i_new = agent, holder = disp)
      agent = en.z;
      j_new = en.w;
      disp = en.y;
      st.job_delta[j_new] = 0.0;
      st.job_partner[j_new] = -1;
    }
    const int64_t rn = static_cast<int64_t>(j_new) * ld, ro = static_cast<int64_t>(j_old) * ld;
    const auto a_new = widen(AT[rn + agent]), a_old = widen(AT[ro + agent]);
    const auto d_old = widen(AT[ro + disp]), d_new = widen(AT[rn + disp]);
    const double dact = en.x < n ? static_cast<double>(delta4(a_new, a_old, d_old, d_new))
                                 : static_cast<double>(delta4(a_new, d_new, d_old, a_old));
    if (dact > eps) {
      Ea.st[l] = kEdgeCommitted;
      Ea.u[l] = agent;
      Ea.v[l] = disp;
      Ea.jold[l] = j_old;
      Ea.del[l] = dact;
      Ea.acur_a[l] = static_cast<double>(a_new);
      Ea.acur_d[l] = static_cast<double>(d_old);
      const uint32_t o1 = atomicOr(fbase[agent % CS] + agent / CS, kTouched);
      const uint32_t o2 = atomicOr(fbase[disp % CS] + disp / CS, kTouched);
      if ((o1 | o2) & kTouched) overlap = 1;
    }
  }
  if (overlap) atomicExch(&C->error, 1);
  cluster.sync();
  if (rank == 0 && tid == 0) tl_mark(C, st.tl, st.tl_cap, 13);

  // ---- P4: apply, then rank log entries and work items ----
  for (int32_t l = tid; l < cnt; l += kNT) {
    const uint8_t s = Ea.st[l];
    if (s == kEdgeCommitted) {
      const int32_t agent = Ea.u[l], disp = Ea.v[l], j_old = Ea.jold[l];
      const int4 en = prop_key(edges[e0 + l], n);
      const int32_t j_new = en.x < n ? en.z : en.w;
      st.sigma[j_new] = agent;
      st.sigma[j_old] = disp;
      st.tau[agent] = j_new;
      st.tau[disp] = j_old;
      if (st.tau16) {
        st.tau16[agent] = static_cast<uint16_t>(j_new);
        st.tau16[disp] = static_cast<uint16_t>(j_old);
      }
      acur[agent] = static_cast<E>(Ea.acur_a[l]);
      acur[disp] = static_cast<E>(Ea.acur_d[l]);
      Ea.rank[l] = atomicAdd(&sc.nlog, 1);
    } else if (s == kEdgeRejected) {
      const int4 en = prop_key(edges[e0 + l], n);
      const int32_t p = en.y;  // the proposer (frozen holder for job-side proposals)
      uint32_t* fp = fbase[p % CS] + p / CS;
      if (st.policy == 0) {
        if (!(*fp & kTouched) && !(atomicOr(fp, kQueued) & kQueued)) {
          // p is untouched, so its job is still the proposal's job en.w
          const bool jflag = (fbase[en.w % CS][en.w / CS] & kJobRejected) != 0;
          Ea.rank[l] = atomicAdd(&sc.nconf, 1) | (jflag ? kJobFlagBit : 0);
          if (jflag) atomicAdd(&sc.nconf_j, 1);
        }
      } else if (!(*fp & kTouched)) {
        // touched_only: an untouched proposer keeps its stale record -> carry it
        const int pos = atomicAdd(&C->edge_count[1 - P], 1);
        st.edges[1 - P][pos] = edges[e0 + l];
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    const int nlog = sc.nlog, nitems = 2 * sc.nlog + sc.nconf;
    sc.base_log = nlog ? atomicAdd(reinterpret_cast<unsigned long long*>(&C->log_count),
                                   static_cast<unsigned long long>(nlog))
                       : 0ull;
    sc.base_items = nitems ? atomicAdd(&C->work_count, nitems) : 0;
    if (nlog) atomicAdd(reinterpret_cast<unsigned long long*>(&C->switches), static_cast<unsigned long long>(nlog));
    if (nitems) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&C->pair_items), static_cast<unsigned long long>(nitems));
      atomicAdd(reinterpret_cast<unsigned long long*>(&C->agent_scans), static_cast<unsigned long long>(nitems));
      atomicAdd(reinterpret_cast<unsigned long long*>(&C->job_scans),
                static_cast<unsigned long long>(2 * sc.nlog + sc.nconf_j));
    }
  }
  __syncthreads();
  const unsigned long long blog = sc.base_log;
  const int bitems = sc.base_items, nlog2 = 2 * sc.nlog;
  for (int32_t l = tid; l < cnt; l += kNT) {
    const int32_t r = Ea.rank[l];
    if (r == kNoEmit) continue;
    if (Ea.st[l] == kEdgeCommitted) {
      st.log[blog + r] = LogEntry{iter, edges[e0 + l].slot, Ea.del[l]};
      st.items[bitems + 2 * r] = static_cast<uint32_t>(Ea.u[l]) | kItemAgent | kItemJob;
      st.items[bitems + 2 * r + 1] = static_cast<uint32_t>(Ea.v[l]) | kItemAgent | kItemJob;
    } else {
      const int32_t p = prop_key(edges[e0 + l], n).y;
      st.items[bitems + nlog2 + (r & ~kJobFlagBit)] =
          static_cast<uint32_t>(p) | kItemAgent | ((r & kJobFlagBit) ? kItemJob : 0u);
    }
  }
  if (rank == 0 && tid == 0) tl_mark(C, st.tl, st.tl_cap, 14);
  cluster.sync();  // every peer is done with this CTA's shared memory
  if (rank == 0 && tid == 0) {
    C->k2_nlog = C->k2_nconf = 0;  // the apply kernel has nothing left to do
    C->iter = iter;
    C->parity = 1 - P;
    C->edge_count[P] = 0;
    C->lfmm_rounds += rounds;
    C->inner_iterations += 1;
    // anytime deadline, acted on by the next commit (solver_state.hpp:13-27)
    if (!st.dist_vote && C->deadline_gt != 0 && globaltimer() >= C->deadline_gt) C->expired = 1;
    tl_mark(C, st.tl, st.tl_cap, kTlCommitEnd);
  }
}

template <class E, int CS>
cudaError_t launch_cs(const DevState& d, const CommitPlan& p, int mode, cudaGraphConditionalHandle cond,
                      int use_cond, cudaStream_t st) {
  auto k = p.wide_keys ? commit_cluster_kernel<E, CS, true> : commit_cluster_kernel<E, CS, false>;
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
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = d.pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, k, d, mode, cond, use_cond, p.edge_cap, p.cta_edge_cap, p.variant);
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
  auto k = commit_cluster_kernel<int32_t, 16, false>;
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
