// commit.cu -- one inner iteration of the reference's batch loop
// (proj/src/parallel.cpp:264-335) minus the scans: conflict check, select,
// apply and re-evaluation list, as one single-CTA kernel.
//
// Conflict check.  check_conflicts_impl (parallel.cpp:35-76) walks agent
// proposals in ascending index order, then job proposals in ascending order,
// and accepts a proposal iff neither agent endpoint is already reserved.  That
// is the lexicographically-first maximal matching (LFMM) of the proposal
// graph under priority slot = i (agent side) / n + j (job side).  It is
// computed here exactly with parallel rounds: every undecided edge posts its
// priority to both endpoints (atomicMax of an epoch-tagged inverted key), an
// edge that is the minimum at both endpoints is accepted and matches them,
// and edges touching a matched vertex are rejected.  The minimum remaining
// edge is always accepted, and an accepted edge has no undecided earlier
// neighbour, so the result equals the sequential walk's.
//
// Select/apply (parallel.cpp:276-310): accepted records are zeroed, the
// improvement is recomputed against the frozen assignment
// (solver_state.hpp:106-122) and committed iff > eps.  Committed exchanges are
// pairwise disjoint, so they are applied concurrently; each appends
// (iteration, slot, delta) to the delta log, from which the host rebuilds the
// reference's ordered value accumulation and objective trace.  The
// disjointness assertion (parallel.cpp:296-302) is kept as an atomic stamp
// check.  Re-evaluation (parallel.cpp:312-330) becomes a work list of agents,
// each item also carrying its job when that job needs a fresh record.
#include <climits>

#include "state.h"

namespace lsapgpu {
namespace {

constexpr uint8_t kEdgeCommitted = 4;
constexpr uint32_t kMatched = 0xFFFFFFFFu;
constexpr uint32_t kKeyShift = 18;            // priorities (slots) < 2^18
constexpr uint32_t kRoundLimit = (1u << 14) - 2;

__device__ __forceinline__ uint32_t make_key(uint32_t round, int32_t slot) {
  return (round << kKeyShift) | (0x3FFFFu - static_cast<uint32_t>(slot));
}

__device__ __forceinline__ int block_sum(int v, int* scratch) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  if ((threadIdx.x & 31) == 0) atomicAdd(scratch, v);
  return v;
}

template <class E>
__global__ void __launch_bounds__(1024, 1)
    commit_kernel(DevState st, int mode, cudaGraphConditionalHandle cond, int use_cond,
                  int keys_in_smem, const uint8_t* acc_agent, const uint8_t* acc_job) {
  extern __shared__ uint32_t skeys[];
  __shared__ int s_cnt, s_items, s_committed, s_ascans, s_jscans, s_abort;
  Ctrl* C = st.ctrl;
  const int32_t n = st.n;
  const int tid = threadIdx.x, NT = blockDim.x;
  const E* A = static_cast<const E*>(st.A);
  E* acur = static_cast<E*>(st.acur);
  const int64_t ld = st.ld;

  const int P = C->parity;
  const int32_t m = C->edge_count[P];
  int32_t* edges = st.edges[P];

  if (tid == 0) {
    s_abort = 0;
    if (mode == kCommitSolve) {
      if (C->expired || C->drain || C->error || C->inner_done) {
        s_abort = 1;
      } else if (m == 0) {
        C->inner_done = 1;
        s_abort = 1;
      } else if (C->deadline_gt != 0 && globaltimer() >= C->deadline_gt) {
        C->expired = 1;
        s_abort = 1;
      } else if (C->log_count + m > st.log_cap) {
        C->drain = 1;
        s_abort = 1;
      }
      if (s_abort) {
        C->work_count = 0;
        if (use_cond) cudaGraphSetConditional(cond, 0);
      }
    }
    s_cnt = 0;
    s_items = 0;
    s_committed = 0;
    s_ascans = 0;
    s_jscans = 0;
  }
  __syncthreads();
  if (s_abort) return;

  const int32_t iter = C->iter + 1;
  uint32_t R = C->round;
  uint32_t* keys = keys_in_smem ? skeys : st.keys;
  if (keys_in_smem)
    for (int32_t x = tid; x < n; x += NT) keys[x] = 0;

  // ---- endpoints of every proposal (agent ids), from the frozen sigma ----
  for (int32_t e = tid; e < m; e += NT) {
    const int32_t slot = edges[e];
    int32_t u, v;
    bool valid;
    if (slot < n) {
      const int32_t part = st.agent_partner[slot];
      valid = part >= 0 && st.agent_delta[slot] > 0.0;
      u = slot;
      v = valid ? st.sigma[part] : -1;
    } else {
      const int32_t j = slot - n;
      const int32_t part = st.job_partner[j];
      valid = part >= 0 && st.job_delta[j] > 0.0;
      u = st.sigma[j];
      v = part;
    }
    if (mode == kCommitApplyOnly)
      valid = valid && (slot < n ? acc_agent[slot] : acc_job[slot - n]);
    st.eu[e] = u;
    st.ev[e] = v;
    st.eprop[e] = u;  // proposer: the agent, or the job's current holder
    st.estate[e] = valid ? (mode == kCommitApplyOnly ? kEdgeAccepted : kEdgeUndecided) : kEdgeNone;
  }
  __syncthreads();

  // ---- LFMM rounds (skipped in apply-only mode) ----
  int rounds = 0;
  if (mode != kCommitApplyOnly) {
    for (;;) {
      if (R >= kRoundLimit) {  // key epoch wrap: keep matches, clear priorities
        for (int32_t x = tid; x < n; x += NT)
          if (keys[x] != kMatched) keys[x] = 0;
        R = 1;
        __syncthreads();
      }
      if (tid == 0) s_cnt = 0;
      __syncthreads();
      int local = 0;
      for (int32_t e = tid; e < m; e += NT) {
        if (st.estate[e] != kEdgeUndecided) continue;
        const int32_t u = st.eu[e], v = st.ev[e];
        if (keys[u] == kMatched || keys[v] == kMatched) {
          st.estate[e] = kEdgeRejected;
        } else {
          const uint32_t k = make_key(R, edges[e]);
          atomicMax(&keys[u], k);
          atomicMax(&keys[v], k);
          ++local;
        }
      }
      block_sum(local, &s_cnt);
      __syncthreads();
      if (s_cnt == 0) break;
      for (int32_t e = tid; e < m; e += NT) {
        if (st.estate[e] != kEdgeUndecided) continue;
        const int32_t u = st.eu[e], v = st.ev[e];
        const uint32_t k = make_key(R, edges[e]);
        if (keys[u] == k && keys[v] == k) {
          st.estate[e] = kEdgeAccepted;
          keys[u] = kMatched;
          keys[v] = kMatched;
        }
      }
      __syncthreads();
      ++R;
      ++rounds;
    }
  }
  if (mode == kCommitCheckOnly) {
    __syncthreads();
    if (!keys_in_smem)
      for (int32_t e = tid; e < m; e += NT)
        if (st.estate[e] == kEdgeAccepted) {
          keys[st.eu[e]] = 0;
          keys[st.ev[e]] = 0;
        }
    if (tid == 0) {
      C->round = R;
      C->lfmm_rounds += rounds;
    }
    return;
  }

  // ---- select: recompute accepted improvements on the frozen state ----
  const double eps = st.eps;
  for (int32_t e = tid; e < m; e += NT) {
    if (st.estate[e] != kEdgeAccepted) continue;
    const int32_t slot = edges[e];
    int32_t agent, j_new, j_old, disp;
    typename Traits<E>::Acc actual;
    if (slot < n) {  // agent_proposal_delta, solver_state.hpp:106-113
      agent = slot;
      j_new = st.agent_partner[slot];
      if (mode == kCommitSolve) {
        st.agent_delta[slot] = 0.0;
        st.agent_partner[slot] = -1;
      }
      j_old = st.tau[agent];
      disp = st.sigma[j_new];
      const int64_t ra = static_cast<int64_t>(agent) * ld, rd = static_cast<int64_t>(disp) * ld;
      actual = delta4(widen(A[ra + j_new]), widen(A[ra + j_old]), widen(A[rd + j_old]),
                      widen(A[rd + j_new]));
    } else {  // job_proposal_delta, solver_state.hpp:115-122
      const int32_t j = slot - n;
      agent = st.job_partner[j];
      j_new = j;
      if (mode == kCommitSolve) {
        st.job_delta[j] = 0.0;
        st.job_partner[j] = -1;
      }
      disp = st.sigma[j];
      j_old = st.tau[agent];
      const int64_t ri = static_cast<int64_t>(agent) * ld, rh = static_cast<int64_t>(disp) * ld;
      actual = delta4(widen(A[ri + j]), widen(A[rh + j]), widen(A[rh + j_old]),
                      widen(A[ri + j_old]));
    }
    const double dact = static_cast<double>(actual);
    if (dact > eps) {
      st.estate[e] = kEdgeCommitted;
      st.eu[e] = agent;
      st.ev[e] = disp;
      st.eprop[e] = j_old;
      st.c_jnew[e] = j_new;
      st.c_delta[e] = dact;
    }
  }
  __syncthreads();

  // ---- apply (disjoint by construction; asserted) ----
  int local_committed = 0;
  for (int32_t e = tid; e < m; e += NT) {
    if (st.estate[e] != kEdgeCommitted) continue;
    const int32_t agent = st.eu[e], disp = st.ev[e], j_old = st.eprop[e], j_new = st.c_jnew[e];
    if (atomicExch(&st.touched_stamp[agent], iter) == iter ||
        atomicExch(&st.touched_stamp[disp], iter) == iter)
      atomicExch(&C->error, 1);
    st.sigma[j_new] = agent;
    st.sigma[j_old] = disp;
    st.tau[agent] = j_new;
    st.tau[disp] = j_old;
    acur[agent] = A[static_cast<int64_t>(agent) * ld + j_new];
    acur[disp] = A[static_cast<int64_t>(disp) * ld + j_old];
    const unsigned long long pos =
        atomicAdd(reinterpret_cast<unsigned long long*>(&C->log_count), 1ull);
    st.log[pos] = LogEntry{iter, edges[e], st.c_delta[e]};
    ++local_committed;
    if (mode == kCommitSolve) {
      const int w = atomicAdd(&s_items, 2);
      st.items[w] = static_cast<uint32_t>(agent) | kItemAgent | kItemJob;
      st.items[w + 1] = static_cast<uint32_t>(disp) | kItemAgent | kItemJob;
    }
  }
  block_sum(local_committed, &s_committed);
  if (mode == kCommitApplyOnly) {
    __syncthreads();
    if (tid == 0) {
      C->switches += s_committed;
      C->iter = iter;
    }
    return;
  }
  for (int32_t e = tid; e < m; e += NT)
    if (st.estate[e] == kEdgeRejected) st.rej_stamp[edges[e]] = iter;
  __syncthreads();

  // ---- re-evaluation list (parallel.cpp:312-330) / carried edges ----
  int local_a = 0, local_j = 0;
  for (int32_t e = tid; e < m; e += NT) {
    if (st.estate[e] != kEdgeRejected) continue;
    const int32_t slot = edges[e];
    const int32_t p = st.eprop[e];
    if (st.policy == 0) {
      if (st.touched_stamp[p] != iter && atomicExch(&st.conf_stamp[p], iter) != iter) {
        const bool jflag = st.rej_stamp[n + st.tau[p]] == iter;
        const int w = atomicAdd(&s_items, 1);
        st.items[w] = static_cast<uint32_t>(p) | kItemAgent | (jflag ? kItemJob : 0u);
        ++local_a;
        if (jflag) ++local_j;
      }
    } else {
      const int32_t holder = slot < n ? slot : st.sigma[slot - n];
      if (st.touched_stamp[holder] != iter) {
        const int pos = atomicAdd(&C->edge_count[1 - P], 1);
        st.edges[1 - P][pos] = slot;
      }
    }
  }
  block_sum(local_a, &s_ascans);
  block_sum(local_j, &s_jscans);
  if (!keys_in_smem) {
    __syncthreads();
    for (int32_t e = tid; e < m; e += NT) {
      const uint8_t s = st.estate[e];
      if (s == kEdgeAccepted || s == kEdgeCommitted) {
        // eu/ev were rewritten for committed edges but still name the endpoints
        keys[st.eu[e]] = 0;
        keys[st.ev[e]] = 0;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    const int touched = 2 * s_committed;
    C->work_count = s_items;
    C->iter = iter;
    C->round = R;
    C->parity = 1 - P;
    C->edge_count[P] = 0;
    C->switches += s_committed;
    C->pair_items += s_items;
    C->agent_scans += touched + s_ascans;
    C->job_scans += touched + s_jscans;
    C->lfmm_rounds += rounds;
    C->inner_iterations += 1;
  }
}

// Edges from full tables (step API check_conflicts / apply): every slot with
// delta > 0 and partner >= 0, in slot order.
__global__ void edges_from_tables_kernel(DevState st) {
  const int32_t n = st.n;
  for (int32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < 2 * n; s += gridDim.x * blockDim.x) {
    const bool active = s < n ? (st.agent_partner[s] >= 0 && st.agent_delta[s] > 0.0)
                              : (st.job_partner[s - n] >= 0 && st.job_delta[s - n] > 0.0);
    if (active) {
      const int pos = atomicAdd(&st.ctrl->edge_count[st.ctrl->parity], 1);
      st.edges[st.ctrl->parity][pos] = s;
    }
  }
}

template <class E>
cudaError_t launch_t(const DevState& d, const CommitPlan& p, int mode,
                     cudaGraphConditionalHandle cond, int use_cond, const uint8_t* aa,
                     const uint8_t* ja, cudaStream_t st) {
  auto k = commit_kernel<E>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(p.smem));
  if (e != cudaSuccess) return e;
  k<<<1, p.threads, p.smem, st>>>(d, mode, cond, use_cond, p.keys_in_smem ? 1 : 0, aa, ja);
  return cudaGetLastError();
}

cudaError_t launch_any(const DevState& d, const CommitPlan& p, int mode,
                       cudaGraphConditionalHandle cond, int use_cond, const uint8_t* aa,
                       const uint8_t* ja, cudaStream_t st) {
  switch (d.storage) {
    case kI16: return launch_t<int16_t>(d, p, mode, cond, use_cond, aa, ja, st);
    case kI32: return launch_t<int32_t>(d, p, mode, cond, use_cond, aa, ja, st);
    case kF32: return launch_t<float>(d, p, mode, cond, use_cond, aa, ja, st);
    case kF64: return launch_t<double>(d, p, mode, cond, use_cond, aa, ja, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

CommitPlan plan_commit(const DevState& d) {
  CommitPlan p;
  p.threads = 1024;
  const size_t kb = static_cast<size_t>(d.n) * sizeof(uint32_t);
  p.keys_in_smem = kb <= 200 * 1024;
  p.smem = p.keys_in_smem ? kb : 0;
  return p;
}

cudaError_t launch_commit(const DevState& d, const CommitPlan& p, int mode,
                          cudaGraphConditionalHandle cond, int use_cond, cudaStream_t st) {
  return launch_any(d, p, mode, cond, use_cond, nullptr, nullptr, st);
}

cudaError_t launch_edges_from_tables(const DevState& d, cudaStream_t st) {
  edges_from_tables_kernel<<<256, 256, 0, st>>>(d);
  return cudaGetLastError();
}

cudaError_t launch_accepted_from_masks(const DevState& d, const uint8_t* agent_acc,
                                       const uint8_t* job_acc, cudaStream_t st) {
  return launch_any(d, plan_commit(d), kCommitApplyOnly, 0, 0, agent_acc, job_acc, st);
}

}  // namespace lsapgpu
