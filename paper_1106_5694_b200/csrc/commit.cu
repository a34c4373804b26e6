// commit.cu -- step-API kernels around the commit phase:
//   * edges_from_tables: proposals {slot, a, b, c} from full SoA tables (the
//     check_conflicts / apply_parallel_switches step APIs take tables, not a
//     scan's output), in the layout the pair scan emits;
//   * apply_kernel: lsap::apply_parallel_switches (parallel.cpp:182-229) for
//     caller-given acceptance masks: improvements recomputed on the frozen
//     assignment (solver_state.hpp:106-122), committed iff > eps, applied
//     concurrently (they are disjoint; overlap is asserted like the
//     reference's "internal: conflict check admitted overlapping exchanges").
//
// The conflict check itself (parallel.cpp:35-76) is computed exactly by the
// cluster kernel in commit_cluster.cu: check_conflicts_impl walks agent
// proposals in ascending index order, then job proposals in ascending order,
// and accepts a proposal iff neither agent endpoint is reserved yet.  That is
// the lexicographically-first maximal matching (LFMM) of the proposal graph
// under priority slot (= i for agent proposals, n + j for job proposals).
// Parallel rounds reproduce it: every undecided edge posts its priority to
// both endpoints, an edge that is the minimum at both endpoints is accepted
// and matches them, edges touching a matched vertex are rejected.  The minimum
// remaining edge is always accepted, and an accepted edge has no undecided
// earlier neighbour (every earlier neighbour was rejected by an earlier
// accepted edge), so by induction the accepted set, the rejected set and hence
// reserved / conflicted / conflicted_jobs equal the sequential walk's.
#include <climits>

#include "state.h"

namespace lsapgpu {
namespace {

constexpr uint8_t kEdgeCommitted = 4;

__global__ void tau_from_sigma_kernel(DevState st) {
  for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < st.n; j += gridDim.x * blockDim.x)
    st.tau[st.sigma[j]] = j;
}

// every slot with delta > 0 and partner >= 0 becomes a proposal entry
__global__ void edges_from_tables_kernel(DevState st) {
  const int32_t n = st.n;
  const int P = st.ctrl->parity;
  for (int32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < 2 * n; s += gridDim.x * blockDim.x) {
    int4 en;
    bool active;
    if (s < n) {
      active = st.agent_partner[s] >= 0 && st.agent_delta[s] > 0.0;
      en = make_int4(s, s, st.agent_partner[s], st.tau[s]);
    } else {
      const int32_t j = s - n;
      active = st.job_partner[j] >= 0 && st.job_delta[j] > 0.0;
      en = make_int4(s, st.sigma[j], st.job_partner[j], j);
    }
    if (active) {
      const int pos = atomicAdd(&st.ctrl->edge_count[P], 1);
      st.edges[P][pos] = en;
    }
  }
}

template <class E>
__global__ void __launch_bounds__(1024, 1)
    apply_kernel(DevState st, const uint8_t* acc_agent, const uint8_t* acc_job) {
  __shared__ int s_committed;
  Ctrl* C = st.ctrl;
  const int32_t n = st.n;
  const int tid = threadIdx.x, NT = blockDim.x;
  const E* A = static_cast<const E*>(st.A);
  E* acur = static_cast<E*>(st.acur);
  const int64_t ld = st.ld;
  const int P = C->parity;
  const int32_t m = C->edge_count[P];
  const int4* edges = st.edges[P];
  const int32_t iter = C->iter + 1;
  if (tid == 0) s_committed = 0;

  // select on the frozen assignment
  for (int32_t e = tid; e < m; e += NT) {
    const int4 en = edges[e];
    st.estate[e] = kEdgeUndecided;
    if (!(en.x < n ? acc_agent[en.x] : acc_job[en.x - n])) continue;
    int32_t agent, j_new, j_old, disp;
    if (en.x < n) {
      agent = en.y;
      j_new = en.z;
      j_old = en.w;
      disp = st.sigma[j_new];
    } else {
      agent = en.z;
      j_new = en.w;
      disp = en.y;
      j_old = st.tau[agent];
    }
    const int64_t ra = static_cast<int64_t>(agent) * ld, rd = static_cast<int64_t>(disp) * ld;
    typename Traits<E>::Acc actual;
    if (en.x < n)
      actual = delta4(widen(A[ra + j_new]), widen(A[ra + j_old]), widen(A[rd + j_old]),
                      widen(A[rd + j_new]));
    else
      actual = delta4(widen(A[ra + j_new]), widen(A[rd + j_new]), widen(A[rd + j_old]),
                      widen(A[ra + j_old]));
    const double dact = static_cast<double>(actual);
    if (dact > st.eps) {
      st.estate[e] = kEdgeCommitted;
      st.eu[e] = agent;
      st.ev[e] = disp;
      st.eprop[e] = j_old;
      st.c_jnew[e] = j_new;
      st.c_delta[e] = dact;
    }
  }
  __syncthreads();
  int local = 0;
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
    const unsigned long long pos = atomicAdd(reinterpret_cast<unsigned long long*>(&C->log_count), 1ull);
    st.log[pos] = LogEntry{iter, edges[e].x, st.c_delta[e]};
    ++local;
  }
  if (local) atomicAdd(&s_committed, local);
  __syncthreads();
  if (tid == 0) {
    C->switches += s_committed;
    C->iter = iter;
  }
}

}  // namespace

CommitPlan plan_commit(const DevState& d) {
  CommitPlan p;
  // cluster kernel: key + flag slices and as many 45-byte proposal slots as fit
  const size_t budget = 220 * 1024;
  p.cluster_smem = budget;
  p.cluster = commit_cluster_size(d, budget);
  const size_t kslice = ((static_cast<size_t>(d.n) + p.cluster - 1) / p.cluster * 4 + 15) / 16 * 16;
  const size_t cap = budget > 2 * kslice + 64 ? (budget - 2 * kslice - 64) / 45 : 0;
  p.edge_cap = static_cast<int>(cap / 16 * 16);
  return p;
}

cudaError_t launch_commit(const DevState& d, const CommitPlan& p, int mode,
                          cudaGraphConditionalHandle cond, int use_cond, cudaStream_t st) {
  if (mode == kCommitApplyOnly) return cudaErrorInvalidValue;  // launch_accepted_from_masks
  return launch_commit_cluster(d, p, mode, cond, use_cond, st);
}

cudaError_t launch_edges_from_tables(const DevState& d, cudaStream_t st) {
  tau_from_sigma_kernel<<<64, 256, 0, st>>>(d);
  edges_from_tables_kernel<<<256, 256, 0, st>>>(d);
  return cudaGetLastError();
}

cudaError_t launch_accepted_from_masks(const DevState& d, const uint8_t* agent_acc,
                                       const uint8_t* job_acc, cudaStream_t st) {
  switch (d.storage) {
    case kI16: apply_kernel<int16_t><<<1, 1024, 0, st>>>(d, agent_acc, job_acc); break;
    case kI32: apply_kernel<int32_t><<<1, 1024, 0, st>>>(d, agent_acc, job_acc); break;
    case kF32: apply_kernel<float><<<1, 1024, 0, st>>>(d, agent_acc, job_acc); break;
    case kF64: apply_kernel<double><<<1, 1024, 0, st>>>(d, agent_acc, job_acc); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace lsapgpu
