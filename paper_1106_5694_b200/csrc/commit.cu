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
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "commit_single.cuh"
#include "commit_apply.cuh"
#include "state.h"

namespace lsapgpu {
namespace {

constexpr uint8_t kEdgeCommitted = 4;

__global__ void tau_from_sigma_kernel(DevState st) {
  for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < st.n; j += gridDim.x * blockDim.x) {
    st.tau[st.sigma[j]] = j;
    if (st.tau16) st.tau16[st.sigma[j]] = static_cast<uint16_t>(j);
  }
}

// every slot with delta > 0 and partner >= 0 becomes a proposal entry (the
// step APIs check conflicts without an instance: no entries of A are read;
// apply_kernel recomputes the exchanges from the instance it is given)
__global__ void edges_from_tables_kernel(DevState st) {
  const int32_t n = st.n;
  const int P = st.ctrl->parity;
  for (int32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < 2 * n; s += gridDim.x * blockDim.x) {
    if (s < n) {
      if (!(st.agent_partner[s] >= 0 && st.agent_delta[s] > 0.0)) continue;
      const int pos = atomicAdd(&st.ctrl->edge_count[P], 1);
      st.edges[P][pos] = agent_prop(st.sigma, st.tau, nullptr, st.storage, st.ld, s, st.agent_partner[s],
                                    st.agent_delta[s]);
    } else {
      const int32_t j = s - n;
      if (!(st.job_partner[j] >= 0 && st.job_delta[j] > 0.0)) continue;
      const int pos = atomicAdd(&st.ctrl->edge_count[P], 1);
      st.edges[P][pos] = job_prop(st.sigma, st.tau, nullptr, st.storage, st.ld, n, j, st.job_partner[j],
                                  st.job_delta[j]);
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
  const Prop* edges = st.edges[P];
  const int32_t iter = C->iter + 1;
  if (tid == 0) s_committed = 0;

  // select on the frozen assignment
  for (int32_t e = tid; e < m; e += NT) {
    const int4 en = prop_key(edges[e], n);
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
    if (st.tau16) {
      st.tau16[agent] = static_cast<uint16_t>(j_new);
      st.tau16[disp] = static_cast<uint16_t>(j_old);
    }
    acur[agent] = A[static_cast<int64_t>(agent) * ld + j_new];
    acur[disp] = A[static_cast<int64_t>(disp) * ld + j_old];
    const unsigned long long pos = atomicAdd(reinterpret_cast<unsigned long long*>(&C->log_count), 1ull);
    st.log[pos] = LogEntry{iter, edges[e].slot, st.c_delta[e]};
    ++local;
  }
  if (local) atomicAdd(&s_committed, local);
  __syncthreads();
  if (tid == 0) {
    C->switches += s_committed;
    C->iter = iter;
  }
}

// Grid-wide second half of the split commit (commit_single.cuh): apply the
// committed exchanges in any order (they are disjoint), append their delta-log
// entries at the reserved positions (the host orders the log by (iter,
// slot)), and write the re-evaluation items: both agents of every committed
// exchange, then every queued conflicted proposer with its job when the job's
// own record was rejected (parallel.cpp:296-330).
template <class E>
__global__ void __launch_bounds__(256) commit_apply_kernel(DevState st) {
  pdl_trigger();
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0) tl_mark(st.ctrl, st.tl, st.tl_cap, 15);
  apply_batch<E>(st, static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
                 static_cast<int64_t>(gridDim.x) * blockDim.x);
}

}  // namespace

cudaError_t launch_commit_apply(const DevState& d, cudaStream_t st) {
  static const unsigned ctas = [] {
    const char* e = std::getenv("LSAPGPU_APPLY_CTAS");
    return e ? static_cast<unsigned>(std::max(1, std::atoi(e))) : 64u;
  }();
  switch (d.storage) {
    case kI16: return launch_pdl(commit_apply_kernel<int16_t>, dim3(ctas), dim3(256), 0, st, d.pdl, d);
    case kI32: return launch_pdl(commit_apply_kernel<int32_t>, dim3(ctas), dim3(256), 0, st, d.pdl, d);
    case kF32: return launch_pdl(commit_apply_kernel<float>, dim3(ctas), dim3(256), 0, st, d.pdl, d);
    case kF64: return launch_pdl(commit_apply_kernel<double>, dim3(ctas), dim3(256), 0, st, d.pdl, d);
    default: return cudaErrorInvalidValue;
  }
}

CommitPlan plan_commit(const DevState& d) {
  CommitPlan p;
  // cluster kernel: key + flag slices and as many 45-byte proposal slots as fit
  const size_t budget = 220 * 1024;
  p.cluster_smem = budget;
  p.cluster = commit_cluster_size(d, budget);
  if (const char* s = std::getenv("LSAPGPU_COMMIT_CS")) p.cluster = std::atoi(s) == 8 ? 8 : p.cluster;
  p.wide_keys = d.n >= (1 << 17) ? 1 : 0;  // slots 0..2n-1 no longer fit the 18-bit field
  if (const char* s = std::getenv("LSAPGPU_LFMM_WIDE")) p.wide_keys = p.wide_keys || std::atoi(s) != 0;
  const size_t slice = (static_cast<size_t>(d.n) + p.cluster - 1) / p.cluster;
  const size_t kslice = 2 * ((slice * 4 + 15) / 16 * 16);  // keys + flags
  const size_t cap = budget > kslice + 64 ? (budget - kslice - 64) / 45 : 0;
  p.edge_cap = static_cast<int>(cap / 16 * 16);
  // split commit (commit_single.cuh): per-agent keys + rejected-job bitmap,
  // 13 B per proposal, in one CTA's shared memory
  // One SM's atomic and load/store throughput makes the split commit slower
  // than the cluster for the large early batches; it wins below a few
  // thousand proposals (measured on B200, C2/C3: 2k-6k best).
  p.cta_edge_cap = std::min(single::edge_capacity(d.n, budget), 4096);
  if (p.cta_edge_cap < 1024) p.cta_edge_cap = 0;
  if (const char* s = std::getenv("LSAPGPU_COMMIT_SINGLE"))
    if (std::atoi(s) == 0) p.cta_edge_cap = 0;
  if (const char* s = std::getenv("LSAPGPU_COMMIT_SINGLE_MAX")) p.cta_edge_cap = std::min(p.cta_edge_cap, std::atoi(s));
  if (const char* s = std::getenv("LSAPGPU_COMMIT_VARIANT")) p.variant = std::atoi(s);
  return p;
}

cudaError_t launch_commit(const DevState& d, const CommitPlan& p, int mode,
                          cudaGraphConditionalHandle cond, int use_cond, cudaStream_t st) {
  if (mode == kCommitApplyOnly) return cudaErrorInvalidValue;  // launch_accepted_from_masks
  cudaError_t e = launch_commit_cluster(d, p, mode, cond, use_cond, st);
  if (e != cudaSuccess || mode != kCommitSolve) return e;
  return launch_commit_apply(d, st);
}

__global__ void tau16_sync_kernel(DevState st) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < st.n; i += gridDim.x * blockDim.x)
    st.tau16[i] = static_cast<uint16_t>(st.tau[i]);
}

cudaError_t launch_tau16_sync(const DevState& d, cudaStream_t st) {
  if (!d.tau16) return cudaSuccess;
  tau16_sync_kernel<<<64, 256, 0, st>>>(d);
  return cudaGetLastError();
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
