// commit_apply.cuh -- the scattered writes of one batch under the split
// commit (select / apply / re-evaluation items, parallel.cpp:276-330), as a
// device function run by every thread of commit_apply_kernel (commit.cu),
// which follows the conflict check on 64 SMs.
#pragma once

#include "state.h"

namespace lsapgpu {

// Thread `gt` of `gn`: committed exchanges (clist) then queued conflicted
// proposers (qlist) of the batch described by the k2_* control fields.
template <class E>
__device__ __forceinline__ void apply_batch(const DevState& st, int64_t gt, int64_t gn) {
  Ctrl* C = st.ctrl;
  const int32_t nlog = __ldcg(&C->k2_nlog), nconf = __ldcg(&C->k2_nconf);
  if (nlog + nconf == 0) return;
  const int32_t n = st.n;
  const Prop* edges = st.edges[__ldcg(&C->k2_parity)];
  const int32_t iter = __ldcg(&C->k2_iter);
  const int64_t base = __ldcg(&C->k2_log_base);
  E* acur = static_cast<E*>(st.acur);
  int jobs = 0;
  for (int64_t x = gt; x < nlog + nconf; x += gn) {
    if (x < nlog) {
      const Prop p = edges[__ldcg(st.clist + x)];
      if (p.slot < n) {
        st.agent_delta[p.a] = 0.0;
        st.agent_partner[p.a] = -1;
      } else {
        st.job_delta[p.j_new] = 0.0;
        st.job_partner[p.j_new] = -1;
      }
      st.sigma[p.j_new] = p.a;
      st.sigma[p.j_old] = p.d;
      st.tau[p.a] = p.j_new;
      st.tau[p.d] = p.j_old;
      if (st.tau16) {
        st.tau16[p.a] = static_cast<uint16_t>(p.j_new);
        st.tau16[p.d] = static_cast<uint16_t>(p.j_old);
      }
      acur[p.a] = static_cast<E>(p.acur_a);
      acur[p.d] = static_cast<E>(p.acur_d);
      st.log[base + x] = LogEntry{iter, p.slot, p.delta};
      st.items[2 * x] = static_cast<uint32_t>(p.a) | kItemAgent | kItemJob;
      st.items[2 * x + 1] = static_cast<uint32_t>(p.d) | kItemAgent | kItemJob;
    } else {
      const int64_t q = x - nlog;
      const Prop p = edges[__ldcg(st.qlist + q)];
      const int32_t owner = p.slot < n ? p.a : p.d;
      const int32_t job = p.slot < n ? p.j_old : p.j_new;  // the owner's (unchanged) job
      const bool jflag = (__ldcg(st.jbits + (job >> 5)) >> (job & 31)) & 1u;
      st.items[2 * nlog + q] = static_cast<uint32_t>(owner) | kItemAgent | (jflag ? kItemJob : 0u);
      jobs += jflag;
    }
  }
  for (int off = 16; off > 0; off >>= 1) jobs += __shfl_down_sync(0xffffffffu, jobs, off);
  if ((threadIdx.x & 31) == 0 && jobs)
    atomicAdd(reinterpret_cast<unsigned long long*>(&C->job_scans), static_cast<unsigned long long>(jobs));
}

}  // namespace lsapgpu
