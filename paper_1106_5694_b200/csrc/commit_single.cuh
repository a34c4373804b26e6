// commit_single.cuh -- the split commit used under the default re-evaluation
// policy (touched_and_conflicted) whenever the batch's vertex state fits one
// SM: the conflict check of one inner iteration (parallel.cpp:35-76) runs in
// ONE CTA with every per-vertex structure in its own shared memory, and the
// scattered writes of select / apply / re-evaluation items
// (parallel.cpp:276-330) run grid-wide in commit_apply_kernel.
//
// Why this is exact.  Under touched_and_conflicted every active record of a
// batch was computed by the scan that ran on this batch's frozen state: the
// previous batch zeroed every accepted record and re-evaluated every touched
// and every conflicted record, so no record survives a batch without being
// rescanned (the full sweep covers the first batch of a pass).  Each
// proposal (Prop) therefore carries the fresh exchange: its delta equals the
// improvement agent_proposal_delta / job_proposal_delta recomputes
// (solver_state.hpp:106-122: the same four entries in the same fp64 order),
// so the select guard `actual > eps` holds for every accepted proposal,
// committed == accepted, and touched == matched by the LFMM.
//
// The conflict check is the lexicographically-first maximal matching of the
// proposal graph (vertices: the two agents of an exchange; priority: the
// record slot), computed by parallel rounds as in commit.cu.
//
// Shared memory: an LFMM key per agent (4 B), the rejected-job bitmap
// (1 bit per job), and 9 B per proposal: slot (4 B), a and d (2 B each:
// the vertex keys alone cap this path at n < 56k) and the state byte.
#pragma once
#include <climits>

#include "state.h"

namespace lsapgpu {
namespace single {

constexpr uint32_t kMatched = 0xFFFFFFFFu;
constexpr uint32_t kQueued = 0xFFFFFFFEu;  // unmatched vertex queued as conflicted (after the rounds)
constexpr uint32_t kKeyShift = 18;         // priorities (slots) < 2^18
constexpr uint32_t kRoundLimit = (1u << 13) - 2;
constexpr int kNT = 1024;

__device__ __forceinline__ uint32_t make_key(uint32_t round, int32_t slot) {
  return (round << kKeyShift) | (0x3FFFFu - static_cast<uint32_t>(slot));
}

struct Scratch {
  int nlog, nconf;
};

// Shared-memory layout: keys[n] | jbits[n/32] | slot[cap] | a[cap] (u16) | d[cap] (u16) | st[cap]
__host__ __device__ inline size_t keys_bytes(int32_t n) { return (static_cast<size_t>(n) * 4 + 15) / 16 * 16; }
__host__ __device__ inline size_t jbits_bytes(int32_t n) { return (static_cast<size_t>(n + 31) / 32 * 4 + 15) / 16 * 16; }
__host__ __device__ inline int edge_capacity(int32_t n, size_t smem) {
  const size_t fixed = keys_bytes(n) + jbits_bytes(n) + 64;
  if (n >= 65536) return 0;
  return smem > fixed ? static_cast<int>((smem - fixed) / 9 / 16 * 16) : 0;
}

// Conflict check + classification of one batch by the calling CTA (P0, the
// control decisions, is the caller's).  Writes the committed and queued
// proposal indices, the rejected-job bitmap and the batch counters for
// commit_apply_kernel; under kCommitCheckOnly writes the step API's
// per-proposal state instead.
//
// Loading the proposals: with `preloaded` the cluster has already written
// slot / a / d / state of every proposal into this CTA's shared memory
// (load_share below), otherwise the CTA loads them itself.
__device__ __forceinline__ void commit_single(const DevState& st, int mode, int edge_cap, unsigned char* smem,
                                              bool preloaded = false, bool early_exit = true) {
  const int tid = threadIdx.x;
  __shared__ Scratch sc;

  Ctrl* C = st.ctrl;
  const int32_t n = st.n;
  const int P = C->parity;
  const int32_t ec0 = C->edge_count[0], ec1 = C->edge_count[1];  // (independent loads)
  const int32_t m = P ? ec1 : ec0;
  const Prop* edges = st.edges[P];
  const int32_t iter = C->iter + 1;

  uint32_t* keys = reinterpret_cast<uint32_t*>(smem);
  uint32_t* jbits = reinterpret_cast<uint32_t*>(smem + keys_bytes(n));
  int32_t* Eslot = reinterpret_cast<int32_t*>(smem + keys_bytes(n) + jbits_bytes(n));
  uint16_t* Ea = reinterpret_cast<uint16_t*>(Eslot + edge_cap);
  uint16_t* Ed = Ea + edge_cap;
  uint8_t* Est = reinterpret_cast<uint8_t*>(Ed + edge_cap);

  if (tid == 0) sc.nlog = sc.nconf = 0;
  for (int32_t x = tid; x < n; x += kNT) keys[x] = 0u;
  for (int32_t x = tid; x < (n + 31) / 32; x += kNT) jbits[x] = 0u;
  if (!preloaded)
    for (int32_t l = tid; l < m; l += kNT) {
      const int4 h = *reinterpret_cast<const int4*>(&edges[l]);  // slot, a, d, j_new
      Eslot[l] = h.x;
      Ea[l] = static_cast<uint16_t>(h.y);
      Ed[l] = static_cast<uint16_t>(h.z);
      Est[l] = kEdgeUndecided;
    }
  __syncthreads();
  if (tid == 0) tl_mark(C, st.tl, st.tl_cap, 5);

  // ---- LFMM rounds ----
  uint32_t R = 1;
  int rounds = 0;
  for (;;) {
    if (R >= kRoundLimit) {
      for (int32_t x = tid; x < n; x += kNT)
        if (keys[x] != kMatched) keys[x] = 0u;
      R = 1;
      __syncthreads();
    }
    int local = 0;
    for (int32_t l = tid; l < m; l += kNT) {
      if (Est[l] != kEdgeUndecided) continue;
      const int32_t u = Ea[l], v = Ed[l];
      const uint32_t cu = keys[u], cv = keys[v];
      if (cu == kMatched || cv == kMatched) {
        Est[l] = kEdgeRejected;
      } else {
        const uint32_t k = make_key(R, Eslot[l]);  // keys only grow within a round
        if (cu < k) atomicMax(&keys[u], k);
        if (cv < k) atomicMax(&keys[v], k);
        local = 1;
      }
    }
    if (__syncthreads_or(local) == 0) break;
    int live = 0;
    for (int32_t l = tid; l < m; l += kNT) {
      if (Est[l] != kEdgeUndecided) continue;
      const int32_t u = Ea[l], v = Ed[l];
      const uint32_t k = make_key(R, Eslot[l]);
      const uint32_t ku = keys[u], kv = keys[v];
      if (ku == k && kv == k) {
        Est[l] = kEdgeAccepted;
        keys[u] = kMatched;
        keys[v] = kMatched;
      } else if (ku != kMatched && kv != kMatched) {
        live = 1;  // may still be accepted (an endpoint not seen matched yet)
      }
    }
    ++R;
    ++rounds;
    // every edge still undecided has an endpoint seen matched (matching is
    // permanent): the next round would only reject them, so do that here and
    // skip its posting pass and barrier
    const bool done = __syncthreads_or(live || !early_exit) == 0;
    if (tid == 0) tl_mark(C, st.tl, st.tl_cap, 6);
    if (done) {
      for (int32_t l = tid; l < m; l += kNT)
        if (Est[l] == kEdgeUndecided) Est[l] = kEdgeRejected;
      __syncthreads();
      break;
    }
  }

  if (mode == kCommitCheckOnly) {  // step API: per-proposal state, proposer first
    for (int32_t l = tid; l < m; l += kNT) {
      const bool agent_rec = Eslot[l] < n;
      st.estate[l] = Est[l];
      st.eu[l] = agent_rec ? Ea[l] : Ed[l];
      st.ev[l] = agent_rec ? Ed[l] : Ea[l];
    }
    if (tid == 0) C->lfmm_rounds += rounds;
    return;
  }

  // ---- classify: committed (= accepted, see header) and rejected ----
  // (list appends are warp-aggregated: one shared atomic per warp and pass)
  const int lane = tid & 31;
  for (int32_t base = tid - lane; base < m; base += kNT) {
    const int32_t l = base + lane;
    const uint8_t s = l < m ? Est[l] : kEdgeUndecided;
    const bool acc = s == kEdgeAccepted;
    const unsigned am = __ballot_sync(0xffffffffu, acc);
    if (am) {
      int r0 = 0;
      if (lane == 0) r0 = atomicAdd(&sc.nlog, __popc(am));
      r0 = __shfl_sync(0xffffffffu, r0, 0);
      if (acc) st.clist[r0 + __popc(am & ((1u << lane) - 1))] = l;
    }
    if (s == kEdgeRejected && Eslot[l] >= n) {
      const int32_t j = Eslot[l] - n;
      atomicOr(&jbits[j >> 5], 1u << (j & 31));
    }
  }
  __syncthreads();
  // conflicted proposers: untouched (unmatched) owners of rejected records,
  // each queued once (the reference's `conflicted` set, parallel.cpp:312-330)
  for (int32_t base = tid - lane; base < m; base += kNT) {
    const int32_t l = base + lane;
    bool q = false;
    if (l < m && Est[l] == kEdgeRejected) {
      const int32_t p = Eslot[l] < n ? Ea[l] : Ed[l];
      q = keys[p] != kMatched && atomicExch(&keys[p], kQueued) != kQueued;
    }
    const unsigned qm = __ballot_sync(0xffffffffu, q);
    if (qm) {
      int r0 = 0;
      if (lane == 0) r0 = atomicAdd(&sc.nconf, __popc(qm));
      r0 = __shfl_sync(0xffffffffu, r0, 0);
      if (q) st.qlist[r0 + __popc(qm & ((1u << lane) - 1))] = l;
    }
  }
  for (int32_t x = tid; x < (n + 31) / 32; x += kNT) st.jbits[x] = jbits[x];
  __syncthreads();
  if (tid == 0) {
    const int nlog = sc.nlog, nitems = 2 * sc.nlog + sc.nconf;
    C->k2_parity = P;
    C->k2_nlog = nlog;
    C->k2_nconf = sc.nconf;
    C->k2_iter = iter;
    C->k2_log_base = C->log_count;
    C->log_count += nlog;
    C->work_count = nitems;
    C->switches += nlog;
    C->pair_items += nitems;
    C->agent_scans += nitems;
    C->job_scans += 2 * nlog;  // + the queued proposers with a rejected job record (apply kernel)
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

// One cluster CTA's share of the proposal load for a preloaded
// commit_single: proposals [l0, l1) written straight into the shared memory
// of the CTA that runs the conflict check (`dst` = its mapped smem base).
__device__ __forceinline__ void load_share(const DevState& st, int edge_cap, unsigned char* dst, int32_t l0,
                                           int32_t l1) {
  const int32_t n = st.n;
  const Prop* edges = st.edges[st.ctrl->parity];
  int32_t* Eslot = reinterpret_cast<int32_t*>(dst + keys_bytes(n) + jbits_bytes(n));
  uint16_t* Ea = reinterpret_cast<uint16_t*>(Eslot + edge_cap);
  uint16_t* Ed = Ea + edge_cap;
  uint8_t* Est = reinterpret_cast<uint8_t*>(Ed + edge_cap);
  for (int32_t l = l0 + static_cast<int32_t>(threadIdx.x); l < l1; l += kNT) {
    const int4 h = *reinterpret_cast<const int4*>(&edges[l]);  // slot, a, d, j_new
    Eslot[l] = h.x;
    Ea[l] = static_cast<uint16_t>(h.y);
    Ed[l] = static_cast<uint16_t>(h.z);
    Est[l] = kEdgeUndecided;
  }
}

}  // namespace single
}  // namespace lsapgpu
