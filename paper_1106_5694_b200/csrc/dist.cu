// dist.cu -- record exchange for the multi-GPU solve (placement
// (ii), or (i) with A held as row blocks): every rank holds AT (and A or its
// row block), scans only the work items it owns (the agents of its row block),
// packs the records it produced, and
// after the caller's allgather (NCCL over NVLink) every rank merges all ranks'
// records into its tables and rebuilds the proposal list.  The commit kernel
// then runs replicated: its result does not depend on proposal order, so all
// ranks apply identical batches and sigma never needs a broadcast.
//
// Exchange buffer per rank: 16-byte header {count, deadline vote} + count x
// Rec (32 B).  The vote is this rank's %globaltimer deadline test at push
// time; the merge ORs every rank's vote into ctrl->expired, so the ranks agree
// on expiry at the same batch (a rank stopping alone would leave its peers
// waiting on a push that never comes).
// Two transports: the caller's allgather (e.g. NCCL) between pack and merge,
// or the peer-memory push below (pack + allgather in one kernel).
#include "state.h"

namespace lsapgpu {
namespace {

struct Rec {
  int32_t agent, job;        // item (agent i, job tau[i]) at scan time
  int32_t agent_partner, job_partner;
  double agent_delta, job_delta;
};
static_assert(sizeof(Rec) == 32, "exchange record layout");

// This rank's share of the work list (or of the identity list for a full sweep).
// Items are owned by agent ROW BLOCKS: rank r scans agents
// [floor(n r / w), floor(n (r+1) / w)) -- the rows of A it holds under the
// row-block placement.
__device__ __forceinline__ int32_t block_owner(int32_t a, int32_t n, int32_t world) {
  return static_cast<int32_t>((static_cast<int64_t>(a + 1) * world - 1) / n);
}

__global__ void own_items_kernel(DevState st, int full, int32_t rank, int32_t world) {
  const int32_t n = st.n;
  const int32_t count = full ? n : st.ctrl->work_count;
  for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < count; k += gridDim.x * blockDim.x) {
    const uint32_t w = full ? (static_cast<uint32_t>(k) | kItemAgent | kItemJob) : st.items[k];
    const int32_t a = static_cast<int32_t>(w & kItemMask);
    if (block_owner(a, n, world) != rank) continue;
    const int pos = atomicAdd(&st.ctrl->own_count, 1);
    st.items_own[pos] = w;
  }
}

__global__ void reset_own_kernel(Ctrl* c) { c->own_count = 0; }

__device__ __forceinline__ long long deadline_vote(const Ctrl* c) {
  return (c->deadline_gt != 0 && globaltimer() >= c->deadline_gt) ? 1 : 0;
}

__global__ void pack_kernel(DevState st, unsigned char* send) {
  const int32_t count = st.ctrl->own_count;
  Rec* out = reinterpret_cast<Rec*>(send + 16);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    reinterpret_cast<long long*>(send)[0] = count;
    reinterpret_cast<long long*>(send)[1] = deadline_vote(st.ctrl);
  }
  for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < count; k += gridDim.x * blockDim.x) {
    const uint32_t w = st.items_own[k];
    const int32_t i = static_cast<int32_t>(w & kItemMask);
    const int32_t j = st.tau[i];
    Rec r;
    r.agent = (w & kItemAgent) ? i : -1;
    r.job = (w & kItemJob) ? j : -1;
    r.agent_partner = st.agent_partner[i];
    r.agent_delta = st.agent_delta[i];
    r.job_partner = st.job_partner[j];
    r.job_delta = st.job_delta[j];
    // holder of the job is i (the item's agent): carried in agent when the
    // agent record is not part of the item
    if (r.agent < 0) r.agent = -2 - i;
    out[k] = r;
  }
}

// Write every rank's records and append the active ones as proposals (Prop,
// the layout the pair scan emits).
__device__ __forceinline__ void merge_body(const DevState& st, const unsigned char* recv, int32_t world,
                                           size_t bytes_per_rank) {
  const int32_t n = st.n;
  const int P = st.ctrl->parity;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    long long vote = 0;
    for (int32_t r = 0; r < world; ++r)
      vote |= reinterpret_cast<const long long*>(recv + static_cast<size_t>(r) * bytes_per_rank)[1];
    if (vote) st.ctrl->expired = 1;  // acted on by the next commit, on every rank alike
  }
  for (int32_t r = 0; r < world; ++r) {
    const unsigned char* base = recv + static_cast<size_t>(r) * bytes_per_rank;
    const int32_t count = static_cast<int32_t>(*reinterpret_cast<const long long*>(base));
    const Rec* in = reinterpret_cast<const Rec*>(base + 16);
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < count; k += gridDim.x * blockDim.x) {
      const Rec rec = in[k];
      const bool has_agent = rec.agent >= 0;
      const int32_t i = has_agent ? rec.agent : -2 - rec.agent;
      if (has_agent) {
        st.agent_delta[i] = rec.agent_delta;
        st.agent_partner[i] = rec.agent_partner;
        if (rec.agent_partner >= 0) {
          const int pos = atomicAdd(&st.ctrl->edge_count[P], 1);
          st.edges[P][pos] = agent_prop(st.sigma, st.tau, st.AT, st.storage, st.ld, i, rec.agent_partner,
                                        rec.agent_delta);
        }
      }
      if (rec.job >= 0) {
        st.job_delta[rec.job] = rec.job_delta;
        st.job_partner[rec.job] = rec.job_partner;
        if (rec.job_partner >= 0) {
          const int pos = atomicAdd(&st.ctrl->edge_count[P], 1);
          st.edges[P][pos] = job_prop(st.sigma, st.tau, st.AT, st.storage, st.ld, n, rec.job, rec.job_partner,
                                      rec.job_delta);
        }
      }
    }
  }
}

__global__ void merge_kernel(DevState st, const unsigned char* recv, int32_t world, size_t bytes_per_rank) {
  merge_body(st, recv, world, bytes_per_rank);
}

// ---- peer-memory exchange (NVLink / NVSwitch P2P) ------------------------
// The pack step stores this rank's records straight into slot `rank` of every
// replica's receive buffer (remote stores through peer mappings), fences at
// system scope and raises this rank's flag in every replica to the round's
// epoch: pack and allgather are one kernel, no collective call.  Receive
// buffers are double-buffered by epoch parity: a rank can only be one round
// ahead of a peer (it waits for every peer's flag before its next push), so it
// never overwrites the buffer that peer is still merging.
__global__ void push_kernel(DevState st, PeerSet ps) {
  const int32_t count = st.ctrl->own_count;
  const uint64_t epoch = st.ctrl->p2p_epoch + 1;  // advanced by the last CTA below
  const size_t slot = static_cast<size_t>(epoch & 1) * ps.world * ps.bytes_per_rank +
                      static_cast<size_t>(ps.rank) * ps.bytes_per_rank;
  if (blockIdx.x == 0 && threadIdx.x < ps.world) {
    reinterpret_cast<long long*>(ps.recv[threadIdx.x] + slot)[0] = count;
    reinterpret_cast<long long*>(ps.recv[threadIdx.x] + slot)[1] = deadline_vote(st.ctrl);
  }
  for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < count; k += gridDim.x * blockDim.x) {
    const uint32_t w = st.items_own[k];
    const int32_t i = static_cast<int32_t>(w & kItemMask);
    const int32_t j = st.tau[i];
    Rec r;
    r.agent = (w & kItemAgent) ? i : -1;
    r.job = (w & kItemJob) ? j : -1;
    r.agent_partner = st.agent_partner[i];
    r.agent_delta = st.agent_delta[i];
    r.job_partner = st.job_partner[j];
    r.job_delta = st.job_delta[j];
    if (r.agent < 0) r.agent = -2 - i;
    for (int32_t q = 0; q < ps.world; ++q) reinterpret_cast<Rec*>(ps.recv[q] + slot + 16)[k] = r;
  }
  // the last CTA to finish raises the flags and advances the epoch
  __threadfence_system();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(&st.ctrl->push_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x < ps.world) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(ps.flags[threadIdx.x] + ps.rank), "l"(epoch)
                 : "memory");
    __syncwarp((1u << ps.world) - 1u);
    if (threadIdx.x == 0) {
      st.ctrl->push_done = 0;
      st.ctrl->p2p_epoch = epoch;
    }
  }
}

// One warp waits until every rank's records of this epoch have landed (lane r
// polls rank r's flag).  10 s without progress flags an error instead of
// hanging the device.
__global__ void peer_wait_kernel(PeerSet ps, Ctrl* c) {
  const int r = threadIdx.x;
  const uint64_t epoch = c->p2p_epoch;
  if (r < ps.world) {
    const uint64_t* f = ps.flags[ps.rank] + r;
    uint64_t t0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    for (;;) {
      uint64_t v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      if (v >= epoch) break;
      uint64_t t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      if (t - t0 > 10000000000ull) {
        c->error = 2;
        break;
      }
      __nanosleep(200);
    }
  }
  __syncwarp();
}

// merge_kernel on this rank's buffer of the current epoch
__global__ void merge_p2p_kernel(DevState st, PeerSet ps) {
  const unsigned char* recv =
      ps.recv[ps.rank] + static_cast<size_t>(st.ctrl->p2p_epoch & 1) * ps.world * ps.bytes_per_rank;
  merge_body(st, recv, ps.world, ps.bytes_per_rank);
}

}  // namespace

cudaError_t launch_dist_push(const DevState& d, const PeerSet& ps, cudaStream_t st) {
  push_kernel<<<148, 256, 0, st>>>(d, ps);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  peer_wait_kernel<<<1, 32, 0, st>>>(ps, d.ctrl);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  merge_p2p_kernel<<<148, 256, 0, st>>>(d, ps);
  return cudaGetLastError();
}

size_t dist_exchange_bytes(int32_t n, int32_t world) {
  const size_t per = (static_cast<size_t>(n) + world - 1) / world;
  return ((16 + per * sizeof(Rec)) + 255) / 256 * 256;
}

cudaError_t launch_dist_own_items(const DevState& d, int full, int32_t rank, int32_t world, cudaStream_t st) {
  reset_own_kernel<<<1, 1, 0, st>>>(d.ctrl);
  own_items_kernel<<<148, 256, 0, st>>>(d, full, rank, world);
  return cudaGetLastError();
}

cudaError_t launch_dist_pack(const DevState& d, void* send, cudaStream_t st) {
  pack_kernel<<<148, 256, 0, st>>>(d, static_cast<unsigned char*>(send));
  return cudaGetLastError();
}

cudaError_t launch_dist_merge(const DevState& d, const void* recv, int32_t world, size_t bytes_per_rank,
                              cudaStream_t st) {
  merge_kernel<<<148, 256, 0, st>>>(d, static_cast<const unsigned char*>(recv), world, bytes_per_rank);
  return cudaGetLastError();
}

}  // namespace lsapgpu
