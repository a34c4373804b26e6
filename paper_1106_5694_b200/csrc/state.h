// state.h -- device-resident solver state shared by the host orchestration
// (lsapgpu.cu) and the kernels (layout.cu, scan.cu, commit.cu).
//
// It is the B200 layout of the reference's detail::SolverState
// (proj/src/solver_state.hpp:33-149): the same vectors (sigma, tau, the
// per-agent current benefit, SoA delta tables), plus the work list, the
// ping-pong active-edge lists that replace argmax + check_conflicts' linear
// walks, and the delta log that replaces the in-loop value/trace update.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace lsapgpu {

struct DevState {
  int32_t n = 0;
  int64_t ld = 0;  // row pitch in elements (multiple of 64)
  int storage = kF64;
  const void* A = nullptr;   // row-major, n x ld
  const void* AT = nullptr;  // transposed, n x ld
  // row-block placement (multi-GPU): this rank holds rows
  // [a_row0, a_row0 + a_rows) of A (and of Q) -- the agents it scans -- and
  // all of AT; every other A[i][j] is read as AT[j][i].  Single GPU: 0, n.
  int32_t a_row0 = 0;
  int32_t a_rows = 0;
  int32_t* sigma = nullptr;  // job -> agent (padded to ld)
  int32_t* tau = nullptr;    // agent -> job (padded to ld)
  uint16_t* tau16 = nullptr; // the same as uint16 when n < 65536 (the resident scan bulk-loads it)
  void* acur = nullptr;      // A[i][tau[i]] (storage type, padded to ld)
  // quantized filter copies for the long-row scan (scan_filter.cuh), pitch ld:
  // Q = ceil(A * qscale), QT = ceil(AT * qscale) as int16 or int8, and the
  // per-launch position array aux[p] = tau[p] | (floor(acur[p] * qscale) + 2^14) << 17
  const void* Q = nullptr;
  const void* QT = nullptr;
  uint32_t* aux = nullptr;
  double qscale = 0.0;
  int filter_check = 0;  // > 0: the filter scan re-verifies every k-th item unfiltered (diagnostics)

  double* agent_delta = nullptr;
  int32_t* agent_partner = nullptr;
  double* job_delta = nullptr;
  int32_t* job_partner = nullptr;

  // active proposals (Prop, common.cuh), capacity 2n each, ping-pong
  Prop* edges[2] = {nullptr, nullptr};
  // split commit: committed / queued-conflicted proposal indices and the
  // rejected-job bitmap of the batch (commit_single.cuh -> commit_apply)
  int32_t* clist = nullptr;
  int32_t* qlist = nullptr;
  uint32_t* jbits = nullptr;
  int32_t* eu = nullptr;                   // LFMM scratch: endpoint u, capacity 2n
  int32_t* ev = nullptr;                   // endpoint v
  int32_t* eprop = nullptr;                // proposer agent (frozen sigma)
  uint8_t* estate = nullptr;               // edge state
  int32_t* c_jnew = nullptr;               // committed exchange: new job
  double* c_delta = nullptr;               // committed exchange: recomputed delta
  double* c_acur = nullptr;                // committed exchange: new acur of agent / displaced (2 x 2n)
  int32_t* c_rank = nullptr;               // per-proposal append rank (cluster commit, global fallback)
  uint32_t* vstate = nullptr;              // per-vertex flags (cluster commit, global fallback)
  uint32_t* keys = nullptr;                // vertex keys when they do not fit in smem
  int32_t* touched_stamp = nullptr;        // agent touched in iteration k
  int32_t* conf_stamp = nullptr;           // agent queued as conflicted in iteration k
  int32_t* rej_stamp = nullptr;            // record slot rejected in iteration k (2n)
  uint32_t* items = nullptr;               // work list (capacity n)
  LogEntry* log = nullptr;                 // committed exchanges, in commit order
  LogEntry* log_sorted = nullptr;          // ... ordered by (iter, slot) on the device (log_order.cu)
  int64_t log_cap = 0;

  // split-item partial results (segmented scans)
  double* part_ad = nullptr;
  int32_t* part_at = nullptr;
  double* part_jd = nullptr;
  int32_t* part_ji = nullptr;
  int32_t* part_arrive = nullptr;  // per item-group arrival counters (zeroed)
  int64_t part_cap = 0;            // capacity in (item, segment) slots

  Ctrl* ctrl = nullptr;
  double eps = 0.0;
  int policy = 0;  // 0 touched_and_conflicted, 1 touched_only

  // multi-GPU (dist.cu): this rank's share of the work list, and whether the
  // scan appends proposals itself (single GPU) or the record merge does
  uint32_t* items_own = nullptr;
  int use_own = 0;
  int emit_edges = 1;
  // multi-rank solve: the anytime deadline is decided at each record exchange
  // (every rank's vote travels in its exchange header and the merge ORs them,
  // dist.cu), never by one rank's commit, so all ranks stop at the same batch
  int dist_vote = 0;
  int pdl = 0;  // launch the inner-loop kernels with programmatic dependent launch
  // device timeline (instrumentation): CTA 0 of every scan / commit launch
  // appends (%globaltimer << 4 | kind); null when disabled
  unsigned long long* tl = nullptr;
  int tl_cap = 0;
};

// ---- launchers (implemented in the .cu files) -------------------------------

// layout.cu
struct LayoutSource {
  int kind = 0;  // 0 memory, 1 uniform int, 2 unit f32, 3 unit scaled, 4 p2p, 5 geom
  const void* src = nullptr;  // memory source (row-major n x n)
  int src_dtype = 0;          // 0 f64, 1 f32, 2 i32, 3 i16
  uint64_t seed = 0;
  double param = 0.0;
  const double* aux = nullptr;  // generator side tables (p2p: up,x,y; geom: xs,ys)
  // row-block placement: write only rows [a_row0, a_row0 + a_rows) of A (and
  // Q), at local row index i - a_row0; AT (and QT) whole.  a_rows < 0: all rows.
  int32_t a_row0 = 0;
  int32_t a_rows = -1;
};
// flags bit0: non-finite present, bit1: not int16-exact, bit2: not int32 (<2^29) exact,
// bit3: not fp32-exact.
// amax (nullable): atomicMax of the float bits of every |entry| rounded up
cudaError_t launch_classify(const LayoutSource& s, int32_t n, int64_t row0, int64_t rows,
                            uint32_t* flags, cudaStream_t st, uint32_t* amax = nullptr);
// Quantized filter copies the layout pass writes alongside A / AT (bits 0: none)
struct QuantTarget {
  void* Q = nullptr;
  void* QT = nullptr;
  double scale = 0.0;
  int bits = 0;
};
cudaError_t launch_build_layout(const LayoutSource& s, int32_t n, int64_t row0, int64_t rows,
                                int storage, void* A, void* AT, int64_t ld, cudaStream_t st);
cudaError_t launch_gen_aux(const LayoutSource& s, int32_t n, double* aux, cudaStream_t st);
// classify + build in one pass for a speculated storage type (flags as launch_classify)
// amax (nullable): atomicMax of the float bits of every |entry| rounded up (the filter's scale);
// qt.bits != 0: also write the quantized copies Q / QT
cudaError_t launch_layout_fused(const LayoutSource& s, int32_t n, int64_t row0, int64_t rows, int storage,
                                void* A, void* AT, int64_t ld, uint32_t* flags, cudaStream_t st,
                                uint32_t* amax = nullptr, QuantTarget qt = QuantTarget{});
// max |entry| of the stored matrix as float bits rounded up, into *out
cudaError_t launch_amax(const DevState& d, uint32_t* out, cudaStream_t st);
// Q = ceil(A * scale), QT = ceil(AT * scale) as int16 (qbits 16) or int8 (qbits 8), padding zeroed
cudaError_t launch_quantize(const DevState& d, int qbits, double scale, void* Q, void* QT, cudaStream_t st);
cudaError_t launch_init_assignment(const DevState& d, cudaStream_t st);  // tau, acur from sigma
// out[j] = A[sigma[j]][j] (fp64); pack: also sigma and tau as int32 after it (2n doubles)
cudaError_t launch_gather_current(const DevState& d, double* out, cudaStream_t st, int pack = 0);
cudaError_t launch_read_rows(const DevState& d, const int32_t* rows, int32_t nrows, double* out,
                             cudaStream_t st);

// scan.cu
struct ScanPlan {
  int m = 1;            // items batched per CTA (share tau/acur streams)
  int passes = 1;       // row chunks per item (rows larger than smem)
  int64_t chunk = 0;    // elements per staged chunk
  int bufs = 2;         // smem stage buffers
  int ctas = 0;         // persistent grid size
  int threads = 256;
  size_t smem = 0;      // dynamic smem per CTA
  int max_segments = 1;
  int resident = 0;     // 1: resident-state kernel (scan_resident.cuh)
  int depth = 2;        // streaming kernel: vector steps of the streamed rows in flight
  int l2_prefetch = 0;  // resident kernel: stages whose rows are prefetched into L2 ahead
  int filter = 0;       // 8 / 16: quantized-filter kernel (scan_filter.cuh) with int8 / int16 copies;
                        // m = row buffers, bufs = chunk slots
  int filter_queue = 1024;  // filter kernel: candidates per item before the exact whole-item fallback
  int filter_tmem = 0;      // filter kernel: the launch's aux words resident in TMEM (n <= 65536)
  int launches() const { return filter ? 2 : 1; }  // kernels per scan (the filter adds the aux build)
  bool operator==(const ScanPlan& o) const {
    return m == o.m && passes == o.passes && chunk == o.chunk && bufs == o.bufs && ctas == o.ctas &&
           threads == o.threads && smem == o.smem && max_segments == o.max_segments && resident == o.resident &&
           depth == o.depth && l2_prefetch == o.l2_prefetch && filter == o.filter &&
           filter_queue == o.filter_queue && filter_tmem == o.filter_tmem;
  }
};
ScanPlan plan_scan(const DevState& d, int num_sms);
// full sweep (identity work list, count n) when full != 0, else the device work list
cudaError_t launch_scan(const DevState& d, const ScanPlan& p, int full, cudaStream_t st);

// dist.cu (multi-GPU record exchange)
size_t dist_exchange_bytes(int32_t n, int32_t world);
cudaError_t launch_dist_own_items(const DevState& d, int full, int32_t rank, int32_t world, cudaStream_t st);
cudaError_t launch_dist_pack(const DevState& d, void* send, cudaStream_t st);
cudaError_t launch_dist_merge(const DevState& d, const void* recv, int32_t world, size_t bytes_per_rank,
                              cudaStream_t st);
constexpr int kMaxPeers = 8;
struct PeerSet {  // receive buffers / flag arrays of every rank, mapped in this process
  unsigned char* recv[kMaxPeers];
  uint64_t* flags[kMaxPeers];
  int32_t world, rank;
  size_t bytes_per_rank;
};
// push this rank's records into every replica (epoch = ++ctrl->p2p_epoch, buffer
// epoch & 1), wait for every rank's flag, merge: the whole exchange, graph-capturable
cudaError_t launch_dist_push(const DevState& d, const PeerSet& ps, cudaStream_t st);

// commit.cu
enum CommitMode : int { kCommitSolve = 0, kCommitCheckOnly = 1, kCommitApplyOnly = 2 };
struct CommitPlan {
  int threads = 1024;
  size_t smem = 0;          // single-CTA kernel (apply-only step API)
  bool keys_in_smem = true;
  int cluster = 8;          // cluster kernel: CTAs per cluster (16 or 8)
  size_t cluster_smem = 0;  // cluster kernel: dynamic smem per CTA
  int edge_cap = 0;         // cluster kernel: proposals per CTA held in smem
  int cta_edge_cap = 0;     // single-CTA path taken when the proposals fit one CTA (0: never)
  int variant = 0;          // cluster kernel bit 0: read keys before the round-1 atomics
  int wide_keys = 0;        // slot-only LFMM keys cleared every round (n >= 2^17, or LSAPGPU_LFMM_WIDE=1)
  int launches() const { return 2; }  // kernels per solve-mode commit: conflict check + commit_apply_kernel
  bool operator==(const CommitPlan& o) const {
    return threads == o.threads && smem == o.smem && keys_in_smem == o.keys_in_smem && cluster == o.cluster &&
           cluster_smem == o.cluster_smem && edge_cap == o.edge_cap && cta_edge_cap == o.cta_edge_cap &&
           variant == o.variant && wide_keys == o.wide_keys;
  }
};
CommitPlan plan_commit(const DevState& d);
cudaError_t launch_commit(const DevState& d, const CommitPlan& p, int mode,
                          cudaGraphConditionalHandle cond, int use_cond, cudaStream_t st);
int commit_cluster_size(const DevState& d, size_t smem);
cudaError_t launch_commit_cluster(const DevState& d, const CommitPlan& p, int mode,
                                  cudaGraphConditionalHandle cond, int use_cond, cudaStream_t st);
// step-API helpers
cudaError_t launch_edges_from_tables(const DevState& d, cudaStream_t st);
cudaError_t launch_tau16_sync(const DevState& d, cudaStream_t st);
// Order the delta log by (iter, slot) into log_sorted (the reference's batch
// order, parallel.cpp:306-310); status in Ctrl::order_bad / order_total.
// False from order_log_fits when the slot bitmap does not fit shared memory.
bool order_log_fits(int32_t n);
cudaError_t launch_order_log(const DevState& d, cudaStream_t st);
cudaError_t launch_accepted_from_masks(const DevState& d, const uint8_t* agent_acc,
                                       const uint8_t* job_acc, cudaStream_t st);

// auction.cu (lsap::auction_solve, auction.cpp)
struct AuctionCtrl {
  int32_t count[2];  // bidder lists (ping-pong)
  int32_t expired;   // deadline fired (decided by CTA 0 at round boundaries)
  int32_t finished;  // every phase converged
  int32_t greedy;    // completed greedily after a deadline
  int32_t pad_;
  int64_t rounds;    // SolveReport::outer_iterations
  int64_t switches;  // awards, including displacements
  int64_t bids;      // agent row scans
  int64_t phases;    // epsilon phases started
  unsigned long long lo_key, hi_key;  // benefit range (order-preserving keys)
};
struct AuctionDev {
  double* prices = nullptr;
  int32_t* owner = nullptr;     // job -> agent (-1 free)
  int32_t* assigned = nullptr;  // agent -> job (-1 unassigned)
  unsigned long long* slot = nullptr;  // per job: {inverted agent, bid key} of the round's best bid
  int32_t* rec_i = nullptr;     // bid records beyond a CTA's shared-memory capacity (CS x n)
  int32_t* rec_j = nullptr;
  double* rec_bid = nullptr;
  int32_t* wl[2] = {nullptr, nullptr};  // bidder lists, one n-entry segment per cluster CTA
  int local_prices = 0;         // 1: every CTA holds a shared-memory replica of the prices
  int row_prefetch = 0;         // 1: L2-prefetch the rows of the next round's bidders
  AuctionCtrl* ctrl = nullptr;
  const double* eps_list = nullptr;  // epsilon of every phase (host-computed schedule)
  int32_t n_eps = 0;
  double* round_prices = nullptr;    // optional on_round snapshots, round_cap x n
  int64_t round_cap = 0;
};
int auction_cluster_size();
int32_t auction_local_price_cap();
cudaError_t launch_auction(const DevState& d, const AuctionDev& a, int64_t remaining_ns, cudaStream_t st);
cudaError_t launch_minmax(const DevState& d, AuctionCtrl* c, cudaStream_t st);
double auction_key_value(unsigned long long key);

// greedy.cu (greedy initial assignment; extension, see the file header)
struct GreedyCtrl {
  int32_t count[2];
  int64_t rounds;
};
struct GreedyDev {
  int32_t* list[2] = {nullptr, nullptr};  // unassigned agents (ping-pong)
  uint32_t* free = nullptr;               // free-job bitmap
  int32_t* claim = nullptr;               // per agent: the job it claims this round
  unsigned long long* slot = nullptr;     // per job: {inverted agent, benefit key} of the best claim
  GreedyCtrl* ctrl = nullptr;
};
// sigma (device) = the greedy assignment of the matrix in d
cudaError_t launch_greedy(const DevState& d, const GreedyDev& g, int num_sms, cudaStream_t st);

}  // namespace lsapgpu
