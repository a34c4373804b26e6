// lsapgpu.cu -- host orchestration behind the C-ABI (include/lsapgpu.h).
//
// The outer loop of lsap::dgs_parallel (proj/src/parallel.cpp:255-346) runs on
// the host, once per full pass: a full pair-scan sweep, then the whole inner
// batch loop as ONE launch of a CUDA graph whose conditional WHILE node
// repeats {commit kernel, pair-scan kernel} until the commit kernel finds no
// active record (the argmax continue test, parallel.cpp:265-267) and clears
// the graph condition on the device.  The host syncs once per outer pass to
// drain the delta log, which it replays in the reference's batch order to
// reproduce SolveReport::objective_trace and the exact `value == f_start`
// termination test (parallel.cpp:306-310, 343-345).
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <type_traits>
#include <thread>
#include <vector>

#include "../../include/lsapgpu.h"
#include "state.h"

using namespace lsapgpu;

namespace lsapgpu {
// Exact host narrowing (host_narrow.cpp, AVX2): false if any value is not
// representable under the storage rule (or is not finite).
bool narrow_to_i16(const double* src, int16_t* dst, size_t cnt);
bool narrow_to_i32(const double* src, int32_t* dst, size_t cnt);
bool narrow_to_f32(const double* src, float* dst, size_t cnt);
}  // namespace lsapgpu

namespace {

constexpr int64_t kTraceCap = 100000;  // parallel.cpp:15

size_t esize(int storage) {
  switch (storage) {
    case kI16: return 2;
    case kI32: return 4;
    case kF32: return 4;
    default: return 8;
  }
}
size_t src_size(int dtype) {
  switch (dtype) {
    case LSAPGPU_F64: return 8;
    case LSAPGPU_F32: return 4;
    case LSAPGPU_I32: return 4;
    default: return 2;
  }
}

__global__ void set_deadline_kernel(Ctrl* c, int64_t remaining_ns) {
  c->expired = 0;
  c->error = 0;
  c->deadline_gt = remaining_ns < 0 ? 0ull : globaltimer() + static_cast<uint64_t>(remaining_ns);
}

// Start of an outer pass (or of a resumed inner loop after a log drain).
__global__ void begin_pass_kernel(Ctrl* c, int full) {
  if (full) {
    c->edge_count[0] = 0;
    c->edge_count[1] = 0;
  }
  c->inner_done = 0;
  c->drain = 0;
  c->log_count = 0;
}

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};

constexpr size_t kUploadChunk = 64ull << 20;  // rows per H2D chunk: ~64 MB of source
constexpr size_t kNarrowChunk = 32ull << 20;  // ... for the host-narrowed upload (no per-chunk barrier)
constexpr int kRing = 4;                       // pinned bounce buffers (pageable fp64 sources)
constexpr int kRingNarrow = 8;                 // ... of the host-narrowed upload (absorbs thread skew)
constexpr int kRingMax = 8;
constexpr size_t kStageKeep = 16ull << 30;     // keep the device staging copy up to this size

int upload_threads() {
  if (const char* e = std::getenv("LSAPGPU_UPLOAD_THREADS")) return std::max(1, std::atoi(e));
  const unsigned hw = std::thread::hardware_concurrency();
  return static_cast<int>(std::max(2u, std::min(16u, hw ? hw : 2u)));
}

// Fixed pool of host threads for the pageable -> pinned copies: run(fn) calls
// fn(t) for t = 0..size()-1, t = 0 on the calling thread, and returns when all
// are done.
class HostPool {
 public:
  explicit HostPool(int n) : n_(n) {
    for (int t = 1; t < n_; ++t) th_.emplace_back([this, t] { loop(t); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return n_; }
  void run(const std::function<void(int)>& fn) {
    {
      std::lock_guard<std::mutex> g(m_);
      fn_ = &fn;
      pending_ = n_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> l(m_);
    done_cv_.wait(l, [this] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void loop(int t) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* f = nullptr;
      {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        f = fn_;
      }
      (*f)(t);
      std::lock_guard<std::mutex> g(m_);
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

}  // namespace

struct lsapgpu_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  std::string err;

  DevState d;
  int32_t n_vec = 0;      // vectors allocated for this n
  int32_t n_matrix = 0;   // matrix present for this n (0 = none)
  std::vector<Buf> vec_bufs;
  Buf mat;                // A and AT (one allocation)
  Buf qmat;               // Q and QT: quantized filter copies (scan_filter.cuh), when the plan uses them
  int32_t place_rank = 0, place_world = 1;  // row-block placement of A (lsapgpu_set_placement)
  int quant_bits = 0;     // copies the last layout pass wrote (0: none) and their scale
  // storage of the last device-source matrix (and its n): a repeated upload
  // of the same shape speculates it without the probe's round trip
  int last_dev_storage = -1;
  int32_t last_dev_n = 0;
  double quant_scale = 0.0;
  bool quant_fused = false;  // the current copies came from the layout pass (no quantize pass)
  std::set<const void*> peer_poisoned;  // peer-transport flag arrays whose epochs a failed solve desynchronised
  Ctrl* ctrl_dev = nullptr;
  Ctrl* ctrl_host = nullptr;  // pinned mirror
  uint32_t* flags_dev = nullptr;

  ScanPlan scan_plan;
  CommitPlan commit_plan;

  // cached inner-loop graph
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  // everything the captured kernels took by value: a new matrix in the same
  // buffers with the same plans (every bench step) reuses the graph
  DevState graph_state;
  ScanPlan graph_scan;
  CommitPlan graph_commit;

  // scan timing (host-stepped mode)
  bool timing = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double scan_ms = 0.0, full_ms = 0.0, commit_ms = 0.0;
  int64_t scan_launches = 0, full_launches = 0, commit_launches = 0;

  // cumulative transfer / launch counters (bench.py's e2e and gpu_launches)
  int64_t h2d = 0, d2h = 0, launches = 0;

  // pinned host mirrors for the solve's device->host reads (one sync each)
  double* obj_pin = nullptr;     // per-job entries of the ordered objective
  int32_t obj_cap = 0;
  LogEntry* log_pin = nullptr;   // delta-log prefix drained with the control block
  std::vector<LogEntry> log_host, log_sorted;  // replay buffers, kept so their pages stay mapped
  int64_t host_log_orders = 0;                 // passes whose log the host had to order (device premise failed)
  static constexpr int64_t kLogPin = 1 << 16;
  int64_t log_hint[4] = {kLogPin, kLogPin, kLogPin, kLogPin};  // log entries per outer pass, last solve

  // host upload pipeline (lsapgpu_set_matrix)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_ready = nullptr;
  cudaEvent_t ev_chunk[kRingMax] = {};
  Buf stage;                      // device copy of the source matrix
  uint32_t* chunk_flags = nullptr;
  int chunk_flags_cap = 0;
  void* ring[kRingMax] = {};      // pinned bounce buffers
  size_t ring_size[kRingMax] = {};
  HostPool* pool = nullptr;

  // auction baseline (auction.cu): per-n vectors (in vec_bufs), the epsilon
  // schedule and the benefit range of the current matrix
  // cached random_perm(n, seed) and the counter base of a solve (pinned)
  int32_t* perm_pin = nullptr;
  int32_t perm_cap = 0, perm_n = -1;
  uint64_t perm_seed = 0;
  Ctrl* ctrl_base = nullptr;

  // multi-GPU inner-loop graph of the peer transport (commit, apply, own
  // items, scan, push / wait / merge), cached like the single-GPU one
  // device-driven outer loop graph (integer storage, single GPU)
  cudaGraphExec_t dist_exec = nullptr;
  cudaGraph_t dist_graph = nullptr;
  DevState dist_state;
  PeerSet dist_ps;

  GreedyDev gr;                    // greedy assignment scratch (per n, in vec_bufs)
  int32_t gr_n = 0;

  AuctionDev au;
  int32_t au_n = 0;
  AuctionCtrl* au_host = nullptr;  // pinned
  double* eps_dev = nullptr;
  size_t eps_cap = 0;
  bool range_ok = false;
  double lo = 0.0, hi = 0.0;
};

namespace {

int fail(lsapgpu_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

cudaError_t cpy(lsapgpu_ctx* ctx, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
                cudaStream_t st) {
  if (kind == cudaMemcpyHostToDevice) ctx->h2d += static_cast<int64_t>(bytes);
  if (kind == cudaMemcpyDeviceToHost) ctx->d2h += static_cast<int64_t>(bytes);
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st);  // UVA: any host/device pointer
}

#define CK(expr)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(ctx, LSAPGPU_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

void drop_graph(lsapgpu_ctx* ctx) {
  if (ctx->exec) cudaGraphExecDestroy(ctx->exec);
  if (ctx->graph) cudaGraphDestroy(ctx->graph);
  ctx->exec = nullptr;
  ctx->graph = nullptr;
}

void free_vectors(lsapgpu_ctx* ctx) {
  for (auto& b : ctx->vec_bufs) cudaFree(b.p);
  ctx->vec_bufs.clear();
  ctx->n_vec = 0;
  ctx->au_n = 0;
  ctx->gr_n = 0;
}

template <class T>
cudaError_t valloc(lsapgpu_ctx* ctx, T** p, size_t count, bool zero) {
  void* q = nullptr;
  const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
  cudaError_t e = cudaMalloc(&q, bytes);
  if (e != cudaSuccess) return e;
  if (zero) {
    e = cudaMemsetAsync(q, 0, bytes, ctx->stream);
    if (e != cudaSuccess) return e;
  }
  ctx->vec_bufs.push_back({q, bytes});
  *p = static_cast<T*>(q);
  return cudaSuccess;
}

int64_t pitch_of(int32_t n) { return (static_cast<int64_t>(n) + 63) / 64 * 64; }

// Per-n vectors (everything except the matrix).
int ensure_vectors(lsapgpu_ctx* ctx, int32_t n) {
  if (ctx->n_vec == n) return LSAPGPU_OK;
  drop_graph(ctx);
  free_vectors(ctx);
  DevState& d = ctx->d;
  const int64_t ld = pitch_of(n);
  const size_t N = static_cast<size_t>(ld), N2 = 2 * N;
  d.n = n;
  d.ld = ld;
  CK(valloc(ctx, &d.sigma, N, true));
  CK(valloc(ctx, &d.tau, N, true));
  d.tau16 = nullptr;
  if (n < 65536) CK(valloc(ctx, &d.tau16, N, true));
  void* acur = nullptr;
  CK(valloc(ctx, reinterpret_cast<double**>(&acur), N, true));  // 8 bytes/elem covers any storage
  d.acur = acur;
  CK(valloc(ctx, &d.agent_delta, N, true));
  CK(valloc(ctx, &d.agent_partner, N, true));
  CK(valloc(ctx, &d.job_delta, N, true));
  CK(valloc(ctx, &d.job_partner, N, true));
  CK(valloc(ctx, &d.edges[0], N2, false));  // Prop proposal entries
  CK(valloc(ctx, &d.edges[1], N2, false));
  CK(valloc(ctx, &d.clist, N, false));
  CK(valloc(ctx, &d.qlist, N2, false));
  CK(valloc(ctx, &d.jbits, N / 32 + 1, true));
  CK(valloc(ctx, &d.eu, N2, false));
  CK(valloc(ctx, &d.ev, N2, false));
  CK(valloc(ctx, &d.eprop, N2, false));
  CK(valloc(ctx, &d.estate, N2, false));
  CK(valloc(ctx, &d.c_jnew, N2, false));
  CK(valloc(ctx, &d.c_delta, N2, false));
  CK(valloc(ctx, &d.c_acur, 2 * N2, false));
  CK(valloc(ctx, &d.c_rank, N2, false));
  CK(valloc(ctx, &d.vstate, N, true));
  CK(valloc(ctx, &d.keys, N, true));
  CK(valloc(ctx, &d.touched_stamp, N, true));
  CK(valloc(ctx, &d.conf_stamp, N, true));
  CK(valloc(ctx, &d.rej_stamp, N2, true));
  CK(valloc(ctx, &d.items, N, false));
  CK(valloc(ctx, &d.items_own, N, false));
  CK(valloc(ctx, &d.aux, N, true));
  d.log_cap = std::max<int64_t>(1 << 20, 8 * static_cast<int64_t>(n));
  // (tests: LSAPGPU_LOG_CAP shrinks the delta log so a pass drains it; a batch
  // appends at most 2n entries, so the cap never goes below that)
  if (const char* e = std::getenv("LSAPGPU_LOG_CAP"))
    d.log_cap = std::max<int64_t>(std::atoll(e), 2 * static_cast<int64_t>(n) + 64);
  CK(valloc(ctx, &d.log, static_cast<size_t>(d.log_cap), false));
  CK(valloc(ctx, &d.log_sorted, static_cast<size_t>(d.log_cap), false));
  d.part_cap = (static_cast<int64_t>(n) + 8) * 16;
  CK(valloc(ctx, &d.part_ad, static_cast<size_t>(d.part_cap), false));
  CK(valloc(ctx, &d.part_at, static_cast<size_t>(d.part_cap), false));
  CK(valloc(ctx, &d.part_jd, static_cast<size_t>(d.part_cap), false));
  CK(valloc(ctx, &d.part_ji, static_cast<size_t>(d.part_cap), false));
  CK(valloc(ctx, &d.part_arrive, N + 8, true));
  d.ctrl = ctx->ctrl_dev;
  ctx->n_vec = n;
  // Key epochs and iteration stamps restart with fresh (zeroed) vectors.
  std::memset(ctx->ctrl_host, 0, sizeof(Ctrl));
  ctx->ctrl_host->round = 1;
  CK(cpy(ctx, ctx->ctrl_dev, ctx->ctrl_host, sizeof(Ctrl), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return LSAPGPU_OK;
}

int pull_ctrl(lsapgpu_ctx* ctx) {
  CK(cpy(ctx, ctx->ctrl_host, ctx->ctrl_dev, sizeof(Ctrl), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return LSAPGPU_OK;
}
int push_ctrl(lsapgpu_ctx* ctx) {
  CK(cpy(ctx, ctx->ctrl_dev, ctx->ctrl_host, sizeof(Ctrl), cudaMemcpyHostToDevice, ctx->stream));
  return LSAPGPU_OK;
}

int storage_of_flags(uint32_t flags) {
  if (!(flags & 2u)) return kI16;
  if (!(flags & 4u)) return kI32;
  if (!(flags & 8u)) return kF32;
  return kF64;
}

// (Re)points A/AT at an allocation large enough for n x ld elements of `storage`.
// Rows of A this context holds: all, or under the row-block placement
// (lsapgpu_set_placement) the block of rank `rank` of `world`.
void placement_rows(const lsapgpu_ctx* ctx, int32_t n, int32_t* row0, int32_t* rows) {
  const int64_t r = ctx->place_rank, w = ctx->place_world;
  *row0 = static_cast<int32_t>(n * r / w);
  *rows = static_cast<int32_t>(n * (r + 1) / w) - *row0;
}

int alloc_matrix(lsapgpu_ctx* ctx, int32_t n, int storage) {
  const int64_t ld = pitch_of(n);
  int32_t row0 = 0, rows = n;
  placement_rows(ctx, n, &row0, &rows);
  const size_t at_bytes = static_cast<size_t>(n) * static_cast<size_t>(ld) * esize(storage);
  const size_t a_bytes = (static_cast<size_t>(rows) * static_cast<size_t>(ld) * esize(storage) + 255) / 256 * 256;
  if (ctx->mat.bytes < a_bytes + at_bytes) {
    if (ctx->mat.p) cudaFree(ctx->mat.p);
    ctx->mat.p = nullptr;
    ctx->mat.bytes = 0;
    CK(cudaMalloc(&ctx->mat.p, a_bytes + at_bytes));
    ctx->mat.bytes = a_bytes + at_bytes;
  }
  DevState& d = ctx->d;
  d.storage = storage;
  d.A = ctx->mat.p;
  d.AT = static_cast<unsigned char*>(ctx->mat.p) + a_bytes;
  d.a_row0 = row0;
  d.a_rows = rows;
  return LSAPGPU_OK;
}

// Single-GPU entry points need every row of A: refuse a row-block context.
int require_full_rows(lsapgpu_ctx* ctx, const char* what) {
  if (ctx->place_world <= 1) return LSAPGPU_OK;
  return fail(ctx, LSAPGPU_ERR_STATE,
              std::string(what) + ": this context holds a row block of the matrix (lsapgpu_set_placement); "
                                  "only the multi-GPU solve of its rank can use it");
}

// the layout source's share of A for this context (all rows: -1)
void set_source_rows(const lsapgpu_ctx* ctx, LayoutSource* src) {
  src->a_row0 = ctx->d.a_row0;
  src->a_rows = ctx->d.a_rows == ctx->d.n ? -1 : ctx->d.a_rows;
}

// Quantized filter copies for the long-row scan (scan_filter.cuh): a
// power-of-two scale with max|a| * scale <= 16383 (int16) or 127 (int8), from
// the max the layout pass reduced into flags_dev[2], then Q / QT.
double quant_scale_for(float amax, int bits) {
  const double limit = bits == 16 ? 16383.0 : 127.0;
  double scale = 1.0;
  if (amax > 0.f) {
    int e = 0;
    std::frexp(limit / static_cast<double>(amax), &e);  // limit / amax in [2^(e-1), 2^e)
    scale = std::ldexp(1.0, std::max(-1000, std::min(1000, e - 1)));
    while (static_cast<double>(amax) * scale > limit) scale *= 0.5;
  }
  return scale;
}

int alloc_quant(lsapgpu_ctx* ctx, int bits, void** Q, void** QT) {
  const DevState& d = ctx->d;
  const size_t qt_bytes = static_cast<size_t>(d.n) * static_cast<size_t>(d.ld) * static_cast<size_t>(bits / 8);
  const size_t q_bytes =  // Q: this context's row block of A
      (static_cast<size_t>(d.a_rows) * static_cast<size_t>(d.ld) * static_cast<size_t>(bits / 8) + 255) / 256 * 256;
  if (ctx->qmat.bytes < q_bytes + qt_bytes) {
    if (ctx->qmat.p) cudaFree(ctx->qmat.p);
    ctx->qmat.p = nullptr;
    ctx->qmat.bytes = 0;
    CK(cudaMalloc(&ctx->qmat.p, q_bytes + qt_bytes));
    ctx->qmat.bytes = q_bytes + qt_bytes;
  }
  *Q = ctx->qmat.p;
  *QT = static_cast<unsigned char*>(ctx->qmat.p) + q_bytes;
  return LSAPGPU_OK;
}

float bits_to_float(uint32_t b) {
  float f = 0.f;
  std::memcpy(&f, &b, sizeof(f));
  return f;
}

// Before a layout pass: if the scan plan for this matrix uses
// the filter copies, size them and pick the scale from the probe rows' max
// |a| so the layout pass writes Q / QT itself (no separate quantize pass);
// finish_matrix checks the scale against the whole matrix's max afterwards.
int prepare_quant(lsapgpu_ctx* ctx, int storage, float probe_amax, QuantTarget* qt) {
  *qt = QuantTarget{};
  ctx->quant_bits = 0;
  DevState tmp = ctx->d;
  tmp.storage = storage;
  const ScanPlan p = plan_scan(tmp, ctx->num_sms);
  if (!p.filter) return LSAPGPU_OK;
  const int rc = alloc_quant(ctx, p.filter, &qt->Q, &qt->QT);
  if (rc) return rc;
  qt->scale = quant_scale_for(probe_amax, p.filter);
  qt->bits = p.filter;
  ctx->quant_bits = p.filter;
  ctx->quant_scale = qt->scale;
  return LSAPGPU_OK;
}

// Quantized filter copies for the long-row scan (scan_filter.cuh): a
// power-of-two scale with max|a| * scale <= 16383 (int16) or 127 (int8), from
// the max the layout pass reduced into flags_dev[2].  Normally the layout pass
// already wrote them with the probe rows' scale; a separate pass runs only if
// that scale does not hold for the whole matrix (or the layout was rebuilt).
int build_filter_copies(lsapgpu_ctx* ctx) {
  DevState& d = ctx->d;
  const ScanPlan& p = ctx->scan_plan;
  if (!ctx->quant_bits) {  // the layout pass did not reduce max|a| (no copies planned then): do it now
    CK(launch_amax(d, ctx->flags_dev + 2, ctx->stream));
    ++ctx->launches;
  }
  uint32_t bits = 0;
  CK(cpy(ctx, &bits, ctx->flags_dev + 2, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const float amax = bits_to_float(bits);
  const double limit = p.filter == 16 ? 16383.0 : 127.0;
  void *Q = nullptr, *QT = nullptr;
  if (ctx->quant_bits == p.filter && static_cast<double>(amax) * ctx->quant_scale <= limit) {
    const int rc = alloc_quant(ctx, p.filter, &Q, &QT);  // (already sized: same pointers)
    if (rc) return rc;
    d.Q = Q;
    d.QT = QT;
    d.qscale = ctx->quant_scale;
    ctx->quant_fused = true;
    return LSAPGPU_OK;
  }
  const double scale = quant_scale_for(amax, p.filter);
  const int rc = alloc_quant(ctx, p.filter, &Q, &QT);
  if (rc) return rc;
  d.Q = Q;
  d.QT = QT;
  d.qscale = scale;
  ctx->quant_fused = false;
  CK(launch_quantize(d, p.filter, scale, Q, QT, ctx->stream));
  ctx->launches += 2;
  return LSAPGPU_OK;
}

int finish_matrix(lsapgpu_ctx* ctx, int32_t n) {
  ctx->scan_plan = plan_scan(ctx->d, ctx->num_sms);
  ctx->commit_plan = plan_commit(ctx->d);
  DevState& d = ctx->d;
  d.Q = d.QT = nullptr;
  d.qscale = 0.0;
  if (ctx->scan_plan.filter) {
    const int rc = build_filter_copies(ctx);
    if (rc) return rc;
  } else if (ctx->qmat.p) {  // free the copies of a previous matrix
    cudaFree(ctx->qmat.p);
    ctx->qmat.p = nullptr;
    ctx->qmat.bytes = 0;
  }
  ctx->n_matrix = n;
  ctx->range_ok = false;
  return LSAPGPU_OK;
}

// Builds A/AT from a layout source; src_rows_dev is a device pointer for memory sources.
// The storage type is speculated from the first 64 rows, then ONE fused pass
// classifies every entry and builds A / AT; only if a later row needs a wider
// type is the layout rebuilt.
int build_from_source(lsapgpu_ctx* ctx, LayoutSource src, int32_t n) {
  int rc = ensure_vectors(ctx, n);
  if (rc) return rc;
  ctx->n_matrix = 0;
  CK(cudaMemsetAsync(ctx->flags_dev, 0, 4 * sizeof(uint32_t), ctx->stream));
  uint32_t fl4[4] = {};
  uint32_t flags = 0;
  int spec;
  // Same n as the last device matrix, whose plan built no filter copies (so
  // no probe max is needed): speculate its storage and skip the probe's
  // sync; the layout pass's flags decide as always (a wrong guess rebuilds).
  if (ctx->last_dev_n == n && ctx->last_dev_storage >= 0 && !ctx->scan_plan.filter && ctx->place_world <= 1) {
    spec = ctx->last_dev_storage;
  } else {
    const int64_t probe = std::min<int64_t>(64, n);
    CK(launch_classify(src, n, 0, probe, ctx->flags_dev, ctx->stream, ctx->flags_dev + 3));
    ++ctx->launches;
    CK(cpy(ctx, fl4, ctx->flags_dev, sizeof(fl4), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    flags = fl4[0];
    if (flags & 1u) return fail(ctx, LSAPGPU_ERR_INVALID, "benefit matrix contains a non-finite entry");
    spec = storage_of_flags(flags);
  }
  ctx->last_dev_storage = -1;  // (set again once this matrix is complete)
  if ((rc = alloc_matrix(ctx, n, spec))) return rc;
  set_source_rows(ctx, &src);
  DevState& d = ctx->d;
  QuantTarget qt;
  if ((rc = prepare_quant(ctx, spec, bits_to_float(fl4[3]), &qt))) return rc;
  CK(launch_layout_fused(src, n, 0, n, spec, const_cast<void*>(d.A), const_cast<void*>(d.AT), d.ld,
                         ctx->flags_dev + 1, ctx->stream, qt.bits ? ctx->flags_dev + 2 : nullptr, qt));
  ++ctx->launches;
  CK(cpy(ctx, &flags, ctx->flags_dev + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (flags & 1u) return fail(ctx, LSAPGPU_ERR_INVALID, "benefit matrix contains a non-finite entry");
  const int storage = storage_of_flags(flags);
  if (storage != spec) {
    ctx->quant_bits = 0;
    if ((rc = alloc_matrix(ctx, n, storage))) return rc;
    set_source_rows(ctx, &src);
    CK(launch_build_layout(src, n, 0, n, storage, const_cast<void*>(d.A), const_cast<void*>(d.AT), d.ld,
                           ctx->stream));
    ++ctx->launches;
    CK(cudaStreamSynchronize(ctx->stream));
  }
  const int frc = finish_matrix(ctx, n);
  if (frc == LSAPGPU_OK) {
    ctx->last_dev_storage = storage;
    ctx->last_dev_n = n;
  }
  return frc;
}

// Host upload (lsapgpu_set_matrix): the matrix crosses PCIe in row chunks
// into a device staging copy while the compute stream classifies each chunk
// (Instance::validate + narrowest-storage choice) and builds its rows of A
// and columns of AT.  The storage type is speculated from chunk 0; if a later
// chunk needs a wider type, the whole layout is rebuilt from the staging copy
// once the last chunk is in (only inputs whose first rows are narrower than
// the rest pay for that).  Pageable host memory is first copied into a ring
// of pinned buffers by a pool of host threads, so it streams at close to the
// pinned PCIe rate instead of the driver's single-threaded pageable path.
// Host-side classification of fp64 entries, the rules of the device's
// entry_flags (layout.cu): bit0 non-finite, bit1 not int16-exact, bit2 not an
// integer below 2^29, bit3 not fp32-exact.
uint32_t host_entry_flags(double v) {
  if (!std::isfinite(v)) return 15u;
  uint32_t f = 0;
  const bool i16 = v >= -32767.0 && v <= 32767.0 && static_cast<double>(static_cast<int32_t>(v)) == v;
  if (!i16) f |= 2u;
  const bool i32 = v > -536870912.0 && v < 536870912.0 && static_cast<double>(static_cast<int32_t>(v)) == v;
  if (!i32) f |= 4u;
  if (std::fabs(v) > 3.4028234663852886e38 || static_cast<double>(static_cast<float>(v)) != v) f |= 8u;
  return f;
}

inline bool narrow_block(const double* src, int16_t* dst, size_t cnt) { return lsapgpu::narrow_to_i16(src, dst, cnt); }
inline bool narrow_block(const double* src, int32_t* dst, size_t cnt) { return lsapgpu::narrow_to_i32(src, dst, cnt); }
inline bool narrow_block(const double* src, float* dst, size_t cnt) { return lsapgpu::narrow_to_f32(src, dst, cnt); }

constexpr int kNarrowFallback = 1000;  // upload_narrow: a value needs a wider type; redo as fp64

// pinned bounce buffers 0..slots-1 of at least `bytes` each
int ensure_ring(lsapgpu_ctx* ctx, int slots, size_t bytes) {
  for (int k = 0; k < slots; ++k) {
    if (ctx->ring[k] && ctx->ring_size[k] >= bytes) continue;
    if (ctx->ring[k]) cudaFreeHost(ctx->ring[k]);
    ctx->ring[k] = nullptr;
    ctx->ring_size[k] = 0;
    CK(cudaMallocHost(&ctx->ring[k], bytes));
    ctx->ring_size[k] = bytes;
  }
  return LSAPGPU_OK;
}

// The host upload with the matrix narrowed on the HOST (pool threads convert
// each chunk into the pinned ring as int16 / int32 / fp32, the storage type
// speculated from the first 64 rows): PCIe then carries 2 or 4 bytes per
// entry instead of 8, and the device builds A / AT from the narrow staging
// copy exactly as from fp64 (the narrowing is exact).  Any value that does
// not fit returns kNarrowFallback and the caller redoes the fp64 upload.
template <class T>
int upload_narrow(lsapgpu_ctx* ctx, const double* data, int32_t n, int storage, int32_t ndtype, float probe_amax) {
  static const bool host_timing = std::getenv("LSAPGPU_HOST_TIMING") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  std::vector<std::pair<const char*, double>> marks;
  auto mark = [&](const char* what) {
    if (host_timing)
      marks.emplace_back(what, std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_start).count());
  };
  const size_t row_bytes = static_cast<size_t>(n) * sizeof(T);
  const size_t total = row_bytes * static_cast<size_t>(n);
  if (ctx->stage.bytes < total) {
    if (ctx->stage.p) cudaFree(ctx->stage.p);
    ctx->stage.p = nullptr;
    ctx->stage.bytes = 0;
    CK(cudaMalloc(&ctx->stage.p, total));
    ctx->stage.bytes = total;
  }
  // chunks of ~32 MB of SOURCE (fp64) rows
  static const size_t chunk_src = std::getenv("LSAPGPU_NARROW_CHUNK_MB")
                                      ? static_cast<size_t>(std::max(1, std::atoi(std::getenv("LSAPGPU_NARROW_CHUNK_MB")))) << 20
                                      : kNarrowChunk;
  int64_t chunk_rows = static_cast<int64_t>(chunk_src / (static_cast<size_t>(n) * 8)) / 32 * 32;
  if (chunk_rows < 32) chunk_rows = 32;
  if (chunk_rows > n) chunk_rows = n;
  // Chunk row ranges: full chunks, except that the last full chunk's rows go
  // out as four quarter chunks -- the copy and layout pass after the last
  // host slice are on the critical path, so the final piece is kept small.
  std::vector<int64_t> cstart;
  for (int64_t r = 0; r < n; r += chunk_rows) cstart.push_back(r);
  if (cstart.size() >= 2 && chunk_rows >= 128) {
    const int64_t last = cstart.back(), q = chunk_rows / 4 / 32 * 32;
    if (n - last >= chunk_rows / 2) {  // a large last chunk: quarter it
      cstart.pop_back();
      for (int64_t k = 0; k < 4 && last + k * q < n; ++k) cstart.push_back(last + k * q);
    } else {  // a small remainder: quarter the full chunk before it
      const int64_t r0 = last - chunk_rows;
      cstart.pop_back();
      cstart.pop_back();
      for (int64_t k = 0; k < 4; ++k) cstart.push_back(r0 + k * q);
      cstart.push_back(last);
    }
  }
  const int nchunks = static_cast<int>(cstart.size());
  cstart.push_back(n);
  if (static_cast<int>(ctx->chunk_flags_cap) < nchunks) {
    if (ctx->chunk_flags) cudaFree(ctx->chunk_flags);
    ctx->chunk_flags = nullptr;
    ctx->chunk_flags_cap = 0;
    CK(cudaMalloc(&ctx->chunk_flags, sizeof(uint32_t) * nchunks));
    ctx->chunk_flags_cap = nchunks;
  }
  CK(cudaMemsetAsync(ctx->chunk_flags, 0, sizeof(uint32_t) * nchunks, ctx->stream));
  CK(cudaMemsetAsync(ctx->flags_dev + 2, 0, sizeof(uint32_t), ctx->stream));  // max |a| (filter scale)
  CK(cudaEventRecord(ctx->ev_ready, ctx->stream));
  CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_ready, 0));
  {
    const int rc = ensure_ring(ctx, kRingNarrow, static_cast<size_t>(chunk_rows) * row_bytes);
    if (rc) return rc;
  }
  if (!ctx->pool) ctx->pool = new HostPool(upload_threads());
  {
    const int rc = alloc_matrix(ctx, n, storage);
    if (rc) return rc;
  }
  QuantTarget qt;
  {
    const int rc = prepare_quant(ctx, storage, probe_amax, &qt);
    if (rc) return rc;
  }
  LayoutSource src;
  src.kind = 0;
  src.src = ctx->stage.p;
  src.src_dtype = ndtype;
  set_source_rows(ctx, &src);
  // No barrier per chunk: every pool thread walks all chunks, converting its
  // slice of each into the chunk's pinned ring slot, and the thread that
  // completes a chunk (the last slice in) enqueues its copy and layout pass
  // (chunks may go out in any order: each layout pass waits on its own copy
  // and writes its own rows / columns).  A thread refills a ring slot only
  // once the copy that last read it has been enqueued and has completed, so
  // the threads run up to kRingNarrow chunks ahead of the DMA instead of
  // meeting at a join per chunk, and no thread waits for the others.
  mark("setup");
  const int T_ = ctx->pool->size();
  std::unique_ptr<std::atomic<int>[]> filled(new std::atomic<int>[nchunks]);
  for (int k = 0; k < nchunks; ++k) filled[k].store(0, std::memory_order_relaxed);
  std::unique_ptr<std::atomic<int>[]> issued(new std::atomic<int>[nchunks]);  // copy + ring event enqueued
  for (int k = 0; k < nchunks; ++k) issued[k].store(0, std::memory_order_relaxed);
  std::mutex issue_mu;  // the enqueue (stream order, context counters) is one thread at a time
  std::atomic<int> stop{0};     // 1: a value needs a wider type, 2: CUDA error
  cudaError_t issue_err = cudaSuccess, wait_err = cudaSuccess;
  const int device = ctx->device;
  cudaSetDevice(device);
  std::vector<double> wait_us(static_cast<size_t>(T_), 0.0), conv_us(static_cast<size_t>(T_), 0.0);
  auto now_us = [] {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  ctx->pool->run([&](int t) {
    if (t) cudaSetDevice(device);  // ring events are waited on, and chunks enqueued, from every thread
    for (int k = 0; k < nchunks && !stop.load(std::memory_order_relaxed); ++k) {
      const int64_t r0 = cstart[static_cast<size_t>(k)];
      const int64_t rows = cstart[static_cast<size_t>(k) + 1] - r0;
      const size_t cnt = static_cast<size_t>(rows) * static_cast<size_t>(n);
      const int b = k % kRingNarrow;
      const double tw0 = host_timing ? now_us() : 0.0;
      if (k >= kRingNarrow) {  // slot b last held chunk k - kRingNarrow
        while (!issued[k - kRingNarrow].load(std::memory_order_acquire) && !stop.load(std::memory_order_relaxed))
          _mm_pause();
        if (stop.load(std::memory_order_relaxed)) break;
        const cudaError_t e = cudaEventSynchronize(ctx->ev_chunk[b]);
        if (e != cudaSuccess) {
          wait_err = e;
          stop.store(2);
          break;
        }
      }
      T* pin = static_cast<T*>(ctx->ring[b]);
      const double* hsrc = data + static_cast<size_t>(r0) * static_cast<size_t>(n);
      // slices of whole 16-byte groups: streaming stores need the alignment
      const size_t a = cnt * t / T_ / 8 * 8, e = t + 1 == T_ ? cnt : cnt * (t + 1) / T_ / 8 * 8;
      const double tw1 = host_timing ? now_us() : 0.0;
      const bool ok_slice = narrow_block(hsrc + a, pin + a, e - a);
      if (host_timing) {
        const double tw2 = now_us();
        wait_us[t] += tw1 - tw0;
        conv_us[t] += tw2 - tw1;
      }
      if (!ok_slice) {
        int z = 0;
        stop.compare_exchange_strong(z, 1);
        break;
      }
      if (filled[k].fetch_add(1, std::memory_order_acq_rel) != T_ - 1) continue;  // not the last slice
      std::lock_guard<std::mutex> lk(issue_mu);
      if (stop.load(std::memory_order_relaxed)) break;
      unsigned char* dst = static_cast<unsigned char*>(ctx->stage.p) + static_cast<size_t>(r0) * row_bytes;
      cudaError_t ce = cpy(ctx, dst, pin, cnt * sizeof(T), cudaMemcpyHostToDevice, ctx->copy_stream);
      if (ce == cudaSuccess) ce = cudaEventRecord(ctx->ev_chunk[b], ctx->copy_stream);
      if (ce == cudaSuccess) ce = cudaStreamWaitEvent(ctx->stream, ctx->ev_chunk[b], 0);
      if (ce == cudaSuccess)
        ce = launch_layout_fused(src, n, r0, rows, storage, const_cast<void*>(ctx->d.A), const_cast<void*>(ctx->d.AT),
                                 ctx->d.ld, ctx->chunk_flags + k, ctx->stream,
                                 qt.bits ? ctx->flags_dev + 2 : nullptr, qt);
      if (ce != cudaSuccess) {
        issue_err = ce;
        stop.store(2);
        break;
      }
      ++ctx->launches;
      issued[k].store(1, std::memory_order_release);
      if (k == 0 || k + 1 == nchunks) mark(k ? "last chunk issued" : "chunk 0 issued");
    }
  });
  if (stop.load() == 2) {
    CK(issue_err);
    CK(wait_err);
  }
  if (stop.load() == 1) {
    CK(cudaStreamSynchronize(ctx->copy_stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return kNarrowFallback;
  }
  mark("host done");
  std::vector<uint32_t> fl(nchunks);
  CK(cpy(ctx, fl.data(), ctx->chunk_flags, sizeof(uint32_t) * nchunks, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  mark("device done");
  uint32_t all = 0;
  for (uint32_t f : fl) all |= f;
  const int final_storage = storage_of_flags(all);
  if (final_storage != storage) {  // (cannot widen: every value passed T's rule; narrower is possible)
    ctx->quant_bits = 0;
    int rc = alloc_matrix(ctx, n, final_storage);
    if (rc) return rc;
    set_source_rows(ctx, &src);
    CK(launch_build_layout(src, n, 0, n, final_storage, const_cast<void*>(ctx->d.A), const_cast<void*>(ctx->d.AT),
                           ctx->d.ld, ctx->stream));
    ++ctx->launches;
    CK(cudaStreamSynchronize(ctx->stream));
  }
  if (total > kStageKeep) {
    cudaFree(ctx->stage.p);
    ctx->stage.p = nullptr;
    ctx->stage.bytes = 0;
  }
  const int frc = finish_matrix(ctx, n);
  mark("finished");
  if (host_timing) {
    std::string line = "lsapgpu upload timing (us, " + std::to_string(nchunks) + " chunks, " +
                       std::to_string(T_) + " threads; thread 1 ring wait " +
                       std::to_string(static_cast<int>(wait_us[T_ > 1 ? 1 : 0])) + " convert " +
                       std::to_string(static_cast<int>(conv_us[T_ > 1 ? 1 : 0])) + "):";
    for (const auto& m : marks) line += std::string(" ") + m.first + "=" + std::to_string(static_cast<int>(m.second));
    std::fprintf(stderr, "%s\n", line.c_str());
  }
  return frc;
}

int upload_host(lsapgpu_ctx* ctx, const void* data, int32_t n, int32_t dtype) {
  int rc = ensure_vectors(ctx, n);
  if (rc) return rc;
  ctx->n_matrix = 0;
  static const bool narrow_env = !(std::getenv("LSAPGPU_HOST_NARROW") && std::atoi(std::getenv("LSAPGPU_HOST_NARROW")) == 0);
  if (dtype == LSAPGPU_F64 && narrow_env) {
    // speculate the storage from the first rows on the host
    const double* a = static_cast<const double*>(data);
    const size_t probe = static_cast<size_t>(std::min<int32_t>(64, n)) * static_cast<size_t>(n);
    if (!ctx->pool) ctx->pool = new HostPool(upload_threads());
    const int T_ = ctx->pool->size();
    std::vector<uint32_t> pf(static_cast<size_t>(T_), 0u);
    std::vector<double> pm(static_cast<size_t>(T_), 0.0);
    ctx->pool->run([&](int t) {
      uint32_t f = 0;
      double m = 0.0;
      for (size_t i = probe * t / T_; i < probe * (t + 1) / T_; ++i) {
        f |= host_entry_flags(a[i]);
        if (std::isfinite(a[i])) m = std::max(m, std::fabs(a[i]));
      }
      pf[t] = f;
      pm[t] = m;
    });
    uint32_t f = 0;
    double pmax = 0.0;
    for (uint32_t x : pf) f |= x;
    for (double x : pm) pmax = std::max(pmax, x);
    // max |a| of the probe rows as a float rounded up (like the device's __double2float_ru)
    float pamax = static_cast<float>(pmax);
    if (static_cast<double>(pamax) < pmax) pamax = std::nextafter(pamax, INFINITY);
    if (f & 1u) return fail(ctx, LSAPGPU_ERR_INVALID, "benefit matrix contains a non-finite entry");
    const int spec = storage_of_flags(f);
    rc = kNarrowFallback;
    if (spec == kI16) rc = upload_narrow<int16_t>(ctx, a, n, kI16, LSAPGPU_I16, pamax);
    else if (spec == kI32) rc = upload_narrow<int32_t>(ctx, a, n, kI32, LSAPGPU_I32, pamax);
    else if (spec == kF32) rc = upload_narrow<float>(ctx, a, n, kF32, LSAPGPU_F32, pamax);
    if (rc != kNarrowFallback) return rc;
  }
  const size_t es = src_size(dtype);
  const size_t row_bytes = static_cast<size_t>(n) * es;
  const size_t total = row_bytes * static_cast<size_t>(n);
  // staging copy of the source matrix (kept for reuse up to 16 GB)
  if (ctx->stage.bytes < total) {
    if (ctx->stage.p) cudaFree(ctx->stage.p);
    ctx->stage.p = nullptr;
    ctx->stage.bytes = 0;
    CK(cudaMalloc(&ctx->stage.p, total));
    ctx->stage.bytes = total;
  }
  int64_t chunk_rows = static_cast<int64_t>(kUploadChunk / row_bytes) / 32 * 32;
  if (chunk_rows < 32) chunk_rows = 32;
  if (chunk_rows > n) chunk_rows = n;
  const int nchunks = static_cast<int>((n + chunk_rows - 1) / chunk_rows);
  if (static_cast<int>(ctx->chunk_flags_cap) < nchunks) {
    if (ctx->chunk_flags) cudaFree(ctx->chunk_flags);
    ctx->chunk_flags = nullptr;
    ctx->chunk_flags_cap = 0;
    CK(cudaMalloc(&ctx->chunk_flags, sizeof(uint32_t) * nchunks));
    ctx->chunk_flags_cap = nchunks;
  }
  CK(cudaMemsetAsync(ctx->chunk_flags, 0, sizeof(uint32_t) * nchunks, ctx->stream));
  CK(cudaMemsetAsync(ctx->flags_dev + 2, 0, sizeof(uint32_t), ctx->stream));  // max |a| (filter scale)
  CK(cudaEventRecord(ctx->ev_ready, ctx->stream));
  CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_ready, 0));

  cudaPointerAttributes attr{};
  const bool pinned = cudaPointerGetAttributes(&attr, data) == cudaSuccess &&
                      (attr.type == cudaMemoryTypeHost || attr.type == cudaMemoryTypeDevice ||
                       attr.type == cudaMemoryTypeManaged);
  cudaGetLastError();
  if (!pinned) {
    const int rc = ensure_ring(ctx, kRing, static_cast<size_t>(chunk_rows) * row_bytes);
    if (rc) return rc;
  }
  if (!pinned && !ctx->pool) ctx->pool = new HostPool(upload_threads());

  int storage = -1;
  QuantTarget qt;
  LayoutSource src;
  src.kind = 0;
  src.src = ctx->stage.p;
  src.src_dtype = dtype;
  for (int k = 0; k < nchunks; ++k) {
    const int64_t r0 = static_cast<int64_t>(k) * chunk_rows;
    const int64_t rows = std::min<int64_t>(chunk_rows, n - r0);
    const size_t off = static_cast<size_t>(r0) * row_bytes, len = static_cast<size_t>(rows) * row_bytes;
    unsigned char* dst = static_cast<unsigned char*>(ctx->stage.p) + off;
    const unsigned char* hsrc = static_cast<const unsigned char*>(data) + off;
    cudaEvent_t done = ctx->ev_chunk[k % kRing];
    if (pinned) {
      CK(cpy(ctx, dst, hsrc, len, cudaMemcpyHostToDevice, ctx->copy_stream));
    } else {
      const int b = k % kRing;
      if (k >= kRing) CK(cudaEventSynchronize(ctx->ev_chunk[b]));  // ring slot's previous DMA done
      unsigned char* pin = static_cast<unsigned char*>(ctx->ring[b]);
      const int T = ctx->pool->size();
      ctx->pool->run([&](int t) {
        const size_t a = len * t / T, e = len * (t + 1) / T;
        std::memcpy(pin + a, hsrc + a, e - a);
      });
      CK(cpy(ctx, dst, pin, len, cudaMemcpyHostToDevice, ctx->copy_stream));
    }
    CK(cudaEventRecord(done, ctx->copy_stream));
    CK(cudaStreamWaitEvent(ctx->stream, done, 0));
    if (k == 0) {  // speculate the storage from the first rows
      CK(cudaMemsetAsync(ctx->flags_dev + 3, 0, sizeof(uint32_t), ctx->stream));
      CK(launch_classify(src, n, r0, std::min<int64_t>(rows, 64), ctx->chunk_flags + k, ctx->stream,
                         ctx->flags_dev + 3));
      ++ctx->launches;
      uint32_t f0 = 0, pa = 0;
      CK(cpy(ctx, &f0, ctx->chunk_flags, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cpy(ctx, &pa, ctx->flags_dev + 3, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      if (f0 & 1u) {
        CK(cudaStreamSynchronize(ctx->copy_stream));
        return fail(ctx, LSAPGPU_ERR_INVALID, "benefit matrix contains a non-finite entry");
      }
      storage = storage_of_flags(f0);
      if ((rc = alloc_matrix(ctx, n, storage)) || (rc = prepare_quant(ctx, storage, bits_to_float(pa), &qt))) {
        cudaStreamSynchronize(ctx->copy_stream);
        return rc;
      }
      set_source_rows(ctx, &src);
    }
    CK(launch_layout_fused(src, n, r0, rows, storage, const_cast<void*>(ctx->d.A),
                           const_cast<void*>(ctx->d.AT), ctx->d.ld, ctx->chunk_flags + k, ctx->stream,
                           qt.bits ? ctx->flags_dev + 2 : nullptr, qt));
    ++ctx->launches;
  }
  std::vector<uint32_t> fl(nchunks);
  CK(cpy(ctx, fl.data(), ctx->chunk_flags, sizeof(uint32_t) * nchunks, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  uint32_t all = 0;
  for (uint32_t f : fl) all |= f;
  if (all & 1u) return fail(ctx, LSAPGPU_ERR_INVALID, "benefit matrix contains a non-finite entry");
  const int final_storage = storage_of_flags(all);
  if (final_storage != storage) {  // a later chunk needs a wider type: rebuild everything
    ctx->quant_bits = 0;
    if ((rc = alloc_matrix(ctx, n, final_storage))) return rc;
    set_source_rows(ctx, &src);
    CK(launch_build_layout(src, n, 0, n, final_storage, const_cast<void*>(ctx->d.A),
                           const_cast<void*>(ctx->d.AT), ctx->d.ld, ctx->stream));
    ++ctx->launches;
    CK(cudaStreamSynchronize(ctx->stream));
  }
  if (total > kStageKeep) {
    cudaFree(ctx->stage.p);
    ctx->stage.p = nullptr;
    ctx->stage.bytes = 0;
  }
  return finish_matrix(ctx, n);
}

bool is_perm(const int32_t* p, int32_t n) {
  std::vector<uint8_t> seen(n, 0);
  for (int32_t k = 0; k < n; ++k) {
    if (p[k] < 0 || p[k] >= n || seen[p[k]]) return false;
    seen[p[k]] = 1;
  }
  return true;
}

// Ordered objective (core.cpp:17-24) over the device matrix and a device sigma.
// Enqueue the objective gather into pinned memory (no sync); objective_sum
// adds it up in job order once the stream has been synchronised.
int enqueue_objective(lsapgpu_ctx* ctx, bool pack = false) {
  const int32_t n = ctx->d.n;
  if (ctx->obj_cap < n) {
    if (ctx->obj_pin) cudaFreeHost(ctx->obj_pin);
    ctx->obj_pin = nullptr;
    ctx->obj_cap = 0;
    CK(cudaMallocHost(&ctx->obj_pin, sizeof(double) * 2 * n));  // room for the packed sigma / tau
    ctx->obj_cap = n;
  }
  double* dv = reinterpret_cast<double*>(ctx->d.c_delta);  // scratch (2n doubles)
  CK(launch_gather_current(ctx->d, dv, ctx->stream, pack ? 1 : 0));
  ++ctx->launches;
  CK(cpy(ctx, ctx->obj_pin, dv, sizeof(double) * (pack ? 2 : 1) * n, cudaMemcpyDeviceToHost, ctx->stream));
  return LSAPGPU_OK;
}
double objective_sum(const lsapgpu_ctx* ctx) {  // core.cpp:17-24: ordered sum over jobs
  double sum = 0.0;
  for (int32_t j = 0; j < ctx->d.n; ++j) sum += ctx->obj_pin[j];
  return sum;
}

int device_objective(lsapgpu_ctx* ctx, double* value) {
  const int32_t n = ctx->d.n;
  double* dv = reinterpret_cast<double*>(ctx->d.c_delta);  // scratch (2n doubles)
  CK(launch_gather_current(ctx->d, dv, ctx->stream));
  ++ctx->launches;
  std::vector<double> hv(n);
  CK(cpy(ctx, hv.data(), dv, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  double sum = 0.0;
  for (int32_t j = 0; j < n; ++j) sum += hv[j];
  *value = sum;
  return LSAPGPU_OK;
}

// Greedy assignment (greedy.cu) into d.sigma on the context's stream.
int run_greedy(lsapgpu_ctx* ctx) {
  DevState& d = ctx->d;
  GreedyDev& g = ctx->gr;
  if (ctx->gr_n != d.n) {
    const size_t N = static_cast<size_t>(d.ld);
    CK(valloc(ctx, &g.list[0], N, false));
    CK(valloc(ctx, &g.list[1], N, false));
    CK(valloc(ctx, &g.free, N / 32 + 1, false));
    CK(valloc(ctx, &g.claim, N, false));
    CK(valloc(ctx, &g.slot, 2 * N, true));  // empty slots; every award resets its slot
    CK(valloc(ctx, &g.ctrl, 1, true));
    ctx->gr_n = d.n;
  }
  CK(launch_greedy(d, g, ctx->num_sms, ctx->stream));
  ++ctx->launches;
  return LSAPGPU_OK;
}

int build_graph(lsapgpu_ctx* ctx) {
  drop_graph(ctx);
  CK(cudaGraphCreate(&ctx->graph, 0));
  cudaGraphConditionalHandle cond;
  CK(cudaGraphConditionalHandleCreate(&cond, ctx->graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = cond;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, ctx->graph, nullptr, 0, &p));
  cudaGraph_t body = p.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal));
  cudaError_t e1 = launch_commit(ctx->d, ctx->commit_plan, kCommitSolve, cond, 1, ctx->stream);
  cudaError_t e2 = launch_scan(ctx->d, ctx->scan_plan, 0, ctx->stream);
  cudaGraph_t captured = body;
  CK(cudaStreamEndCapture(ctx->stream, &captured));
  CK(e1);
  CK(e2);
  CK(cudaGraphInstantiate(&ctx->exec, ctx->graph, 0));
  ctx->graph_state = ctx->d;
  ctx->graph_scan = ctx->scan_plan;
  ctx->graph_commit = ctx->commit_plan;
  return LSAPGPU_OK;
}

// Inner-loop graph of the multi-GPU peer transport: no host step inside a
// batch, so the whole {commit, apply, own items, scan, push, wait, merge}
// loop is one conditional WHILE node, like the single-GPU graph.
int build_dist_graph(lsapgpu_ctx* ctx, const PeerSet& ps) {
  if (ctx->dist_exec) cudaGraphExecDestroy(ctx->dist_exec);
  if (ctx->dist_graph) cudaGraphDestroy(ctx->dist_graph);
  ctx->dist_exec = nullptr;
  ctx->dist_graph = nullptr;
  CK(cudaGraphCreate(&ctx->dist_graph, 0));
  cudaGraphConditionalHandle cond;
  CK(cudaGraphConditionalHandleCreate(&cond, ctx->dist_graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = cond;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, ctx->dist_graph, nullptr, 0, &p));
  cudaGraph_t body = p.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  const DevState& d = ctx->d;
  cudaError_t e = launch_commit(d, ctx->commit_plan, kCommitSolve, cond, 1, ctx->stream);
  if (e == cudaSuccess) e = launch_dist_own_items(d, 0, ps.rank, ps.world, ctx->stream);
  DevState ds = d;
  ds.use_own = 1;
  ds.emit_edges = 0;
  if (e == cudaSuccess) e = launch_scan(ds, ctx->scan_plan, 0, ctx->stream);
  if (e == cudaSuccess) e = launch_dist_push(d, ps, ctx->stream);
  cudaGraph_t captured = body;
  CK(cudaStreamEndCapture(ctx->stream, &captured));
  CK(e);
  CK(cudaGraphInstantiate(&ctx->dist_exec, ctx->dist_graph, 0));
  ctx->dist_state = d;
  ctx->dist_ps = ps;
  return LSAPGPU_OK;
}

int run_scan(lsapgpu_ctx* ctx, int full) {
  if (ctx->timing) CK(cudaEventRecord(ctx->ev0, ctx->stream));
  CK(launch_scan(ctx->d, ctx->scan_plan, full, ctx->stream));
  ctx->launches += ctx->scan_plan.launches();
  if (ctx->timing) {
    CK(cudaEventRecord(ctx->ev1, ctx->stream));
    CK(cudaEventSynchronize(ctx->ev1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    ctx->scan_ms += ms;
    ++ctx->scan_launches;
    if (full) {
      ctx->full_ms += ms;
      ++ctx->full_launches;
    }
  }
  return LSAPGPU_OK;
}

// Stable two-pass counting sort of the delta log by (iter, slot): O(entries + slots).
void order_log(const LogEntry* in, size_t N, std::vector<LogEntry>& out, int32_t slots) {
  out.resize(N);
  if (N == 0) return;
  static thread_local std::vector<LogEntry> tmp;
  static thread_local std::vector<int64_t> count;
  tmp.resize(N);
  count.assign(static_cast<size_t>(slots) + 1, 0);
  for (size_t k = 0; k < N; ++k) ++count[static_cast<size_t>(in[k].slot) + 1];
  for (size_t k = 1; k < count.size(); ++k) count[k] += count[k - 1];
  for (size_t k = 0; k < N; ++k) tmp[static_cast<size_t>(count[in[k].slot]++)] = in[k];
  int32_t lo = tmp[0].iter, hi = tmp[0].iter;
  for (const auto& e : tmp) {
    lo = std::min(lo, e.iter);
    hi = std::max(hi, e.iter);
  }
  count.assign(static_cast<size_t>(hi - lo) + 2, 0);
  for (const auto& e : tmp) ++count[static_cast<size_t>(e.iter - lo) + 1];
  for (size_t k = 1; k < count.size(); ++k) count[k] += count[k - 1];
  for (const auto& e : tmp) out[static_cast<size_t>(count[e.iter - lo]++)] = e;
}

struct TraceSink {
  int64_t* ts;
  double* tv;
  int64_t cap;
  int64_t len = 0;
  void push(int64_t sw, double v, bool force = false) {
    if (!force && len >= kTraceCap) return;
    if (ts && tv && len < cap) {
      ts[len] = sw;
      tv[len] = v;
    }
    ++len;
  }
};

}  // namespace

extern "C" {

const char* lsapgpu_version(void) { return "paper_1106_5694_b200 lsapgpu 0.1 (sm_100a)"; }

int lsapgpu_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
  return c;
}

int lsapgpu_create(lsapgpu_ctx** out, int device) {
  if (!out) return LSAPGPU_ERR_INVALID;
  *out = nullptr;
  auto* ctx = new lsapgpu_ctx();
  ctx->device = device;
  int major = 0;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess) {
    delete ctx;
    return LSAPGPU_ERR_CUDA;
  }
  if (major < 10) {
    delete ctx;
    return LSAPGPU_ERR_CUDA;
  }
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  ctx->d.pdl = 1;  // programmatic dependent launch for the inner-loop kernels (LSAPGPU_PDL=0: off)
  if (const char* e = std::getenv("LSAPGPU_PDL")) ctx->d.pdl = std::atoi(e) != 0;
  if (const char* e = std::getenv("LSAPGPU_FILTER_CHECK")) ctx->d.filter_check = std::max(0, std::atoi(e));
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&ctx->ctrl_dev, sizeof(Ctrl)) != cudaSuccess ||
      cudaMallocHost(&ctx->ctrl_host, sizeof(Ctrl)) != cudaSuccess ||
      cudaMalloc(&ctx->flags_dev, 4 * sizeof(uint32_t)) != cudaSuccess ||
      cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_ready, cudaEventDisableTiming) != cudaSuccess) {
    lsapgpu_destroy(ctx);
    return LSAPGPU_ERR_CUDA;
  }
  for (auto& e : ctx->ev_chunk) {
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      lsapgpu_destroy(ctx);
      return LSAPGPU_ERR_CUDA;
    }
  }
  std::memset(ctx->ctrl_host, 0, sizeof(Ctrl));
  ctx->ctrl_host->round = 1;
  cudaMemcpy(ctx->ctrl_dev, ctx->ctrl_host, sizeof(Ctrl), cudaMemcpyHostToDevice);
  *out = ctx;
  return LSAPGPU_OK;
}

void lsapgpu_destroy(lsapgpu_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  drop_graph(ctx);
  if (ctx->dist_exec) cudaGraphExecDestroy(ctx->dist_exec);
  if (ctx->dist_graph) cudaGraphDestroy(ctx->dist_graph);
  free_vectors(ctx);
  if (ctx->mat.p) cudaFree(ctx->mat.p);
  if (ctx->qmat.p) cudaFree(ctx->qmat.p);
  if (ctx->ctrl_dev) cudaFree(ctx->ctrl_dev);
  if (ctx->ctrl_host) cudaFreeHost(ctx->ctrl_host);
  if (ctx->flags_dev) cudaFree(ctx->flags_dev);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->d.tl) cudaFree(ctx->d.tl);
  if (ctx->obj_pin) cudaFreeHost(ctx->obj_pin);
  if (ctx->au_host) cudaFreeHost(ctx->au_host);
  if (ctx->perm_pin) cudaFreeHost(ctx->perm_pin);
  if (ctx->ctrl_base) cudaFreeHost(ctx->ctrl_base);
  if (ctx->eps_dev) cudaFree(ctx->eps_dev);
  if (ctx->log_pin) cudaFreeHost(ctx->log_pin);
  if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
  if (ctx->stage.p) cudaFree(ctx->stage.p);
  if (ctx->chunk_flags) cudaFree(ctx->chunk_flags);
  for (auto& r : ctx->ring)
    if (r) cudaFreeHost(r);
  delete ctx->pool;
  for (auto& e : ctx->ev_chunk)
    if (e) cudaEventDestroy(e);
  if (ctx->ev_ready) cudaEventDestroy(ctx->ev_ready);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* lsapgpu_last_error(const lsapgpu_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void* lsapgpu_stream(lsapgpu_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int32_t lsapgpu_n(const lsapgpu_ctx* ctx) { return ctx ? ctx->n_matrix : 0; }
int32_t lsapgpu_storage(const lsapgpu_ctx* ctx) { return ctx && ctx->n_matrix ? ctx->d.storage : -1; }

int lsapgpu_set_placement(lsapgpu_ctx* ctx, int32_t rank, int32_t world) {
  if (!ctx) return LSAPGPU_ERR_INVALID;
  if (world < 1 || rank < 0 || rank >= world) return fail(ctx, LSAPGPU_ERR_INVALID, "invalid rank / world");
  if (ctx->place_rank != rank || ctx->place_world != world) {
    ctx->place_rank = rank;
    ctx->place_world = world;
    ctx->n_matrix = 0;  // the layout depends on it: set the matrix again
    drop_graph(ctx);
  }
  return LSAPGPU_OK;
}

int lsapgpu_set_matrix_device(lsapgpu_ctx* ctx, const void* dev_data, int32_t n, int32_t dtype) {
  if (!ctx) return LSAPGPU_ERR_INVALID;
  CK(cudaSetDevice(ctx->device));
  if (n < 1) return fail(ctx, LSAPGPU_ERR_INVALID, "instance size must be >= 1, got " + std::to_string(n));
  if (dtype < 0 || dtype > 3) return fail(ctx, LSAPGPU_ERR_INVALID, "unknown matrix dtype");
  if (n >= (1 << 30)) return fail(ctx, LSAPGPU_ERR_INVALID, "n >= 2^30 is not supported by this build");
  LayoutSource s;
  s.kind = 0;
  s.src = dev_data;
  s.src_dtype = dtype;
  return build_from_source(ctx, s, n);
}

int lsapgpu_set_matrix(lsapgpu_ctx* ctx, const void* data, int32_t n, int32_t dtype) {
  if (!ctx) return LSAPGPU_ERR_INVALID;
  CK(cudaSetDevice(ctx->device));
  if (n < 1) return fail(ctx, LSAPGPU_ERR_INVALID, "instance size must be >= 1, got " + std::to_string(n));
  if (dtype < 0 || dtype > 3) return fail(ctx, LSAPGPU_ERR_INVALID, "unknown matrix dtype");
  if (n >= (1 << 30)) return fail(ctx, LSAPGPU_ERR_INVALID, "n >= 2^30 is not supported by this build");
  if (!data) return fail(ctx, LSAPGPU_ERR_INVALID, "null benefit matrix");
  return upload_host(ctx, data, n, dtype);
}

int lsapgpu_generate(lsapgpu_ctx* ctx, int32_t kind, int32_t n, uint64_t seed, double param) {
  if (!ctx) return LSAPGPU_ERR_INVALID;
  CK(cudaSetDevice(ctx->device));
  if (n < 1) return fail(ctx, LSAPGPU_ERR_INVALID, "instance size must be >= 1, got " + std::to_string(n));
  if (kind < 1 || kind > 5) return fail(ctx, LSAPGPU_ERR_INVALID, "unknown generator kind");
  if (n >= (1 << 30)) return fail(ctx, LSAPGPU_ERR_INVALID, "n >= 2^30 is not supported by this build");
  if (kind == LSAPGPU_GEN_UNIFORM_INT && !(param >= 1.0))
    return fail(ctx, LSAPGPU_ERR_INVALID, "uniform int modulus must be >= 1");
  if (kind == LSAPGPU_GEN_GEOM && !(param > 0.0)) return fail(ctx, LSAPGPU_ERR_INVALID, "geom: bound must be > 0");
  double* aux = nullptr;
  CK(cudaMalloc(&aux, sizeof(double) * 3 * static_cast<size_t>(n)));
  LayoutSource s;
  s.kind = kind;
  s.seed = seed;
  s.param = param;
  s.aux = aux;
  cudaError_t e = launch_gen_aux(s, n, aux, ctx->stream);
  int rc = e == cudaSuccess ? build_from_source(ctx, s, n)
                            : fail(ctx, LSAPGPU_ERR_CUDA, cudaGetErrorString(e));
  cudaStreamSynchronize(ctx->stream);
  cudaFree(aux);
  return rc;
}

int lsapgpu_read_rows(lsapgpu_ctx* ctx, const int32_t* rows, int32_t nrows, double* out) {
  if (!ctx || !ctx->n_matrix) return fail(ctx, LSAPGPU_ERR_STATE, "no matrix set");
  CK(cudaSetDevice(ctx->device));
  const int32_t n = ctx->n_matrix;
  for (int32_t r = 0; r < nrows; ++r)
    if (rows[r] < 0 || rows[r] >= n) return fail(ctx, LSAPGPU_ERR_INVALID, "row index out of range");
  int32_t* drows = nullptr;
  double* dout = nullptr;
  CK(cudaMalloc(&drows, sizeof(int32_t) * std::max(nrows, 1)));
  CK(cudaMalloc(&dout, sizeof(double) * std::max<size_t>(1, static_cast<size_t>(nrows) * n)));
  CK(cpy(ctx, drows, rows, sizeof(int32_t) * nrows, cudaMemcpyHostToDevice, ctx->stream));
  CK(launch_read_rows(ctx->d, drows, nrows, dout, ctx->stream));
  ++ctx->launches;
  CK(cpy(ctx, out, dout, sizeof(double) * static_cast<size_t>(nrows) * n, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  cudaFree(drows);
  cudaFree(dout);
  return LSAPGPU_OK;
}

void lsapgpu_random_perm(int32_t n, uint64_t seed, int32_t* p) {
  // rng.hpp:37-46 (Fisher-Yates over splitmix64)
  for (int32_t i = 0; i < n; ++i) p[i] = i;
  uint64_t state = seed;
  for (int32_t i = n - 1; i > 0; --i) {
    uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    const int32_t j = static_cast<int32_t>(z % static_cast<uint64_t>(i + 1));
    std::swap(p[i], p[j]);
  }
}

int lsapgpu_objective(lsapgpu_ctx* ctx, const int32_t* sigma, double* value) {
  if (!ctx || !ctx->n_matrix) return fail(ctx, LSAPGPU_ERR_STATE, "no matrix set");
  CK(cudaSetDevice(ctx->device));
  const int32_t n = ctx->n_matrix;
  if (!is_perm(sigma, n)) return fail(ctx, LSAPGPU_ERR_INVALID, "invalid assignment: not a permutation");
  CK(cpy(ctx, ctx->d.sigma, sigma, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  return device_objective(ctx, value);
}

int lsapgpu_counters(const lsapgpu_ctx* ctx, int64_t* h2d_bytes, int64_t* d2h_bytes,
                     int64_t* kernel_launches) {
  if (!ctx) return LSAPGPU_ERR_INVALID;
  if (h2d_bytes) *h2d_bytes = ctx->h2d;
  if (d2h_bytes) *d2h_bytes = ctx->d2h;
  if (kernel_launches) *kernel_launches = ctx->launches;
  return LSAPGPU_OK;
}

int lsapgpu_set_scan_timing(lsapgpu_ctx* ctx, int enabled) {
  if (!ctx) return LSAPGPU_ERR_INVALID;
  ctx->timing = enabled != 0;
  return LSAPGPU_OK;
}

int lsapgpu_set_timeline(lsapgpu_ctx* ctx, int32_t capacity) {
  if (!ctx) return LSAPGPU_ERR_INVALID;
  CK(cudaSetDevice(ctx->device));
  if (ctx->d.tl) cudaFree(ctx->d.tl);
  if (ctx->obj_pin) cudaFreeHost(ctx->obj_pin);
  if (ctx->log_pin) cudaFreeHost(ctx->log_pin);
  ctx->d.tl = nullptr;
  ctx->d.tl_cap = 0;
  if (capacity > 0) {
    CK(cudaMalloc(&ctx->d.tl, sizeof(unsigned long long) * capacity));
    ctx->d.tl_cap = capacity;
  }
  drop_graph(ctx);  // the graph captured the old DevState
  return LSAPGPU_OK;
}

int32_t lsapgpu_timeline(lsapgpu_ctx* ctx, uint64_t* out, int32_t capacity) {
  if (!ctx || !ctx->d.tl) return 0;
  if (pull_ctrl(ctx)) return 0;
  const int32_t cnt = std::min(ctx->ctrl_host->tl_count, std::min(capacity, ctx->d.tl_cap));
  if (cnt > 0 && cudaMemcpy(out, ctx->d.tl, sizeof(uint64_t) * cnt, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  ctx->ctrl_host->tl_count = 0;
  push_ctrl(ctx);
  cudaStreamSynchronize(ctx->stream);
  return cnt;
}

int lsapgpu_scan_plan(const lsapgpu_ctx* ctx, int32_t* info, int32_t cap) {
  if (!ctx || !info || cap < 0) return LSAPGPU_ERR_INVALID;
  const ScanPlan& p = ctx->scan_plan;
  const int32_t v[10] = {p.filter ? 2 : (p.resident ? 1 : 0), p.m, p.bufs, p.filter, p.ctas, p.threads,
                         static_cast<int32_t>(p.smem), static_cast<int32_t>(p.chunk), p.filter_queue, p.filter_tmem};
  const int32_t k = cap < 10 ? cap : 10;
  for (int32_t q = 0; q < k; ++q) info[q] = v[q];
  return k;
}

int lsapgpu_scan_timing(const lsapgpu_ctx* ctx, double* total_ms, int64_t* launches,
                        double* full_sweep_ms, int64_t* full_sweeps, double* commit_ms,
                        int64_t* commit_launches) {
  if (!ctx) return LSAPGPU_ERR_INVALID;
  if (commit_ms) *commit_ms = ctx->commit_ms;
  if (commit_launches) *commit_launches = ctx->commit_launches;
  if (total_ms) *total_ms = ctx->scan_ms;
  if (launches) *launches = ctx->scan_launches;
  if (full_sweep_ms) *full_sweep_ms = ctx->full_ms;
  if (full_sweeps) *full_sweeps = ctx->full_launches;
  return LSAPGPU_OK;
}

int lsapgpu_evaluate_all(lsapgpu_ctx* ctx, const int32_t* sigma, double eps, double* agent_delta,
                         int32_t* agent_partner, double* job_delta, int32_t* job_partner) {
  if (!ctx || !ctx->n_matrix) return fail(ctx, LSAPGPU_ERR_STATE, "no matrix set");
  if (int rc = require_full_rows(ctx, "evaluate_all_parallel")) return rc;
  CK(cudaSetDevice(ctx->device));
  if (!(eps >= 0.0)) return fail(ctx, LSAPGPU_ERR_INVALID, "improvement_epsilon must be >= 0");
  const int32_t n = ctx->n_matrix;
  if (!is_perm(sigma, n)) return fail(ctx, LSAPGPU_ERR_INVALID, "invalid assignment: not a permutation");
  DevState& d = ctx->d;
  d.eps = eps;
  CK(cpy(ctx, d.sigma, sigma, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(launch_init_assignment(d, ctx->stream));
  ++ctx->launches;
  begin_pass_kernel<<<1, 1, 0, ctx->stream>>>(ctx->ctrl_dev, 1);
  ++ctx->launches;
  CK(cudaGetLastError());
  int rc = run_scan(ctx, 1);
  if (rc) return rc;
  CK(cpy(ctx, agent_delta, d.agent_delta, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cpy(ctx, agent_partner, d.agent_partner, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cpy(ctx, job_delta, d.job_delta, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cpy(ctx, job_partner, d.job_partner, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return LSAPGPU_OK;
}

int lsapgpu_check_conflicts(lsapgpu_ctx* ctx, int32_t n, const double* agent_delta,
                            const int32_t* agent_partner, const double* job_delta,
                            const int32_t* job_partner, const int32_t* sigma,
                            uint8_t* agent_accepted, uint8_t* job_accepted, uint8_t* reserved_mask,
                            uint8_t* conflicted_mask, int32_t* conflicted_jobs,
                            int32_t* n_conflicted_jobs) {
  if (!ctx) return LSAPGPU_ERR_INVALID;
  CK(cudaSetDevice(ctx->device));
  if (n < 1) return fail(ctx, LSAPGPU_ERR_INVALID, "delta tables do not match assignment size");
  if (n >= (1 << 30)) return fail(ctx, LSAPGPU_ERR_INVALID, "n >= 2^30 is not supported by this build");
  for (int32_t k = 0; k < n; ++k)
    if (agent_partner[k] >= n || job_partner[k] >= n || agent_partner[k] < -1 || job_partner[k] < -1)
      return fail(ctx, LSAPGPU_ERR_INVALID, "record partner out of range");
  if (!is_perm(sigma, n)) return fail(ctx, LSAPGPU_ERR_INVALID, "invalid assignment: not a permutation");
  if (ctx->n_vec != n) ctx->n_matrix = 0;
  int rc = ensure_vectors(ctx, n);
  if (rc) return rc;
  DevState d = ctx->d;
  if (!ctx->n_matrix) d.storage = kI32;  // the commit kernel template needs some storage type
  CK(cpy(ctx, d.sigma, sigma, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cpy(ctx, d.agent_delta, agent_delta, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cpy(ctx, d.agent_partner, agent_partner, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cpy(ctx, d.job_delta, job_delta, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cpy(ctx, d.job_partner, job_partner, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  begin_pass_kernel<<<1, 1, 0, ctx->stream>>>(ctx->ctrl_dev, 1);
  ++ctx->launches;
  CK(cudaGetLastError());
  CK(launch_edges_from_tables(d, ctx->stream));
  ++ctx->launches;
  CK(launch_commit(d, plan_commit(d), kCommitCheckOnly, 0, 0, ctx->stream));
  ++ctx->launches;
  rc = pull_ctrl(ctx);
  if (rc) return rc;
  const int32_t m = ctx->ctrl_host->edge_count[ctx->ctrl_host->parity];
  std::vector<Prop> slots(m);
  std::vector<int32_t> eu(m), ev(m);
  std::vector<uint8_t> est(m);
  if (m) {
    const int P = ctx->ctrl_host->parity;
    CK(cpy(ctx, slots.data(), d.edges[P], sizeof(Prop) * m, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cpy(ctx, eu.data(), d.eu, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cpy(ctx, ev.data(), d.ev, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cpy(ctx, est.data(), d.estate, m, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  std::memset(agent_accepted, 0, n);
  std::memset(job_accepted, 0, n);
  std::memset(reserved_mask, 0, n);
  std::memset(conflicted_mask, 0, n);
  std::vector<int32_t> cj;
  for (int32_t e = 0; e < m; ++e) {
    const int32_t s = slots[e].slot;
    if (est[e] == kEdgeAccepted) {
      (s < n ? agent_accepted[s] : job_accepted[s - n]) = 1;
      reserved_mask[eu[e]] = 1;
      reserved_mask[ev[e]] = 1;
    } else if (est[e] == kEdgeRejected) {
      conflicted_mask[eu[e]] = 1;  // the proposer (the job's holder on the job side)
      if (s >= n) cj.push_back(s - n);
    }
  }
  std::sort(cj.begin(), cj.end());
  for (size_t k = 0; k < cj.size(); ++k) conflicted_jobs[k] = cj[k];
  *n_conflicted_jobs = static_cast<int32_t>(cj.size());
  // restore the edge lists for the next user
  ctx->ctrl_host->edge_count[0] = ctx->ctrl_host->edge_count[1] = 0;
  return push_ctrl(ctx);
}

int lsapgpu_apply_parallel_switches(lsapgpu_ctx* ctx, int32_t* sigma, int32_t* tau, double* value,
                                    const double* agent_delta, const int32_t* agent_partner,
                                    const uint8_t* agent_active, const double* job_delta,
                                    const int32_t* job_partner, const uint8_t* job_active,
                                    const uint8_t* agent_accepted, const uint8_t* job_accepted,
                                    double eps, int32_t* applied_agent, int32_t* applied_new_job,
                                    int32_t* applied_old_job, int32_t* applied_displaced,
                                    double* applied_delta, int32_t* n_applied) {
  if (ctx && ctx->n_matrix && ctx->place_world > 1) return require_full_rows(ctx, "apply_parallel_switches");
  if (!ctx || !ctx->n_matrix) return fail(ctx, LSAPGPU_ERR_STATE, "no matrix set");
  CK(cudaSetDevice(ctx->device));
  if (!(eps >= 0.0)) return fail(ctx, LSAPGPU_ERR_INVALID, "improvement_epsilon must be >= 0");
  const int32_t n = ctx->n_matrix;
  if (!is_perm(sigma, n)) return fail(ctx, LSAPGPU_ERR_INVALID, "assignment does not match instance");
  for (int32_t k = 0; k < n; ++k)
    if (agent_partner[k] >= n || job_partner[k] >= n) return fail(ctx, LSAPGPU_ERR_INVALID, "record partner out of range");
  DevState& d = ctx->d;
  d.eps = eps;
  // active flag folded into the delta, exactly as the select guard reads it
  std::vector<double> ad(n), jd(n);
  for (int32_t k = 0; k < n; ++k) {
    ad[k] = agent_active[k] ? agent_delta[k] : 0.0;
    jd[k] = job_active[k] ? job_delta[k] : 0.0;
  }
  uint8_t* masks = nullptr;
  CK(cudaMalloc(&masks, 2 * static_cast<size_t>(n)));
  CK(cpy(ctx, masks, agent_accepted, n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cpy(ctx, masks + n, job_accepted, n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cpy(ctx, d.sigma, sigma, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cpy(ctx, d.tau, tau, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(launch_tau16_sync(d, ctx->stream));
  CK(cpy(ctx, d.agent_delta, ad.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cpy(ctx, d.agent_partner, agent_partner, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cpy(ctx, d.job_delta, jd.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cpy(ctx, d.job_partner, job_partner, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  begin_pass_kernel<<<1, 1, 0, ctx->stream>>>(ctx->ctrl_dev, 1);
  ++ctx->launches;
  CK(cudaGetLastError());
  CK(launch_edges_from_tables(d, ctx->stream));
  ++ctx->launches;
  CK(launch_accepted_from_masks(d, masks, masks + n, ctx->stream));
  ++ctx->launches;
  int rc = pull_ctrl(ctx);
  cudaFree(masks);
  if (rc) return rc;
  Ctrl& C = *ctx->ctrl_host;
  const int64_t cnt = C.log_count;
  std::vector<LogEntry> log(static_cast<size_t>(cnt));
  if (cnt) {
    CK(cpy(ctx, log.data(), d.log, sizeof(LogEntry) * cnt, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  const int err = C.error;
  C.error = 0;
  C.log_count = 0;
  C.edge_count[0] = C.edge_count[1] = 0;
  rc = push_ctrl(ctx);
  if (rc) return rc;
  if (err) return fail(ctx, LSAPGPU_ERR_INTERNAL, "internal: conflict check admitted overlapping exchanges");
  std::sort(log.begin(), log.end(), [](const LogEntry& a, const LogEntry& b) { return a.slot < b.slot; });
  // applied list in the reference's commit order, recovered from the frozen input
  std::vector<int32_t> s0(sigma, sigma + n), t0(tau, tau + n);
  double v = *value;
  int32_t k = 0;
  for (const auto& L : log) {
    int32_t agent, j_new;
    if (L.slot < n) {
      agent = L.slot;
      j_new = agent_partner[L.slot];
    } else {
      agent = job_partner[L.slot - n];
      j_new = L.slot - n;
    }
    const int32_t j_old = t0[agent], disp = s0[j_new];
    applied_agent[k] = agent;
    applied_new_job[k] = j_new;
    applied_old_job[k] = j_old;
    applied_displaced[k] = disp;
    applied_delta[k] = L.delta;
    sigma[j_new] = agent;
    sigma[j_old] = disp;
    tau[agent] = j_new;
    tau[disp] = j_old;
    v += L.delta;
    ++k;
  }
  *value = v;
  *n_applied = k;
  return LSAPGPU_OK;
}

size_t lsapgpu_dist_exchange_bytes(int32_t n, int32_t world) {
  return world < 1 || n < 1 ? 0 : dist_exchange_bytes(n, world);
}

int lsapgpu_solve(lsapgpu_ctx* ctx, const lsapgpu_params* params, int32_t* sigma_out,
                  int32_t* tau_out, lsapgpu_stats* stats, int64_t* trace_switch, double* trace_value,
                  int64_t trace_cap, int64_t* trace_len) {
  return lsapgpu_solve_dist(ctx, params, nullptr, sigma_out, tau_out, stats, trace_switch, trace_value,
                            trace_cap, trace_len);
}

int lsapgpu_solve_dist(lsapgpu_ctx* ctx, const lsapgpu_params* params, const lsapgpu_dist* dist,
                       int32_t* sigma_out, int32_t* tau_out, lsapgpu_stats* stats, int64_t* trace_switch,
                       double* trace_value, int64_t trace_cap, int64_t* trace_len) {
  if (!ctx) return LSAPGPU_ERR_INVALID;
  if (!ctx->n_matrix) return fail(ctx, LSAPGPU_ERR_STATE, "no matrix set");
  if (!params || !sigma_out) return fail(ctx, LSAPGPU_ERR_INVALID, "null argument");
  CK(cudaSetDevice(ctx->device));
  const auto t_start = std::chrono::steady_clock::now();
  const lsapgpu_params& P = *params;
  if (!(P.eps >= 0.0)) return fail(ctx, LSAPGPU_ERR_INVALID, "improvement_epsilon must be >= 0");
  if (P.reeval != 0 && P.reeval != 1) return fail(ctx, LSAPGPU_ERR_INVALID, "unknown reeval policy");
  const int32_t n = ctx->n_matrix;
  DevState& d = ctx->d;
  const bool multi = dist && dist->world > 1;
  if (dist && (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world))
    return fail(ctx, LSAPGPU_ERR_INVALID, "invalid rank / world");
  const bool p2p = multi && dist->peer_recv && dist->peer_flags;
  const bool dist_graph = p2p && params && params->use_graph;  // the peer transport loop runs as a graph
  if (multi && !p2p && (!dist->allgather || !dist->send_dev || !dist->recv_dev))
    return fail(ctx, LSAPGPU_ERR_INVALID, "multi-GPU solve needs an allgather callback and exchange buffers");
  if (p2p && dist->world > kMaxPeers) return fail(ctx, LSAPGPU_ERR_INVALID, "peer transport: at most 8 ranks");
  if (ctx->place_world > 1 && !(multi && dist->world == ctx->place_world && dist->rank == ctx->place_rank))
    return fail(ctx, LSAPGPU_ERR_STATE,
                "this context holds row block " + std::to_string(ctx->place_rank) + " of " +
                    std::to_string(ctx->place_world) + " of the matrix: solve it as that rank of that many");
  if (ctx->place_world > 1 && params->init_mode == LSAPGPU_INIT_GREEDY)
    return fail(ctx, LSAPGPU_ERR_STATE, "the greedy start needs every row of A (full replicas)");
  const size_t xbytes = multi ? dist_exchange_bytes(n, dist->world) : 0;
  PeerSet ps{};
  if (p2p) {
    for (int r = 0; r < dist->world; ++r) {
      if (!dist->peer_recv[r] || !dist->peer_flags[r])
        return fail(ctx, LSAPGPU_ERR_INVALID, "peer transport: missing peer buffer");
      ps.recv[r] = static_cast<unsigned char*>(dist->peer_recv[r]);
      ps.flags[r] = dist->peer_flags[r];
    }
    ps.world = dist->world;
    ps.rank = dist->rank;
    ps.bytes_per_rank = xbytes;
    // the round epoch continues from this rank's own flag (its last push):
    // ranks that finished the previous solve on these buffers agree on it.
    // (Not the highest flag: a faster peer may already have pushed the first
    // round of this solve.)  A solve that ended on a transport error leaves
    // the epochs out of step, so the buffers are refused until the caller
    // builds a fresh exchange (zeroed flags) on every rank.
    if (ctx->peer_poisoned.count(dist->peer_flags[dist->rank]))
      return fail(ctx, LSAPGPU_ERR_STATE,
                  "peer exchange: a previous solve on these buffers failed; create a new exchange on every rank");
    uint64_t e = 0;
    CK(cudaMemcpyAsync(&e, dist->peer_flags[dist->rank] + dist->rank, sizeof(e), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpyAsync(&ctx->ctrl_dev->p2p_epoch, &e, sizeof(e), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  // one distributed step: this rank's items -> scan -> pack -> allgather -> merge
  auto dist_round = [&](int full) -> int {
    CK(launch_dist_own_items(d, full, dist->rank, dist->world, ctx->stream));
    ctx->launches += 2;
    DevState ds = d;
    ds.use_own = 1;
    ds.emit_edges = 0;
    if (ctx->timing) CK(cudaEventRecord(ctx->ev0, ctx->stream));
    CK(launch_scan(ds, ctx->scan_plan, 0, ctx->stream));
    ctx->launches += ctx->scan_plan.launches();
    if (ctx->timing) {  // this rank's scan of its share (host-stepped solves with timing on)
      CK(cudaEventRecord(ctx->ev1, ctx->stream));
      CK(cudaEventSynchronize(ctx->ev1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
      ctx->scan_ms += ms;
      ++ctx->scan_launches;
      if (full) {
        ctx->full_ms += ms;
        ++ctx->full_launches;
      }
    }
    if (p2p) {  // pack + allgather in one kernel over peer memory, then wait + merge
      CK(launch_dist_push(d, ps, ctx->stream));
      ctx->launches += 3;
      return LSAPGPU_OK;
    }
    CK(launch_dist_pack(d, dist->send_dev, ctx->stream));
    ++ctx->launches;
    if (dist->allgather(dist->user, dist->send_dev, dist->recv_dev, xbytes, ctx->stream) != 0)
      return fail(ctx, LSAPGPU_ERR_CUDA, "allgather callback failed");
    CK(launch_dist_merge(d, dist->recv_dev, dist->world, xbytes, ctx->stream));
    ++ctx->launches;
    return LSAPGPU_OK;
  };

  // initial permutation: random_perm(seed) is sequential by nature and a pure
  // function of (n, seed), so the last one is kept in pinned memory
  if (P.init_mode != LSAPGPU_INIT_RANDOM && P.init_mode != LSAPGPU_INIT_GREEDY)
    return fail(ctx, LSAPGPU_ERR_INVALID, "unknown init mode");
  if (P.init_sigma) {
    if (!is_perm(P.init_sigma, n)) return fail(ctx, LSAPGPU_ERR_INVALID, "invalid assignment: not a permutation");
    CK(cpy(ctx, d.sigma, P.init_sigma, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  } else if (P.init_mode == LSAPGPU_INIT_GREEDY) {
    int grc = run_greedy(ctx);
    if (grc) return grc;
  } else {
    if (ctx->perm_n != n || ctx->perm_seed != P.seed) {
      CK(cudaStreamSynchronize(ctx->stream));  // a previous upload may still read the buffer
      if (ctx->perm_cap < n) {
        if (ctx->perm_pin) cudaFreeHost(ctx->perm_pin);
        ctx->perm_pin = nullptr;
        ctx->perm_cap = 0;
        CK(cudaMallocHost(&ctx->perm_pin, sizeof(int32_t) * n));
        ctx->perm_cap = n;
      }
      lsapgpu_random_perm(n, P.seed, ctx->perm_pin);
      ctx->perm_n = n;
      ctx->perm_seed = P.seed;
    }
    CK(cpy(ctx, d.sigma, ctx->perm_pin, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  }
  CK(launch_init_assignment(d, ctx->stream));
  ++ctx->launches;
  // initial objective and the counter base: enqueued now, read at the first
  // sync the solve needs anyway (the device starts the first sweep at once)
  int rc = enqueue_objective(ctx);
  if (rc) return rc;
  if (!ctx->ctrl_base) CK(cudaMallocHost(&ctx->ctrl_base, sizeof(Ctrl)));
  CK(cpy(ctx, ctx->ctrl_base, ctx->ctrl_dev, sizeof(Ctrl), cudaMemcpyDeviceToHost, ctx->stream));
  double value = 0.0;
  const int64_t host_orders0 = ctx->host_log_orders;
  Ctrl base;
  std::memset(&base, 0, sizeof(base));
  bool inited = false;
  TraceSink trace{trace_switch, trace_value, trace_cap};
  auto ensure_init = [&]() -> int {
    if (inited) return LSAPGPU_OK;
    CK(cudaStreamSynchronize(ctx->stream));
    value = objective_sum(ctx);
    base = *ctx->ctrl_base;  // counters are cumulative per context
    trace.push(0, value);
    inited = true;
    return LSAPGPU_OK;
  };
  lsapgpu_stats S;
  std::memset(&S, 0, sizeof(S));
  S.storage = d.storage;

  auto elapsed_ns = [&]() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t_start)
        .count();
  };
  // LSAPGPU_HOST_TIMING=1: host-side phase marks of this solve on stderr
  static const bool host_timing = std::getenv("LSAPGPU_HOST_TIMING") != nullptr;
  std::vector<std::pair<const char*, int64_t>> hmarks;
  auto hmark = [&](const char* what) {
    if (host_timing) hmarks.emplace_back(what, elapsed_ns());
  };
  hmark("init+objective");
  // multi-rank: only the budget 0 is decided here (identically on every rank);
  // any other expiry is agreed at a record exchange (dist.cu)
  bool expired = P.deadline_ns >= 0 && (multi ? P.deadline_ns == 0 : elapsed_ns() >= P.deadline_ns);

  d.eps = P.eps;
  d.dist_vote = multi ? 1 : 0;
  d.policy = P.reeval;
  if (!expired) {
    set_deadline_kernel<<<1, 1, 0, ctx->stream>>>(
        ctx->ctrl_dev, P.deadline_ns < 0 ? -1 : std::max<int64_t>(0, P.deadline_ns - elapsed_ns()));
    ++ctx->launches;
    CK(cudaGetLastError());
    if (P.use_graph && !multi &&
        (!ctx->exec || std::memcmp(&ctx->graph_state, &d, sizeof(DevState)) != 0 ||
         !(ctx->graph_scan == ctx->scan_plan) || !(ctx->graph_commit == ctx->commit_plan))) {
      rc = build_graph(ctx);
      if (rc) return rc;
    }
    if (dist_graph && (!ctx->dist_exec || std::memcmp(&ctx->dist_state, &d, sizeof(DevState)) != 0 ||
                       std::memcmp(&ctx->dist_ps, &ps, sizeof(PeerSet)) != 0)) {
      rc = build_dist_graph(ctx, ps);
      if (rc) return rc;
    }
  }
  ctx->scan_ms = ctx->full_ms = ctx->commit_ms = 0.0;
  ctx->scan_launches = ctx->full_launches = ctx->commit_launches = 0;
  if (!ctx->log_pin) CK(cudaMallocHost(&ctx->log_pin, sizeof(LogEntry) * lsapgpu_ctx::kLogPin));
  // Replay order: see the log read-back below
  const bool need_order = (trace_switch && trace_value) || d.storage == kF32 || d.storage == kF64;
  static const bool host_order_env = std::getenv("LSAPGPU_HOST_LOG_ORDER") && std::atoi(std::getenv("LSAPGPU_HOST_LOG_ORDER"));
  const bool dev_order = need_order && !host_order_env && order_log_fits(n) && d.log_sorted != nullptr;
  std::vector<LogEntry>& log = ctx->log_host;
  std::vector<LogEntry>& sorted = ctx->log_sorted;
  int64_t switches = 0;
  int64_t launches = 0;
  int64_t graph_launches = 0;
  bool prefetched = false;  // ctrl + log prefix already read back with the graph's sync
  int64_t pin_len = 0;      // entries of that prefix

  while (!expired) {
    double f_start = value;  // (first pass: set once the initial objective is read)
    const bool first_pass = !inited;
    ++S.outer_iterations;
    begin_pass_kernel<<<1, 1, 0, ctx->stream>>>(ctx->ctrl_dev, 1);
    ++ctx->launches;
    CK(cudaGetLastError());
    if (multi) {
      rc = dist_round(1);
    } else {
      rc = run_scan(ctx, 1);
    }
    if (rc) return rc;
    ++launches;
    S.pair_items += n;
    S.agent_scans += n;
    S.job_scans += n;
    for (;;) {  // inner loop; repeats only to drain a full delta log
      bool graph_pass = false;
      if (multi && !dist_graph) {
        for (;;) {
          CK(launch_commit(d, ctx->commit_plan, kCommitSolve, 0, 0, ctx->stream));
          ctx->launches += ctx->commit_plan.launches();  // conflict check (+ apply)
          rc = pull_ctrl(ctx);
          if (rc) return rc;
          const Ctrl& C = *ctx->ctrl_host;
          if (C.inner_done || C.expired || C.drain || C.error) break;
          rc = dist_round(0);
          if (rc) return rc;
          ++launches;
        }
      } else if (P.use_graph) {
        CK(cudaGraphLaunch(dist_graph ? ctx->dist_exec : ctx->exec, ctx->stream));
        ++graph_launches;
        graph_pass = true;
        if (dev_order) {  // the pass's log in batch order, before the read-back below
          CK(launch_order_log(d, ctx->stream));
          ++ctx->launches;
        }
        // control block and the first kLogPin log entries with one sync
        CK(cpy(ctx, ctx->ctrl_host, ctx->ctrl_dev, sizeof(Ctrl), cudaMemcpyDeviceToHost, ctx->stream));
        // log prefix sized from what this pass produced in the previous solve
        // (bench steps repeat a solve): the rest, if any, follows with a sync
        const int hp = std::min<int>(static_cast<int>(S.outer_iterations) - 1, 3);
        pin_len = std::min<int64_t>(std::min<int64_t>(lsapgpu_ctx::kLogPin, d.log_cap),
                                    ctx->log_hint[hp] + ctx->log_hint[hp] / 4 + 1024);
        CK(cpy(ctx, ctx->log_pin, dev_order ? d.log_sorted : d.log, sizeof(LogEntry) * pin_len,
               cudaMemcpyDeviceToHost, ctx->stream));
        hmark("graph launched");
        CK(cudaStreamSynchronize(ctx->stream));
        hmark("graph done");
        prefetched = true;
      } else {
        for (;;) {
          if (ctx->timing) CK(cudaEventRecord(ctx->ev0, ctx->stream));
          CK(launch_commit(d, ctx->commit_plan, kCommitSolve, 0, 0, ctx->stream));
          if (ctx->timing) {
            CK(cudaEventRecord(ctx->ev1, ctx->stream));
            CK(cudaEventSynchronize(ctx->ev1));
            float cms = 0.f;
            CK(cudaEventElapsedTime(&cms, ctx->ev0, ctx->ev1));
            ctx->commit_ms += cms;
            ++ctx->commit_launches;
          }
          ctx->launches += ctx->commit_plan.launches();  // conflict check (+ apply)
          rc = run_scan(ctx, 0);
          if (rc) return rc;
          ++launches;
          rc = pull_ctrl(ctx);
          if (rc) return rc;
          const Ctrl& C = *ctx->ctrl_host;
          if (C.inner_done || C.expired || C.drain || C.error) break;
        }
      }
      if (dev_order && !graph_pass) {  // host-stepped passes: order the log now
        CK(launch_order_log(d, ctx->stream));
        ++ctx->launches;
        if ((rc = pull_ctrl(ctx))) return rc;
      }
      if ((rc = ensure_init())) return rc;
      if (first_pass) f_start = value;
      Ctrl& C = *ctx->ctrl_host;
      if (C.error) {
        const int code = C.error;
        C.error = 0;
        push_ctrl(ctx);
        if (code == 2) {
          if (p2p) ctx->peer_poisoned.insert(dist->peer_flags[dist->rank]);
          return fail(ctx, LSAPGPU_ERR_CUDA, "peer exchange: a rank's records did not arrive (timeout)");
        }
        return fail(ctx, LSAPGPU_ERR_INTERNAL, "internal: conflict check admitted overlapping exchanges");
      }
      const int64_t cnt = C.log_count;
      if (!C.drain) ctx->log_hint[std::min<int>(static_cast<int>(S.outer_iterations) - 1, 3)] = cnt;
      // Replay in the reference's batch order (iteration, then ascending slot:
      // agents then jobs, parallel.cpp:306-310), normally ordered on the device
      // (log_order.cu); the host orders the raw log only if the device could
      // not.  Integer deltas sum exactly in any order, so without a trace the
      // order only matters for float storage.
      const bool sorted_ok = dev_order && C.order_bad == 0 && static_cast<int64_t>(C.order_total) == cnt;
      const LogEntry* src_dev = sorted_ok ? d.log_sorted : d.log;
      // (the pinned prefix holds the device-ordered log whenever dev_order)
      const int64_t have = prefetched && (sorted_ok || !dev_order) ? std::min<int64_t>(cnt, pin_len) : 0;
      const LogEntry* entries = ctx->log_pin;
      if (cnt > have) {
        log.resize(static_cast<size_t>(cnt));
        if (have) std::memcpy(log.data(), ctx->log_pin, sizeof(LogEntry) * have);
        CK(cpy(ctx, log.data() + have, src_dev + have, sizeof(LogEntry) * (cnt - have), cudaMemcpyDeviceToHost,
               ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        entries = log.data();
      }
      prefetched = false;
      hmark("log read");
      if (need_order) {
        if (!sorted_ok) {
          order_log(entries, static_cast<size_t>(cnt), sorted, 2 * n);
          entries = sorted.data();
          ++ctx->host_log_orders;
        }
        hmark("log ordered");
        if ((d.storage == kI16 || d.storage == kI32) && n < (1 << 22)) {
          // integer storage: every delta and partial sum is an integer below
          // 2^53 (n * 2^30 at most), so an int64 running sum converts to the
          // very doubles the sequential fp64 sum produces, without the fp64
          // add's latency on the critical path
          int64_t iv = static_cast<int64_t>(value);
          for (int64_t k = 0; k < cnt; ++k) {
            iv += static_cast<int64_t>(entries[k].delta);
            ++switches;
            trace.push(switches, static_cast<double>(iv));
          }
          value = static_cast<double>(iv);
        } else {
          for (int64_t k = 0; k < cnt; ++k) {
            value += entries[k].delta;
            ++switches;
            trace.push(switches, value);
          }
        }
      } else {
        // integer storage, no trace: every delta and partial sum is an exact
        // integer, so independent partial sums give the sequential result
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        int64_t k = 0;
        for (; k + 4 <= cnt; k += 4)
          for (int q = 0; q < 4; ++q) acc[q] += entries[k + q].delta;
        for (; k < cnt; ++k) acc[0] += entries[k].delta;
        value += (acc[0] + acc[1]) + (acc[2] + acc[3]);
        switches += cnt;
        trace.len = std::min<int64_t>(kTraceCap, trace.len + cnt);  // what push() would count
      }
      hmark("log replayed");
      const bool drained = C.drain;
      if (C.expired) expired = true;
      if (!drained || expired) break;
      // the log filled up mid-pass: empty it and continue the inner loop (a
      // new pass's begin_pass resets it otherwise)
      begin_pass_kernel<<<1, 1, 0, ctx->stream>>>(ctx->ctrl_dev, 0);
      ++ctx->launches;  // log_count = 0, drain = 0
      CK(cudaGetLastError());
    }
    if (expired) break;
    if (!multi && P.deadline_ns >= 0 && elapsed_ns() >= P.deadline_ns) {
      expired = true;
      break;
    }
    if (trace.len >= kTraceCap) trace.push(switches, value, true);
    if (value == f_start) break;
  }

  if ((rc = ensure_init())) return rc;  // (a solve cut before its first pass)
  // final counters, sigma / tau and the ordered objective with ONE sync (in
  // graph mode the control block came with the last graph's read-back and no
  // kernel since changed the counters)
  const bool ctrl_current = P.use_graph && (!multi || dist_graph) && S.outer_iterations > 0 && !expired;
  if (!ctrl_current) CK(cpy(ctx, ctx->ctrl_host, ctx->ctrl_dev, sizeof(Ctrl), cudaMemcpyDeviceToHost, ctx->stream));
  rc = enqueue_objective(ctx, true);  // snapshot_assignment (solver_state.hpp:141-148) + sigma / tau
  if (rc) return rc;
  hmark("final enqueued");
  CK(cudaStreamSynchronize(ctx->stream));
  const double final_value = objective_sum(ctx);
  {
    const int32_t* packed = reinterpret_cast<const int32_t*>(ctx->obj_pin + n);
    std::memcpy(sigma_out, packed, sizeof(int32_t) * n);
    if (tau_out) std::memcpy(tau_out, packed + n, sizeof(int32_t) * n);
  }
  hmark("final done");
  if (host_timing) {
    std::string line = "lsapgpu host timing (us):";
    for (const auto& m : hmarks) line += std::string(" ") + m.first + "=" + std::to_string(m.second / 1000);
    std::fprintf(stderr, "%s\n", line.c_str());
  }
  const Ctrl& C = *ctx->ctrl_host;
  S.inner_iterations = C.inner_iterations - base.inner_iterations;
  S.pair_items += C.pair_items - base.pair_items;
  S.agent_scans += C.agent_scans - base.agent_scans;
  S.job_scans += C.job_scans - base.job_scans;
  S.lfmm_rounds = C.lfmm_rounds - base.lfmm_rounds;
  S.scan_filter = ctx->scan_plan.filter;
  S.filter_kept = C.filter_kept - base.filter_kept;
  S.filter_overflows = C.filter_overflows - base.filter_overflows;
  S.host_log_orders = ctx->host_log_orders - host_orders0;
  if (C.fchk_mismatch) {  // LSAPGPU_FILTER_CHECK diagnostics
    char msg[256];
    std::snprintf(msg, sizeof msg,
                  "filter check: %d mismatching records; first %s %d (queue %d): want (%.17g, %d) got (%.17g, %d); "
                  "wanted position %d aux_ok %d U %d t0 %d tmax %d",
                  C.fchk_mismatch, C.fchk_side ? "job" : "agent", C.fchk_item, C.fchk_cnt, C.fchk_want_d,
                  C.fchk_want_k, C.fchk_got_d, C.fchk_got_k, C.fchk_p, C.fchk_aux_ok, C.fchk_u, C.fchk_t0,
                  C.fchk_tmax);
    Ctrl& Cm = *ctx->ctrl_host;
    Cm.fchk_mismatch = 0;
    push_ctrl(ctx);
    return fail(ctx, LSAPGPU_ERR_INTERNAL, msg);
  }
  S.switches_applied = switches;
  const bool graphed = P.use_graph && (!multi || dist_graph);
  S.scan_launches = graphed ? S.outer_iterations + S.inner_iterations + graph_launches : launches;
  // every body pass of the graph is a commit (conflict check + apply) and a
  // scan launch; the last pass per graph launch finds no active record and
  // exits early
  if (graphed) {
    const int per_pass = (ctx->commit_plan.launches()) +
                         (dist_graph ? 2 /* own items */ + 3 /* push, wait, merge */ : 0) +
                         ctx->scan_plan.launches();
    ctx->launches += per_pass * (S.inner_iterations + graph_launches);
  }
  S.bytes_scanned = S.pair_items * 2 * static_cast<int64_t>(n) * static_cast<int64_t>(esize(d.storage));
  S.terminated_by = expired ? 1 : 0;

  S.value = final_value;
  S.elapsed_ms = static_cast<double>(elapsed_ns()) / 1e6;
  if (stats) *stats = S;
  if (trace_len) *trace_len = trace.len;
  return LSAPGPU_OK;
}

}  // extern "C"

// ---- auction baseline: lsap::auction_solve (auction.cpp:110-153) ----------

int lsapgpu_auction_solve(lsapgpu_ctx* ctx, const lsapgpu_auction_params* params, int32_t* sigma_out,
                          int32_t* tau_out, lsapgpu_auction_stats* stats, double* prices_out,
                          double* round_prices, int64_t round_cap) {
  if (!ctx) return LSAPGPU_ERR_INVALID;
  if (!ctx->n_matrix) return fail(ctx, LSAPGPU_ERR_STATE, "no matrix set");
  if (!params || !sigma_out) return fail(ctx, LSAPGPU_ERR_INVALID, "null argument");
  if (int rc = require_full_rows(ctx, "auction_solve")) return rc;
  const lsapgpu_auction_params& P = *params;
  // AuctionConfig::validate (baselines.hpp:22-25)
  if (P.has_epsilon && !(P.epsilon > 0.0)) return fail(ctx, LSAPGPU_ERR_INVALID, "auction: epsilon must be > 0");
  if (!(P.scale_factor > 1.0)) return fail(ctx, LSAPGPU_ERR_INVALID, "auction: scale_factor must be > 1");
  if (round_cap < 0 || (round_cap > 0 && !round_prices))
    return fail(ctx, LSAPGPU_ERR_INVALID, "round_prices needs round_cap entries");
  CK(cudaSetDevice(ctx->device));
  const auto t_start = std::chrono::steady_clock::now();
  auto elapsed_ns = [&]() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t_start)
        .count();
  };
  const int32_t n = ctx->n_matrix;
  DevState& d = ctx->d;
  AuctionDev& a = ctx->au;
  if (!ctx->au_host) CK(cudaMallocHost(&ctx->au_host, sizeof(AuctionCtrl)));
  if (ctx->au_n != n) {
    const size_t N = static_cast<size_t>(d.ld), NC = N * 16;  // segments for up to 16 cluster CTAs
    CK(valloc(ctx, &a.prices, N, false));
    CK(valloc(ctx, &a.owner, N, false));
    CK(valloc(ctx, &a.assigned, N, false));
    CK(valloc(ctx, &a.slot, 2 * N, false));
    CK(valloc(ctx, &a.rec_i, NC, false));
    CK(valloc(ctx, &a.rec_j, NC, false));
    CK(valloc(ctx, &a.rec_bid, NC, false));
    CK(valloc(ctx, &a.wl[0], NC, false));
    CK(valloc(ctx, &a.wl[1], NC, false));
    CK(valloc(ctx, &a.ctrl, 1, false));
    ctx->au_n = n;
  }
  a.local_prices = n <= auction_local_price_cap() ? 1 : 0;
  if (const char* e = std::getenv("LSAPGPU_AUCTION_LOCAL_PRICES")) a.local_prices = a.local_prices && std::atoi(e);
  // rows of the next round's bidders are L2-prefetched when A does not stay
  // L2-resident by itself (measured: -3 % at C3's 200 MB, +2 % at C2's 50 MB)
  a.row_prefetch = static_cast<size_t>(n) * static_cast<size_t>(d.ld) * esize(d.storage) > (64u << 20) ? 1 : 0;
  if (const char* e = std::getenv("LSAPGPU_AUCTION_ROW_PF")) a.row_prefetch = std::atoi(e);
  AuctionCtrl& H = *ctx->au_host;

  // benefit range (std::minmax_element, auction.cpp:116-117), once per matrix
  if (!ctx->range_ok) {
    std::memset(&H, 0, sizeof(H));
    H.lo_key = ~0ull;
    CK(cpy(ctx, a.ctrl, &H, sizeof(H), cudaMemcpyHostToDevice, ctx->stream));
    CK(launch_minmax(d, a.ctrl, ctx->stream));
    ++ctx->launches;
    CK(cpy(ctx, &H, a.ctrl, sizeof(H), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->lo = auction_key_value(H.lo_key);
    ctx->hi = auction_key_value(H.hi_key);
    ctx->range_ok = true;
  }
  const double range = ctx->hi - ctx->lo;
  const double eps_target = P.has_epsilon ? P.epsilon : (range > 0.0 ? range / (2.0 * n) : 1.0);
  // the epsilon schedule (auction.cpp:125-135)
  std::vector<double> eps_list;
  if (P.scaling) {
    double eps = std::max(eps_target, range > 0.0 ? range / 2.0 : eps_target);
    while (true) {
      eps_list.push_back(eps);
      if (eps <= eps_target) break;
      eps = std::max(eps_target, eps / P.scale_factor);
    }
  } else {
    eps_list.push_back(eps_target);
  }
  if (ctx->eps_cap < eps_list.size()) {
    if (ctx->eps_dev) cudaFree(ctx->eps_dev);
    ctx->eps_dev = nullptr;
    ctx->eps_cap = 0;
    CK(cudaMalloc(&ctx->eps_dev, sizeof(double) * eps_list.size()));
    ctx->eps_cap = eps_list.size();
  }
  CK(cpy(ctx, ctx->eps_dev, eps_list.data(), sizeof(double) * eps_list.size(), cudaMemcpyHostToDevice,
         ctx->stream));
  a.eps_list = ctx->eps_dev;
  a.n_eps = static_cast<int32_t>(eps_list.size());
  double* rp_dev = nullptr;
  if (round_cap > 0) CK(cudaMallocAsync(&rp_dev, sizeof(double) * round_cap * n, ctx->stream));
  a.round_prices = rp_dev;
  a.round_cap = round_cap;

  const size_t N = static_cast<size_t>(d.ld);
  CK(cudaMemsetAsync(a.prices, 0, sizeof(double) * N, ctx->stream));
  CK(cudaMemsetAsync(a.slot, 0, sizeof(unsigned long long) * 2 * N, ctx->stream));
  const unsigned long long lo_key = H.lo_key, hi_key = H.hi_key;
  std::memset(&H, 0, sizeof(H));
  H.lo_key = lo_key;
  H.hi_key = hi_key;
  CK(cpy(ctx, a.ctrl, &H, sizeof(H), cudaMemcpyHostToDevice, ctx->stream));
  const int64_t remaining = P.deadline_ns < 0 ? -1 : std::max<int64_t>(0, P.deadline_ns - elapsed_ns());
  CK(launch_auction(d, a, remaining, ctx->stream));
  ++ctx->launches;
  // make_assignment (core.cpp:36-50): tau from sigma, ordered objective
  CK(launch_init_assignment(d, ctx->stream));
  ++ctx->launches;
  int rc = enqueue_objective(ctx);
  if (rc) return rc;
  CK(cpy(ctx, &H, a.ctrl, sizeof(H), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cpy(ctx, sigma_out, d.sigma, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, ctx->stream));
  if (tau_out) CK(cpy(ctx, tau_out, d.tau, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, ctx->stream));
  if (prices_out) CK(cpy(ctx, prices_out, a.prices, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  if (rp_dev) {
    CK(cpy(ctx, round_prices, rp_dev, sizeof(double) * round_cap * n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaFreeAsync(rp_dev, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  const double value = objective_sum(ctx);
  const double ms = static_cast<double>(elapsed_ns()) / 1e6;
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->outer_iterations = H.rounds;
    stats->switches_applied = H.switches;
    stats->terminated_by = H.finished ? 0 : 1;
    stats->completed_greedily = H.greedy;
    stats->value = value;
    stats->elapsed_ms = ms;
    stats->bids = H.bids;
    stats->phases = H.phases;
    stats->epsilon = eps_target;
    stats->bytes_scanned = H.bids * static_cast<int64_t>(n) * static_cast<int64_t>(esize(d.storage) + 8);
    stats->storage = d.storage;
  }
  return LSAPGPU_OK;
}

int lsapgpu_greedy_assignment(lsapgpu_ctx* ctx, int32_t* sigma_out, int64_t* rounds) {
  if (!ctx) return LSAPGPU_ERR_INVALID;
  if (!ctx->n_matrix) return fail(ctx, LSAPGPU_ERR_STATE, "no matrix set");
  if (!sigma_out) return fail(ctx, LSAPGPU_ERR_INVALID, "null argument");
  if (int rc0 = require_full_rows(ctx, "greedy_assignment")) return rc0;
  CK(cudaSetDevice(ctx->device));
  int rc = run_greedy(ctx);
  if (rc) return rc;
  GreedyCtrl gc;
  CK(cpy(ctx, sigma_out, ctx->d.sigma, sizeof(int32_t) * ctx->n_matrix, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cpy(ctx, &gc, ctx->gr.ctrl, sizeof(gc), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (rounds) *rounds = gc.rounds;
  return LSAPGPU_OK;
}

size_t lsapgpu_dist_p2p_bytes(int32_t n, int32_t world) {
  return 2 * static_cast<size_t>(world) * dist_exchange_bytes(n, world);  // double-buffered by epoch parity
}

int lsapgpu_dev_alloc(int device, size_t bytes, void** dev_ptr) {
  if (!dev_ptr) return LSAPGPU_ERR_INVALID;
  if (cudaSetDevice(device) != cudaSuccess || cudaMalloc(dev_ptr, bytes) != cudaSuccess ||
      cudaMemset(*dev_ptr, 0, bytes) != cudaSuccess)
    return LSAPGPU_ERR_CUDA;
  return LSAPGPU_OK;
}

int lsapgpu_dev_free(int device, void* dev_ptr) {
  if (cudaSetDevice(device) != cudaSuccess || cudaFree(dev_ptr) != cudaSuccess) return LSAPGPU_ERR_CUDA;
  return LSAPGPU_OK;
}

int lsapgpu_ipc_handle(const void* dev_ptr, void* handle64) {
  if (!dev_ptr || !handle64) return LSAPGPU_ERR_INVALID;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)) != cudaSuccess) return LSAPGPU_ERR_CUDA;
  static_assert(sizeof(h) == 64, "CUDA IPC handle size");
  std::memcpy(handle64, &h, sizeof(h));
  return LSAPGPU_OK;
}

int lsapgpu_ipc_open(const void* handle64, void** dev_ptr) {
  if (!handle64 || !dev_ptr) return LSAPGPU_ERR_INVALID;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  return cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? LSAPGPU_OK
                                                                                         : LSAPGPU_ERR_CUDA;
}

int lsapgpu_ipc_close(void* dev_ptr) {
  return cudaIpcCloseMemHandle(dev_ptr) == cudaSuccess ? LSAPGPU_OK : LSAPGPU_ERR_CUDA;
}
