// scan.cu -- scan plan and dispatch for the fused pair-scan kernel
// (scan_kernel.cuh; instantiated per storage type in scan_<type>.cu).
#include <algorithm>
#include <cstdlib>

#include "state.h"

namespace lsapgpu {

constexpr int kPacked32 = 0, kPacked64 = 1, kFloat = 2;
constexpr size_t kStaticSmem = 14 * 1024;  // ebuf + item metadata + counters (+ slack)

template <class E, int KM>
cudaError_t launch_scan_typed(const DevState& d, const ScanPlan& p, int full, cudaStream_t st);
template <class E, int KM>
cudaError_t launch_scan_res_typed(const DevState& d, const ScanPlan& p, int full, cudaStream_t st);
template <class E>
cudaError_t launch_scan_filter_typed(const DevState& d, const ScanPlan& p, int full, cudaStream_t st);

// Quantized-filter kernel geometry (scan_filter.cuh): row buffers of the
// quantized A rows, a ring of QT chunk slots, two candidate queues.
constexpr int32_t kFilterChunk = 4096;
constexpr int kFilterQueueMax = 1024;
size_t filter_smem(int64_t ld, int qbytes, int rb, int ns, int qcap, int32_t chunk = kFilterChunk) {
  const size_t row = (static_cast<size_t>(ld) * qbytes + 127) / 128 * 128;
  const size_t slot = static_cast<size_t>(chunk) * qbytes;
  return rb * row + ns * slot + 2 * static_cast<size_t>(qcap) * 8 + (rb + 2 * 8 + 4) * 8;
}

// Resident-state kernel geometry (scan_resident.cuh): 15 consumer warps + 1
// producer, tau16 + acur resident, double-buffered (A row, AT row) stages.
constexpr int kResWarps = 23;  // reduction scratch sized for the widest resident CTA
constexpr int kMaxBufs = 4;
size_t res_smem_bytes(int64_t ld, size_t es, int M, int bufs) {
  const size_t row = static_cast<size_t>(ld) * es;
  const size_t tau = (static_cast<size_t>(ld) * 2 + 127) / 128 * 128;
  const size_t acur = (row + 127) / 128 * 128;
  return tau + acur + static_cast<size_t>(bufs) * 2 * M * row + 4 * kMaxBufs * 8 +
         static_cast<size_t>(bufs) * kResWarps * 2 * M * 16;
}

namespace {
size_t elem_size(int storage) {
  switch (storage) {
    case kI16: return 2;
    case kI32: return 4;
    case kF32: return 4;
    default: return 8;
  }
}

}  // namespace

ScanPlan plan_scan(const DevState& d, int num_sms) {
  ScanPlan p;
  const size_t es = elem_size(d.storage);
  // dynamic smem per CTA we plan against; LSAPGPU_SCAN_BUDGET (bytes) and
  // LSAPGPU_SCAN_M override the plan so tests can reach every code path
  // (multi-pass chunking, single buffering, item batching) at small n.
  size_t budget = 200 * 1024;
  if (const char* b = std::getenv("LSAPGPU_SCAN_BUDGET")) budget = std::strtoull(b, nullptr, 10);
  int force_m = 0;
  if (const char* m = std::getenv("LSAPGPU_SCAN_M")) force_m = std::atoi(m);
  const size_t row = static_cast<size_t>(d.ld) * es;
  const size_t reserve = 256 + 4 * 16 * 8 * 16;  // barriers + reduction scratch (B x NW x 2M tracks)
  p.threads = 512;
  int force_bufs = 0;
  if (const char* bb = std::getenv("LSAPGPU_SCAN_BUFS")) force_bufs = std::atoi(bb);
  // Two co-resident 256-thread CTAs per SM, single-buffered, interleave their
  // staging and compute better than one double-buffered CTA (measured on
  // B200, n=10k: int16 3.9 vs 3.4 TB/s full sweep, fp32 3.7 vs 3.1).  Batch
  // as many items per stage as still allows two CTAs per SM.
  const size_t two_cta = (227 * 1024) / 2 - kStaticSmem - 1024 - reserve;
  if (row <= budget) {
    p.passes = 1;
    p.chunk = d.ld;
    p.bufs = 1;
    p.m = 0;
    for (int m : {4, 2, 1})
      if (static_cast<size_t>(m) * row <= two_cta) {
        p.m = m;
        break;
      }
    if (p.m == 0) {  // one row per CTA does not fit twice: one 512-thread CTA per SM
      p.m = 1;
      p.threads = 512;
    } else {
      p.threads = 256;
    }
    if (force_m == 1 || force_m == 2 || force_m == 4) p.m = force_m;
    if (force_bufs >= 1 && force_bufs <= 4 && static_cast<size_t>(force_bufs) * p.m * row <= budget)
      p.bufs = force_bufs;
    if (const char* t = std::getenv("LSAPGPU_SCAN_NT")) p.threads = std::atoi(t) == 256 ? 256 : 512;
  } else {  // row longer than the budget: single-buffered chunks (every pass rescans all positions)
    p.m = 1;
    p.bufs = 1;
    const size_t per_buf = budget;
    p.passes = static_cast<int>((row + per_buf - 1) / per_buf);
    int64_t ch = (d.ld + p.passes - 1) / p.passes;
    ch = (ch + 63) / 64 * 64;
    p.chunk = ch;
  }
  // streaming kernel, single-buffered rows: L2-prefetch the next stage's rows
  // (LSAPGPU_SCAN_L2PF=0 disables)
  p.l2_prefetch = p.bufs == 1 ? 1 : 0;
  if (const char* pf = std::getenv("LSAPGPU_SCAN_L2PF")) p.l2_prefetch = p.bufs == 1 ? std::atoi(pf) : 0;
  p.smem = static_cast<size_t>(p.bufs) * p.m * p.chunk * es + reserve;
  int per_sm = static_cast<int>((227 * 1024) / (p.smem + kStaticSmem + 1024));
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 512 / p.threads) per_sm = 512 / p.threads;  // register budget: 512 threads per SM
  p.ctas = num_sms * per_sm;
  p.max_segments = static_cast<int>(d.n / 2048);
  if (p.max_segments < 1) p.max_segments = 1;
  if (p.max_segments > 16) p.max_segments = 16;
  if (const char* s = std::getenv("LSAPGPU_SCAN_SEGMENTS")) p.max_segments = std::atoi(s);
  // streaming kernel: two vector steps in flight for float storage (fp64
  // tracks leave registers for one more stream set), one for integer keys
  p.depth = (d.storage == kF32 || d.storage == kF64) && p.m <= 2 ? 3 : 2;
  if (const char* dd = std::getenv("LSAPGPU_SCAN_DEPTH")) p.depth = std::atoi(dd) == 3 ? 3 : 2;
  // Resident-state kernel when tau16 + acur + two (A, AT) stages fit on chip
  // (LSAPGPU_SCAN_RESIDENT=0 forces the streaming kernel).
  int resident = 1;
  if (const char* r = std::getenv("LSAPGPU_SCAN_RESIDENT")) resident = std::atoi(r);
  if (resident && d.n < 65536 && d.tau16 && !std::getenv("LSAPGPU_SCAN_BUDGET")) {
    const size_t limit = 227 * 1024 - 14 * 1024;
    int m = 0;
    for (int mm : {4, 2, 1})
      if (res_smem_bytes(d.ld, es, mm, 2) <= limit) {
        m = mm;
        break;
      }
    if (force_m == 1 || force_m == 2 || force_m == 4)
      m = res_smem_bytes(d.ld, es, force_m, 2) <= limit ? force_m : 0;
    int bufs = 2;
    if (force_bufs >= 2 && force_bufs <= 4 && m && res_smem_bytes(d.ld, es, m, force_bufs) <= limit)
      bufs = force_bufs;
    if (m) {
      p.resident = 1;
      p.m = m;
      p.bufs = bufs;
      p.passes = 1;
      p.chunk = d.ld;
      p.threads = 512;
      if (const char* t = std::getenv("LSAPGPU_SCAN_RES_NT")) p.threads = std::atoi(t);
      p.smem = res_smem_bytes(d.ld, es, m, bufs);
      p.ctas = num_sms;
      // splitting items over CTAs re-stages whole rows per segment and adds a
      // cross-CTA merge; measured slower than whole items at every list size
      // (even lists shorter than the grid), so it is opt-in
      p.max_segments = 1;
      if (const char* sg = std::getenv("LSAPGPU_SCAN_SEGMENTS")) p.max_segments = std::atoi(sg);
      // L2 prefetch of the rows one stage ahead: C3 (n = 10k) solve -1.6 %, but
      // +0.9 % at n = 5k and neutral at 1k (tools/ab.py, round 2): rows of
      // 16 KB and up only; distance 2 -0.8 %, 4 +8 % at C3
      p.l2_prefetch = d.n >= 8192 ? 1 : 0;
      if (const char* pf = std::getenv("LSAPGPU_SCAN_L2PF")) p.l2_prefetch = std::atoi(pf);
      if (p.l2_prefetch >= 32 / m) p.l2_prefetch = 32 / m - 1;
    }
  }
  // Long rows (any storage the resident kernel cannot hold on chip): the
  // quantized-filter kernel (scan_filter.cuh) reads int16 (or int8) copies
  // of the rows and verifies the few surviving candidates exactly.  LSAPGPU_SCAN_FILTER=0 disables it, =2 forces it at
  // any n (tests); LSAPGPU_FILTER_BITS=8|16, LSAPGPU_FILTER_RB=1|2 and
  // LSAPGPU_FILTER_QUEUE=k pin the geometry so tests reach every path.
  int filt = 1;
  if (const char* f = std::getenv("LSAPGPU_SCAN_FILTER")) filt = std::atoi(f);
  if (filt && d.n < 131072 && (!p.resident || filt >= 2) &&
      !std::getenv("LSAPGPU_SCAN_BUDGET")) {
    const size_t limit = 232448 - 8 * 1024;  // dynamic smem next to the kernel's static ~7 KB
    int want_bits = 0, want_rb = 0;
    if (const char* b = std::getenv("LSAPGPU_FILTER_BITS")) want_bits = std::atoi(b);
    if (const char* r = std::getenv("LSAPGPU_FILTER_RB")) want_rb = std::atoi(r);
    int want_q = -1;
    if (const char* qq = std::getenv("LSAPGPU_FILTER_QUEUE")) want_q = std::max(0, std::min(kFilterQueueMax, std::atoi(qq)));
    const int threads = 32 * 19;  // 16 consumer warps x 8 positions per lane + 3 role warps
    const int32_t chunk = kFilterChunk;
    // aux[] resident in tensor memory where it fits (n <= 65536; measured at
    // C4: full sweep 0.85 -> 0.69 ms); LSAPGPU_FILTER_TMEM=0 keeps it in L2
    int tmem_aux = 1;
    if (const char* t = std::getenv("LSAPGPU_FILTER_TMEM")) tmem_aux = std::atoi(t) != 0;
    // prefer int16 copies, then double-buffered rows with a 1024-entry queue
    // and >= 3 slots, then one row buffer (its refill streams from L2: the
    // next row is prefetched; measured faster at C5 than two rows with a
    // 3-slot ring), then a 512-entry queue
    bool done = false;
    for (int qb : {2, 1}) {
      if (want_bits && want_bits != 8 * qb) continue;
      for (int qcap : {kFilterQueueMax, kFilterQueueMax / 2}) {
        if (want_q >= 0) qcap = want_q;
        for (int rb : {2, 1}) {
          if (want_rb && want_rb != rb) continue;
          int ns = 8;
          while (ns >= 3 && filter_smem(d.ld, qb, rb, ns, qcap, chunk) > limit) --ns;
          if (ns < 3) continue;
          p.filter = 8 * qb;
          p.m = rb;
          p.bufs = ns;
          p.resident = 0;
          p.passes = 1;
          p.chunk = chunk;
          p.threads = threads;
          p.smem = filter_smem(d.ld, qb, rb, ns, qcap, chunk);
          p.ctas = num_sms;
          p.max_segments = 1;
          p.l2_prefetch = 0;
          p.filter_queue = qcap;
          // aux[] in tensor memory: the first 16 chunks (512 columns; all of
          // it for n <= 65536), the rest from L2
          p.filter_tmem = tmem_aux;
          done = true;
          break;
        }
        if (done) break;
      }
      if (done) break;
    }
  }
  return p;
}

cudaError_t launch_scan(const DevState& d, const ScanPlan& p, int full, cudaStream_t st) {
  if (p.filter) {
    if (!d.Q || !d.QT || !d.aux) return cudaErrorInvalidValue;
    switch (d.storage) {
      case kI16: return launch_scan_filter_typed<int16_t>(d, p, full, st);
      case kI32: return launch_scan_filter_typed<int32_t>(d, p, full, st);
      case kF32: return launch_scan_filter_typed<float>(d, p, full, st);
      case kF64: return launch_scan_filter_typed<double>(d, p, full, st);
      default: return cudaErrorInvalidValue;
    }
  }
  if (p.resident) {
    switch (d.storage) {
      case kI16:
        return d.n <= 16384 ? launch_scan_res_typed<int16_t, kPacked32>(d, p, full, st)
                            : launch_scan_res_typed<int16_t, kPacked64>(d, p, full, st);
      case kI32: return launch_scan_res_typed<int32_t, kPacked64>(d, p, full, st);
      case kF32: return launch_scan_res_typed<float, kFloat>(d, p, full, st);
      case kF64: return launch_scan_res_typed<double, kFloat>(d, p, full, st);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (d.storage) {
    case kI16:
      return d.n <= 16384 ? launch_scan_typed<int16_t, kPacked32>(d, p, full, st)
                          : launch_scan_typed<int16_t, kPacked64>(d, p, full, st);
    case kI32: return launch_scan_typed<int32_t, kPacked64>(d, p, full, st);
    case kF32: return launch_scan_typed<float, kFloat>(d, p, full, st);
    case kF64: return launch_scan_typed<double, kFloat>(d, p, full, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lsapgpu
