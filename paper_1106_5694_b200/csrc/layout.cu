// layout.cu -- device-resident instance layout (replaces Instance::validate,
// proj/src/core.cpp:9-15, and SolverState::build_columns,
// proj/src/solver_state.hpp:67-76), on-device synthetic instance generators
// (geom.cpp:15-33), and the O(n) assignment helpers.
//
// classify: one pass over the fp64 (or narrower) source that decides the
//   narrowest lossless storage type and detects non-finite entries.
// build_layout: 32x32 smem-tiled convert + transpose writing A and AT in one
//   pass (read 1x, write 2x).  The generators plug in as the tile source, so a
//   100k x 100k instance never exists in host memory or as an fp64 copy.
#include <cmath>

#include "state.h"

namespace lsapgpu {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// k-th draw of SplitMix64(seed) (rng.hpp:11-22): counter-based.
__device__ __forceinline__ uint64_t draw(uint64_t seed, uint64_t k) {
  return mix64(seed + (k + 1) * 0x9E3779B97F4A7C15ull);
}
// rng.hpp:32-34: u / (2^64 - 1); the divisor rounds to 2^64 in fp64.
__device__ __forceinline__ double unit_double(uint64_t u) {
  return __ddiv_rn(__ull2double_rn(u), 18446744073709551615.0);
}

struct Src {
  LayoutSource s;
  int32_t n;
  // row-block placement: does this rank hold row i of A, and where
  __device__ __forceinline__ bool own(int64_t i) const {
    return s.a_rows < 0 || (i >= s.a_row0 && i < static_cast<int64_t>(s.a_row0) + s.a_rows);
  }
  __device__ __forceinline__ int64_t local(int64_t i) const { return s.a_rows < 0 ? i : i - s.a_row0; }
  __device__ __forceinline__ double operator()(int64_t i, int64_t j) const {
    const int64_t k = i * n + j;
    switch (s.kind) {
      case 0:
        switch (s.src_dtype) {
          case 0: return static_cast<const double*>(s.src)[k];
          case 1: return static_cast<double>(static_cast<const float*>(s.src)[k]);
          case 2: return static_cast<double>(static_cast<const int32_t*>(s.src)[k]);
          default: return static_cast<double>(static_cast<const int16_t*>(s.src)[k]);
        }
      case 1:
        return __ull2double_rn(draw(s.seed, static_cast<uint64_t>(k)) %
                               static_cast<uint64_t>(s.param));
      case 2:
        return static_cast<double>(__double2float_rn(unit_double(draw(s.seed, static_cast<uint64_t>(k)))));
      case 3:
        return __dmul_rn(unit_double(draw(s.seed, static_cast<uint64_t>(k))), s.param);
      case 4: {  // p2p: aux = up[n], x[n], y[n]
        if (i == j) return 0.0;
        const double* up = s.aux;
        const double* xs = s.aux + n;
        const double* ys = s.aux + 2 * static_cast<int64_t>(n);
        const int64_t dx = llabs(static_cast<int64_t>(xs[i]) - static_cast<int64_t>(xs[j]));
        const int64_t dy = llabs(static_cast<int64_t>(ys[i]) - static_cast<int64_t>(ys[j]));
        const int64_t lat = 1 + (dx + dy) / 16;
        return static_cast<double>(static_cast<int64_t>(up[i]) * (256 - lat));
      }
      default: {  // geom: aux = xs[n], ys[n]
        const double dx = __dsub_rn(s.aux[i], s.aux[j]);
        const double dy = __dsub_rn(s.aux[n + i], s.aux[n + j]);
        return __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
      }
    }
  }
};

__global__ void gen_aux_kernel(LayoutSource s, int32_t n, double* aux) {
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  if (s.kind == 4) {
    aux[k] = static_cast<double>(1ll << (draw(s.seed, static_cast<uint64_t>(k)) % 6));
    aux[n + k] = static_cast<double>(draw(s.seed, static_cast<uint64_t>(n) + 2ull * k) % 1024);
    aux[2 * static_cast<int64_t>(n) + k] =
        static_cast<double>(draw(s.seed, static_cast<uint64_t>(n) + 2ull * k + 1) % 1024);
  } else if (s.kind == 5) {
    aux[k] = __dmul_rn(unit_double(draw(s.seed, 2ull * k)), s.param);
    aux[n + k] = __dmul_rn(unit_double(draw(s.seed, 2ull * k + 1)), s.param);
  }
}

// Storage flags of one entry (bit0 non-finite, bit1 not int16-exact, bit2 not
// an integer below 2^29, bit3 not fp32-exact) from the entry and its two
// conversions (iv = the saturating double->int, fv = the nearest float),
// branch-free: the layout pass reuses the same conversions as the stored
// narrow value, so a C3 entry costs one F2I and one F2F plus compares.
__device__ __forceinline__ uint32_t entry_flags_c(double v, int32_t iv, float fv) {
  const bool integral = static_cast<double>(iv) == v;  // (false for NaN / inf)
  const uint32_t a = static_cast<uint32_t>(iv < 0 ? -static_cast<int64_t>(iv) : iv);
  uint32_t f = (integral && a <= 32767u) ? 0u : 2u;
  f |= (integral && a < 536870912u) ? 0u : 4u;
  f |= (static_cast<double>(fv) == v) ? 0u : 8u;
  return isfinite(v) ? f : 15u;
}

// The same, one conversion pair for the common integer case (classify probe).
__device__ __forceinline__ uint32_t entry_flags(double v) {
  if (!isfinite(v)) return 1u | 2u | 4u | 8u;
  const int32_t iv = __double2int_rz(v);  // saturates
  const bool integral = static_cast<double>(iv) == v;
  const uint32_t a = static_cast<uint32_t>(iv < 0 ? -static_cast<int64_t>(iv) : iv);
  if (integral && a <= 32767u) return 0u;
  uint32_t f = 2u;
  if (!(integral && a < 536870912u)) f |= 4u;
  if (static_cast<double>(__double2float_rn(v)) != v) f |= 8u;
  return f;
}

__global__ void classify_kernel(Src src, int64_t row0, int64_t rows, uint32_t* flags, uint32_t* amax) {
  uint32_t f = 0;
  float vmax = 0.f;
  const int64_t total = rows * src.n;  // flat over the block of rows: every thread busy
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = src(row0 + e / src.n, static_cast<int32_t>(e % src.n));
    f |= entry_flags(v);
    if (isfinite(v)) vmax = fmaxf(vmax, __double2float_ru(fabs(v)));
  }
  if (amax) {  // (per-thread atomics: the probe is 64 rows)
    for (int off = 16; off > 0; off >>= 1) vmax = fmaxf(vmax, __shfl_down_sync(0xffffffffu, vmax, off));
    if ((threadIdx.x & 31) == 0 && vmax > 0.f) atomicMax(amax, __float_as_uint(vmax));
  }
  // warp then block OR, one atomic per block
  for (int off = 16; off > 0; off >>= 1) f |= __shfl_down_sync(0xffffffffu, f, off);
  __shared__ uint32_t wf[32];
  if ((threadIdx.x & 31) == 0) wf[threadIdx.x >> 5] = f;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t r = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) r |= wf[w];
    if (r) atomicOr(flags, r);
  }
}

template <class E>
__device__ __forceinline__ E narrow(double v) {
  // (truncating conversion: the stored values are exact integers, and it is
  // the same instruction entry_flags issues)
  if constexpr (sizeof(E) == 2)
    return static_cast<int16_t>(__double2int_rz(v));
  else if constexpr (Traits<E>::kInt)
    return static_cast<int32_t>(__double2int_rz(v));
  else if constexpr (sizeof(E) == 4)
    return __double2float_rn(v);
  else
    return v;
}

// narrow<E> from the conversions entry_flags_c already made (non-finite -> 0)
template <class E>
__device__ __forceinline__ E narrow_c(double v, int32_t iv, float fv) {
  const bool fin = isfinite(v);
  if constexpr (Traits<E>::kInt)
    return static_cast<E>(fin ? iv : 0);
  else if constexpr (sizeof(E) == 4)
    return fin ? fv : 0.f;
  else
    return fin ? v : 0.0;
}

// 32x32 tiles, 32x8 threads: A tile written row-major, AT tile through smem.
template <class E>
__global__ void build_layout_kernel(Src src, int64_t row0, int64_t rows, E* A, E* AT, int64_t ld) {
  __shared__ E tile[32][33];
  const int64_t bi = row0 + static_cast<int64_t>(blockIdx.y) * 32;  // agent block
  const int64_t bj = static_cast<int64_t>(blockIdx.x) * 32;         // job block
  const int n = src.n;
  const int64_t rend = row0 + rows;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t i = bi + r, j = bj + threadIdx.x;
    if (i < rend && j < n) {
      const E v = narrow<E>(src(i, j));
      if (src.own(i)) A[src.local(i) * ld + j] = v;
      tile[r][threadIdx.x] = v;
    }
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t j = bj + r, i = bi + threadIdx.x;
    if (j < n && i < rend) AT[j * ld + i] = tile[threadIdx.x][r];
  }
}

// Fused layout pass: classify (flags as classify_kernel) and build (narrow +
// transpose as build_layout_kernel) in ONE read of the source, for a storage
// type speculated from the first rows (the caller rebuilds in the rare case
// the flags demand a wider type).  64x64 tiles, 256 threads: each lane owns
// two adjacent columns, so the source reads, the A-row writes and the AT-row
// writes are all coalesced.
// Two adjacent elements in one store (the pair is 2-element aligned: ld is a
// multiple of 64 and the column even).
template <class E>
struct Pair;
template <>
struct Pair<int16_t> {
  __device__ static void st(int16_t* p, int16_t a, int16_t b) {
    *reinterpret_cast<uint32_t*>(p) = static_cast<uint16_t>(a) | (static_cast<uint32_t>(static_cast<uint16_t>(b)) << 16);
  }
};
template <>
struct Pair<int32_t> {
  __device__ static void st(int32_t* p, int32_t a, int32_t b) { *reinterpret_cast<int2*>(p) = make_int2(a, b); }
};
template <>
struct Pair<float> {
  __device__ static void st(float* p, float a, float b) { *reinterpret_cast<float2*>(p) = make_float2(a, b); }
};
template <>
struct Pair<double> {
  __device__ static void st(double* p, double a, double b) { *reinterpret_cast<double2*>(p) = make_double2(a, b); }
};

// Quantized filter copies written by the layout pass itself (scan_filter.cuh):
// element k of `Q` = ceil(v * scale) as int16 / int8 (exact: scale is a power
// of two).  Two adjacent elements, the second only when `both`.
__device__ __forceinline__ void qstore_pair(const QuantTarget& qt, int64_t k, double v0, double v1, bool both) {
  const int32_t q0 = static_cast<int32_t>(ceil(v0 * qt.scale)), q1 = static_cast<int32_t>(ceil(v1 * qt.scale));
  if (qt.bits == 16) {
    int16_t* Q = static_cast<int16_t*>(qt.Q);
    if (both)
      *reinterpret_cast<uint32_t*>(Q + k) =
          static_cast<uint16_t>(q0) | (static_cast<uint32_t>(static_cast<uint16_t>(q1)) << 16);
    else
      Q[k] = static_cast<int16_t>(q0);
  } else {
    int8_t* Q = static_cast<int8_t*>(qt.Q);
    if (both)
      *reinterpret_cast<uint16_t*>(Q + k) =
          static_cast<uint16_t>(static_cast<uint8_t>(q0) | (static_cast<uint16_t>(static_cast<uint8_t>(q1)) << 8));
    else
      Q[k] = static_cast<int8_t>(q0);
  }
}

// The common case on its own: an fp64 matrix in memory with an even n, every
// row of A held, no max|a| and no filter copies (C1-C3 from a device matrix
// or the host fallback).  Same tiles and results as layout_fused_kernel, with
// no per-element guards beyond the row / column range and incremented
// pointers, so the pass is no longer instruction-bound.
template <class E>
__global__ void __launch_bounds__(256) layout_plain_kernel(const double* __restrict__ src, int32_t n, int64_t row0,
                                                           int64_t rows, E* __restrict__ A, E* __restrict__ AT,
                                                           int64_t ld, uint32_t* flags) {
  __shared__ E tile[64][66];
  const int64_t bi = row0 + static_cast<int64_t>(blockIdx.y) * 64;  // agent block
  const int32_t bj = static_cast<int32_t>(blockIdx.x) * 64;         // job block
  const int lane = threadIdx.x & 31, rg = threadIdx.x >> 5;         // 8 row groups
  const int32_t j = bj + 2 * lane;
  const bool jv = j < n;  // (n even: both columns of the lane, or neither)
  const int64_t rend = row0 + rows;
  const int64_t left = rend - bi - rg;  // rows of this thread in the tile: rg, rg + 8, ...
  const int nq = left <= 0 ? 0 : (left >= 57 ? 8 : static_cast<int>((left + 7) / 8));
  double2 v[8];
  const double* sp = src + (bi + rg) * static_cast<int64_t>(n) + j;
#pragma unroll
  for (int q = 0; q < 8; ++q)
    v[q] = (q < nq && jv) ? __ldg(reinterpret_cast<const double2*>(sp + static_cast<int64_t>(8 * q) * n))
                          : make_double2(0.0, 0.0);
  uint32_t f = 0;
  E* ap = A + (bi + rg) * ld + j;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (q >= nq) break;
    const int32_t i0 = __double2int_rz(v[q].x), i1 = __double2int_rz(v[q].y);
    const float f0 = __double2float_rn(v[q].x), f1 = __double2float_rn(v[q].y);
    const E e0 = narrow_c<E>(v[q].x, i0, f0), e1 = narrow_c<E>(v[q].y, i1, f1);
    if (jv) {
      f |= entry_flags_c(v[q].x, i0, f0) | entry_flags_c(v[q].y, i1, f1);
      Pair<E>::st(ap + static_cast<int64_t>(8 * q) * ld, e0, e1);
    }
    tile[rg + 8 * q][2 * lane] = e0;
    tile[rg + 8 * q][2 * lane + 1] = e1;
  }
  __syncthreads();
  // AT rows bj .. bj+63, columns (agents) bi .. bi+63
  const int64_t ia = bi + 2 * lane;
  const bool iv1 = ia + 1 < rend, iv0 = ia < rend;
  E* atp = AT + static_cast<int64_t>(bj + rg) * ld + ia;
#pragma unroll
  for (int c = rg; c < 64; c += 8, atp += 8 * ld) {
    if (bj + c >= n) break;
    if (iv1)
      Pair<E>::st(atp, tile[2 * lane][c], tile[2 * lane + 1][c]);
    else if (iv0)
      atp[0] = tile[2 * lane][c];
  }
  for (int off = 16; off > 0; off >>= 1) f |= __shfl_down_sync(0xffffffffu, f, off);
  __shared__ uint32_t wf[8];
  if (lane == 0) wf[rg] = f;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t r = 0;
    for (int w = 0; w < 8; ++w) r |= wf[w];
    if (r) atomicOr(flags, r);
  }
}

// kF64: the source is an fp64 matrix in memory with an even n (the bench's
// and every host upload's fallback case): direct 16-byte loads, and none of
// the generic source code is compiled into the instantiation.
template <class E, bool kF64>
__global__ void __launch_bounds__(256) layout_fused_kernel(Src src, int64_t row0, int64_t rows, E* A, E* AT,
                                                           int64_t ld, uint32_t* flags, uint32_t* amax,
                                                           QuantTarget qt) {
  __shared__ E tile[64][66];
  const int64_t bi = row0 + static_cast<int64_t>(blockIdx.y) * 64;  // agent block
  const int64_t bj = static_cast<int64_t>(blockIdx.x) * 64;         // job block
  const int n = src.n;
  const int64_t rend = row0 + rows;
  const int lane = threadIdx.x & 31, rg = threadIdx.x >> 5;  // 8 row groups
  const int64_t j = bj + 2 * lane;
  uint32_t f = 0;
  float vmax = 0.f;  // max |entry| rounded up to fp32 (the filter scan's quantization scale)
  // all eight rows' loads first (8 x 16 B in flight per lane), then classify / store
  double v[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int64_t i = bi + rg + 8 * q;
    v[q][0] = v[q][1] = 0.0;
    if (i >= rend) continue;
    if constexpr (kF64) {  // (n even: j < n implies j + 1 < n)
      if (j < n) {
        const double2 w = __ldg(reinterpret_cast<const double2*>(static_cast<const double*>(src.s.src) + i * n + j));
        v[q][0] = w.x;
        v[q][1] = w.y;
      }
    } else {
      if (j < n) v[q][0] = src(i, j);
      if (j + 1 < n) v[q][1] = src(i, j + 1);
    }
  }
  // column guards (kF64: n even, so both columns of a lane are in or out together)
  const bool jv0 = j < n, jv1 = kF64 ? jv0 : j + 1 < n;
  const bool all_rows = src.s.a_rows < 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int r = rg + 8 * q;
    const int64_t i = bi + r;
    if (i >= rend) break;
    const double v0 = v[q][0], v1 = v[q][1];
    const int32_t i0 = __double2int_rz(v0), i1 = __double2int_rz(v1);
    const float f0 = __double2float_rn(v0), f1 = __double2float_rn(v1);
    f |= (jv0 ? entry_flags_c(v0, i0, f0) : 0u) | (jv1 ? entry_flags_c(v1, i1, f1) : 0u);
    if (amax) {
      if (jv0 && isfinite(v0)) vmax = fmaxf(vmax, __double2float_ru(fabs(v0)));
      if (jv1 && isfinite(v1)) vmax = fmaxf(vmax, __double2float_ru(fabs(v1)));
    }
    const E e0 = narrow_c<E>(v0, i0, f0), e1 = narrow_c<E>(v1, i1, f1);
    const bool own = all_rows || src.own(i);  // row-block placement: A / Q rows of this rank only
    const int64_t li = all_rows ? i : src.local(i);
    if (own && jv1)
      Pair<E>::st(A + li * ld + j, e0, e1);
    else if (own && jv0)
      A[li * ld + j] = e0;
    tile[r][2 * lane] = e0;
    tile[r][2 * lane + 1] = e1;
    if (qt.bits && own && jv0)
      qstore_pair(qt, li * ld + j, static_cast<double>(e0), static_cast<double>(e1), jv1);
  }
  __syncthreads();
  // AT rows bj .. bj+63, columns (agents) bi .. bi+63
  const int64_t ia = bi + 2 * lane;
  for (int c = rg; c < 64; c += 8) {
    const int64_t jj = bj + c;
    if (jj >= n) break;
    E* at = AT + jj * ld + ia;
    if (ia + 1 < rend)
      Pair<E>::st(at, tile[2 * lane][c], tile[2 * lane + 1][c]);
    else if (ia < rend)
      at[0] = tile[2 * lane][c];
    if (qt.bits && ia < rend)  // QT = the same values quantized, transposed
      qstore_pair(QuantTarget{qt.QT, nullptr, qt.scale, qt.bits}, jj * ld + ia, static_cast<double>(tile[2 * lane][c]),
                  static_cast<double>(tile[2 * lane + 1][c]), ia + 1 < rend);
  }
  for (int off = 16; off > 0; off >>= 1) f |= __shfl_down_sync(0xffffffffu, f, off);
  __shared__ uint32_t wf[8];
  __shared__ float wm[8];
  if (lane == 0) wf[rg] = f;
  if (amax) {
    for (int off = 16; off > 0; off >>= 1) vmax = fmaxf(vmax, __shfl_down_sync(0xffffffffu, vmax, off));
    if (lane == 0) wm[rg] = vmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t r = 0;
    for (int w = 0; w < 8; ++w) r |= wf[w];
    if (r) atomicOr(flags, r);
    if (amax) {
      float m = 0.f;
      for (int w = 0; w < 8; ++w) m = fmaxf(m, wm[w]);
      if (m > 0.f) atomicMax(amax, __float_as_uint(m));  // non-negative floats order as their bits
    }
  }
}

// Filter copies (scan_filter.cuh): Q = ceil(A * scale) as int16 / int8, an
// upper bound of every entry in units of 1/scale (scale is a power of two, so
// the product is exact in fp64 and so is the ceiling); padding columns 0.
template <class E, class Qt>
__global__ void quantize_kernel(const E* __restrict__ src, Qt* __restrict__ dst, int64_t total, int32_t n,
                                int64_t ld, double scale) {
  for (int64_t k = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8; k < total;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x * 8) {
    const int64_t col = k % ld;  // ld is a multiple of 64: the 8 elements share a row
    Qt out[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      out[e] = col + e < n ? static_cast<Qt>(ceil(static_cast<double>(src[k + e]) * scale)) : Qt(0);
    if constexpr (sizeof(Qt) == 2) {
      uint4 w;
      w.x = static_cast<uint16_t>(out[0]) | (static_cast<uint32_t>(static_cast<uint16_t>(out[1])) << 16);
      w.y = static_cast<uint16_t>(out[2]) | (static_cast<uint32_t>(static_cast<uint16_t>(out[3])) << 16);
      w.z = static_cast<uint16_t>(out[4]) | (static_cast<uint32_t>(static_cast<uint16_t>(out[5])) << 16);
      w.w = static_cast<uint16_t>(out[6]) | (static_cast<uint32_t>(static_cast<uint16_t>(out[7])) << 16);
      *reinterpret_cast<uint4*>(dst + k) = w;
    } else {
      uint2 w;
      w.x = 0;
      w.y = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        w.x |= static_cast<uint32_t>(static_cast<uint8_t>(out[e])) << (8 * e);
        w.y |= static_cast<uint32_t>(static_cast<uint8_t>(out[4 + e])) << (8 * e);
      }
      *reinterpret_cast<uint2*>(dst + k) = w;
    }
  }
}

template <class E>
__global__ void init_assignment_kernel(DevState d) {
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d.n) return;
  const E* AT = static_cast<const E*>(d.AT);  // A[i][j] = AT[j][i] (A may be a row block)
  const int32_t i = d.sigma[j];
  d.tau[i] = j;
  if (d.tau16) d.tau16[i] = static_cast<uint16_t>(j);
  static_cast<E*>(d.acur)[i] = AT[static_cast<int64_t>(j) * d.ld + i];
}

template <class E>
__global__ void gather_current_kernel(DevState d, double* out, int pack) {
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d.n) return;
  const E* AT = static_cast<const E*>(d.AT);
  const int32_t sj = d.sigma[j];
  out[j] = static_cast<double>(AT[static_cast<int64_t>(j) * d.ld + sj]);
  if (pack) {  // [values | sigma | tau] for one device->host copy
    int32_t* w = reinterpret_cast<int32_t*>(out + d.n);
    w[j] = sj;
    w[d.n + j] = d.tau[j];
  }
}

template <class E>
__global__ void read_rows_kernel(DevState d, const int32_t* rows, int32_t nrows, double* out) {
  const E* AT = static_cast<const E*>(d.AT);  // (A may be a row block; AT is whole)
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       k < static_cast<int64_t>(nrows) * d.n; k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = k / d.n, j = k % d.n;
    out[k] = static_cast<double>(AT[j * d.ld + rows[r]]);
  }
}

template <template <class> class K, class... Args>
cudaError_t dispatch(int storage, dim3 g, dim3 b, cudaStream_t st, Args... args) {
  switch (storage) {
    case kI16: K<int16_t>::run(g, b, st, args...); break;
    case kI32: K<int32_t>::run(g, b, st, args...); break;
    case kF32: K<float>::run(g, b, st, args...); break;
    case kF64: K<double>::run(g, b, st, args...); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <class E>
struct BuildK {
  static void run(dim3 g, dim3 b, cudaStream_t st, Src s, int64_t r0, int64_t rows, void* A, void* AT,
                  int64_t ld) {
    build_layout_kernel<E><<<g, b, 0, st>>>(s, r0, rows, static_cast<E*>(A), static_cast<E*>(AT), ld);
  }
};
template <class E>
struct FusedK {
  static void run(dim3 g, dim3 b, cudaStream_t st, Src s, int64_t r0, int64_t rows, void* A, void* AT,
                  int64_t ld, uint32_t* flags, uint32_t* amax, QuantTarget qt) {
    if (s.s.kind == 0 && s.s.src_dtype == 0 && (s.n & 1) == 0 && s.s.a_rows < 0 && !amax && !qt.bits)
      layout_plain_kernel<E><<<g, b, 0, st>>>(static_cast<const double*>(s.s.src), s.n, r0, rows, static_cast<E*>(A),
                                              static_cast<E*>(AT), ld, flags);
    else if (s.s.kind == 0 && s.s.src_dtype == 0 && (s.n & 1) == 0)
      layout_fused_kernel<E, true><<<g, b, 0, st>>>(s, r0, rows, static_cast<E*>(A), static_cast<E*>(AT), ld, flags,
                                                    amax, qt);
    else
      layout_fused_kernel<E, false><<<g, b, 0, st>>>(s, r0, rows, static_cast<E*>(A), static_cast<E*>(AT), ld,
                                                     flags, amax, qt);
  }
};
template <class E>
struct QuantK {
  static void run(dim3 g, dim3 b, cudaStream_t st, const void* src, void* dst, int64_t total, int32_t n,
                  int64_t ld, double scale, int qbits) {
    if (qbits == 16)
      quantize_kernel<E, int16_t><<<g, b, 0, st>>>(static_cast<const E*>(src), static_cast<int16_t*>(dst), total, n,
                                                   ld, scale);
    else
      quantize_kernel<E, int8_t><<<g, b, 0, st>>>(static_cast<const E*>(src), static_cast<int8_t*>(dst), total, n,
                                                  ld, scale);
  }
};
template <class E>
struct InitK {
  static void run(dim3 g, dim3 b, cudaStream_t st, DevState d) {
    init_assignment_kernel<E><<<g, b, 0, st>>>(d);
  }
};
template <class E>
struct GatherK {
  static void run(dim3 g, dim3 b, cudaStream_t st, DevState d, double* out, int pack) {
    gather_current_kernel<E><<<g, b, 0, st>>>(d, out, pack);
  }
};
template <class E>
struct RowsK {
  static void run(dim3 g, dim3 b, cudaStream_t st, DevState d, const int32_t* rows, int32_t nr,
                  double* out) {
    read_rows_kernel<E><<<g, b, 0, st>>>(d, rows, nr, out);
  }
};

}  // namespace

cudaError_t launch_gen_aux(const LayoutSource& s, int32_t n, double* aux, cudaStream_t st) {
  gen_aux_kernel<<<(n + 255) / 256, 256, 0, st>>>(s, n, aux);
  return cudaGetLastError();
}

cudaError_t launch_classify(const LayoutSource& s, int32_t n, int64_t row0, int64_t rows,
                            uint32_t* flags, cudaStream_t st, uint32_t* amax) {
  Src src{s, n};
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  classify_kernel<<<sms * 8, 256, 0, st>>>(src, row0, rows, flags, amax);
  return cudaGetLastError();
}

cudaError_t launch_build_layout(const LayoutSource& s, int32_t n, int64_t row0, int64_t rows,
                                int storage, void* A, void* AT, int64_t ld, cudaStream_t st) {
  Src src{s, n};
  dim3 g(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  return dispatch<BuildK>(storage, g, dim3(32, 8), st, src, row0, rows, A, AT, ld);
}

cudaError_t launch_layout_fused(const LayoutSource& s, int32_t n, int64_t row0, int64_t rows, int storage,
                                void* A, void* AT, int64_t ld, uint32_t* flags, cudaStream_t st, uint32_t* amax,
                                QuantTarget qt) {
  Src src{s, n};
  dim3 g(static_cast<unsigned>((n + 63) / 64), static_cast<unsigned>((rows + 63) / 64));
  return dispatch<FusedK>(storage, g, dim3(256), st, src, row0, rows, A, AT, ld, flags, amax, qt);
}

// max |a| over the stored matrix (AT: whole on every rank), float bits rounded up
template <class E>
__global__ void amax_kernel(const E* __restrict__ AT, int32_t n, int64_t ld, uint32_t* out) {
  float m = 0.f;
  const int64_t total = static_cast<int64_t>(n) * ld;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (k % ld < n) m = fmaxf(m, __double2float_ru(fabs(static_cast<double>(AT[k]))));
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_down_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(out, __float_as_uint(m));
}
template <class E>
struct AmaxK {
  static void run(dim3 g, dim3 b, cudaStream_t st, const void* AT, int32_t n, int64_t ld, uint32_t* out) {
    amax_kernel<E><<<g, b, 0, st>>>(static_cast<const E*>(AT), n, ld, out);
  }
};

cudaError_t launch_amax(const DevState& d, uint32_t* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  return dispatch<AmaxK>(d.storage, dim3(148 * 8), dim3(256), st, d.AT, d.n, d.ld, out);
}

cudaError_t launch_quantize(const DevState& d, int qbits, double scale, void* Q, void* QT, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(d.n) * d.ld;
  const int64_t a_total = static_cast<int64_t>(d.a_rows) * d.ld;  // A / Q: this rank's row block
  const dim3 g(148 * 8), b(256);
  cudaError_t e = dispatch<QuantK>(d.storage, g, b, st, d.A, Q, a_total, d.n, d.ld, scale, qbits);
  if (e != cudaSuccess) return e;
  return dispatch<QuantK>(d.storage, g, b, st, d.AT, QT, total, d.n, d.ld, scale, qbits);
}

cudaError_t launch_init_assignment(const DevState& d, cudaStream_t st) {
  return dispatch<InitK>(d.storage, dim3((d.n + 255) / 256), dim3(256), st, d);
}

cudaError_t launch_gather_current(const DevState& d, double* out, cudaStream_t st, int pack) {
  return dispatch<GatherK>(d.storage, dim3((d.n + 255) / 256), dim3(256), st, d, out, pack);
}

cudaError_t launch_read_rows(const DevState& d, const int32_t* rows, int32_t nrows, double* out,
                             cudaStream_t st) {
  return dispatch<RowsK>(d.storage, dim3(1024), dim3(256), st, d, rows, nrows, out);
}

}  // namespace lsapgpu
