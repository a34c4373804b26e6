// host_narrow.cpp -- exact fp64 -> int16 / int32 / fp32 narrowing of a host
// matrix chunk (the host half of the upload, lsapgpu.cu upload_narrow): the
// copy threads convert while they read, so PCIe carries 2 or 4 bytes per
// entry instead of 8.  AVX2 when the CPU has it (4 entries per instruction;
// the scalar loop does not vectorise because of the exactness reduction),
// the same rules in scalar code otherwise.  Compiled by the host compiler
// (build.py), not nvcc.
#include <immintrin.h>

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdlib>

namespace lsapgpu {

namespace {

constexpr double kF32Max = 3.4028234663852886e38;

// streaming stores (default) or plain stores (LSAPGPU_NARROW_NT=0: the ring
// slot stays in the cache hierarchy for the DMA engine to read)
bool use_nt() {
  static const bool v = !(std::getenv("LSAPGPU_NARROW_NT") && std::atoi(std::getenv("LSAPGPU_NARROW_NT")) == 0);
  return v;
}

// Software prefetch 4 KB ahead of the read (LSAPGPU_NARROW_PF, bytes; 0 =
// none): measured on the B200 box's 16 host cores, the exact int16
// narrowing of the 800 MB C3 matrix runs at 137 GB/s with it and 95 GB/s
// without (tools/micro/host_read.cpp; the plain read roofline is ~170 GB/s).
size_t pf_entries() {
  static const size_t v =
      (std::getenv("LSAPGPU_NARROW_PF") ? static_cast<size_t>(std::atoll(std::getenv("LSAPGPU_NARROW_PF"))) : 4096) / 8;
  return v;
}

template <class T>
bool narrow_scalar(const double* __restrict__ src, T* __restrict__ dst, size_t cnt, double lim) {
  bool ok = true;
  for (size_t i = 0; i < cnt; ++i) {
    const double v = src[i];
    if constexpr (sizeof(T) == 4 && static_cast<T>(0.5) != 0) {  // float
      const bool in = std::fabs(v) <= kF32Max;  // (false for NaN / inf)
      const float f = static_cast<float>(in ? v : 0.0);
      ok &= in & (static_cast<double>(f) == v);
      dst[i] = f;
    } else {
      const bool in = (v >= -lim) & (v <= lim);
      const int32_t x = static_cast<int32_t>(in ? v : 0.0);
      ok &= in & (static_cast<double>(x) == v);
      dst[i] = static_cast<T>(x);
    }
  }
  return ok;
}

// integer storage: |v| <= lim, integral; 8 entries per iteration
template <class T>
__attribute__((target("avx2"))) bool narrow_int_avx2(const double* __restrict__ src, T* __restrict__ dst, size_t cnt,
                                                     double lim) {
  const __m256d hi = _mm256_set1_pd(lim), lo = _mm256_set1_pd(-lim);
  __m256d ok = _mm256_castsi256_pd(_mm256_set1_epi64x(-1));
  size_t i = 0;
  const bool nt = use_nt() && (reinterpret_cast<uintptr_t>(dst) & 15) == 0 && (8 * sizeof(T)) % 16 == 0;
  const size_t pf = pf_entries();
  for (; i + 8 <= cnt; i += 8) {
    if (pf && i + pf < cnt) _mm_prefetch(reinterpret_cast<const char*>(src + i + pf), _MM_HINT_T0);
    const __m256d v0 = _mm256_loadu_pd(src + i), v1 = _mm256_loadu_pd(src + i + 4);
    const __m256d in0 = _mm256_and_pd(_mm256_cmp_pd(v0, lo, _CMP_GE_OQ), _mm256_cmp_pd(v0, hi, _CMP_LE_OQ));
    const __m256d in1 = _mm256_and_pd(_mm256_cmp_pd(v1, lo, _CMP_GE_OQ), _mm256_cmp_pd(v1, hi, _CMP_LE_OQ));
    const __m128i x0 = _mm256_cvttpd_epi32(_mm256_and_pd(v0, in0));
    const __m128i x1 = _mm256_cvttpd_epi32(_mm256_and_pd(v1, in1));
    const __m256d e0 = _mm256_cmp_pd(_mm256_cvtepi32_pd(x0), v0, _CMP_EQ_OQ);
    const __m256d e1 = _mm256_cmp_pd(_mm256_cvtepi32_pd(x1), v1, _CMP_EQ_OQ);
    ok = _mm256_and_pd(ok, _mm256_and_pd(_mm256_and_pd(in0, e0), _mm256_and_pd(in1, e1)));
    // streaming (non-temporal) stores when the destination is 16-byte
    // aligned: the pinned ring is written once and read by the DMA engine,
    // so reading its lines into the cache first (write-allocate) is waste
    if constexpr (sizeof(T) == 2) {
      if (nt) _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), _mm_packs_epi32(x0, x1));
      else _mm_storeu_si128(reinterpret_cast<__m128i*>(dst + i), _mm_packs_epi32(x0, x1));
    } else {
      if (nt) {
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), x0);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 4), x1);
      } else {
        _mm_storeu_si128(reinterpret_cast<__m128i*>(dst + i), x0);
        _mm_storeu_si128(reinterpret_cast<__m128i*>(dst + i + 4), x1);
      }
    }
  }
  if (nt) _mm_sfence();
  const bool vok = _mm256_movemask_pd(ok) == 0xF;
  return narrow_scalar<T>(src + i, dst + i, cnt - i, lim) && vok;
}

__attribute__((target("avx2"))) bool narrow_f32_avx2(const double* __restrict__ src, float* __restrict__ dst,
                                                     size_t cnt) {
  const __m256d mx = _mm256_set1_pd(kF32Max);
  const __m256d absmask = _mm256_castsi256_pd(_mm256_set1_epi64x(0x7fffffffffffffffLL));
  __m256d ok = _mm256_castsi256_pd(_mm256_set1_epi64x(-1));
  size_t i = 0;
  const bool nt = use_nt() && (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  const size_t pf = pf_entries();
  for (; i + 8 <= cnt; i += 8) {
    if (pf && i + pf < cnt) _mm_prefetch(reinterpret_cast<const char*>(src + i + pf), _MM_HINT_T0);
    const __m256d v0 = _mm256_loadu_pd(src + i), v1 = _mm256_loadu_pd(src + i + 4);
    const __m256d in0 = _mm256_cmp_pd(_mm256_and_pd(v0, absmask), mx, _CMP_LE_OQ);
    const __m256d in1 = _mm256_cmp_pd(_mm256_and_pd(v1, absmask), mx, _CMP_LE_OQ);
    const __m128 f0 = _mm256_cvtpd_ps(_mm256_and_pd(v0, in0));
    const __m128 f1 = _mm256_cvtpd_ps(_mm256_and_pd(v1, in1));
    const __m256d e0 = _mm256_cmp_pd(_mm256_cvtps_pd(f0), v0, _CMP_EQ_OQ);
    const __m256d e1 = _mm256_cmp_pd(_mm256_cvtps_pd(f1), v1, _CMP_EQ_OQ);
    ok = _mm256_and_pd(ok, _mm256_and_pd(_mm256_and_pd(in0, e0), _mm256_and_pd(in1, e1)));
    if (nt) {
      _mm_stream_ps(dst + i, f0);
      _mm_stream_ps(dst + i + 4, f1);
    } else {
      _mm_storeu_ps(dst + i, f0);
      _mm_storeu_ps(dst + i + 4, f1);
    }
  }
  if (nt) _mm_sfence();
  const bool vok = _mm256_movemask_pd(ok) == 0xF;
  return narrow_scalar<float>(src + i, dst + i, cnt - i, 0.0) && vok;
}

bool have_avx2() {
  static const bool h = __builtin_cpu_supports("avx2");
  return h;
}

}  // namespace

// false if any value is not exactly representable under the storage rule
// (int16: |v| <= 32767 integral; int32: |v| < 2^29 integral; fp32: exact, finite)
__attribute__((visibility("hidden"))) bool narrow_to_i16(const double* src, int16_t* dst, size_t cnt) {
  return have_avx2() ? narrow_int_avx2<int16_t>(src, dst, cnt, 32767.0)
                     : narrow_scalar<int16_t>(src, dst, cnt, 32767.0);
}
__attribute__((visibility("hidden"))) bool narrow_to_i32(const double* src, int32_t* dst, size_t cnt) {
  return have_avx2() ? narrow_int_avx2<int32_t>(src, dst, cnt, 536870911.0)
                     : narrow_scalar<int32_t>(src, dst, cnt, 536870911.0);
}
__attribute__((visibility("hidden"))) bool narrow_to_f32(const double* src, float* dst, size_t cnt) {
  return have_avx2() ? narrow_f32_avx2(src, dst, cnt) : narrow_scalar<float>(src, dst, cnt, 0.0);
}

}  // namespace lsapgpu
