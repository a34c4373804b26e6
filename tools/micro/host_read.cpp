// host_read.cpp -- the host-side roofline of the pageable upload: how fast
// can T threads of this box READ an 800 MB fp64 matrix (the C3 instance) at
// all?  Prints, per thread count, the read-only bandwidth (AVX2 sum of every
// entry) and a read + 2-byte write pass (the int16 narrowing's traffic
// shape, streaming stores into a separate buffer).
//   g++ -O2 -mavx2 -pthread tools/micro/host_read.cpp -o tools/micro/host_read
//   ./tools/micro/host_read [n=10000]
#include <immintrin.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

// the library's own exact narrowing (host_narrow.cpp), timed in place
#include "../../paper_1106_5694_b200/csrc/host_narrow.cpp"

static double sum_slice(const double* p, size_t cnt) {
  __m256d a0 = _mm256_setzero_pd(), a1 = a0, a2 = a0, a3 = a0;
  size_t i = 0;
  for (; i + 16 <= cnt; i += 16) {
    a0 = _mm256_add_pd(a0, _mm256_loadu_pd(p + i));
    a1 = _mm256_add_pd(a1, _mm256_loadu_pd(p + i + 4));
    a2 = _mm256_add_pd(a2, _mm256_loadu_pd(p + i + 8));
    a3 = _mm256_add_pd(a3, _mm256_loadu_pd(p + i + 12));
  }
  double t[4];
  _mm256_storeu_pd(t, _mm256_add_pd(_mm256_add_pd(a0, a1), _mm256_add_pd(a2, a3)));
  double s = t[0] + t[1] + t[2] + t[3];
  for (; i < cnt; ++i) s += p[i];
  return s;
}

static void narrow_slice(const double* p, int16_t* q, size_t cnt) {
  size_t i = 0;
  for (; i + 8 <= cnt; i += 8) {
    const __m128i x0 = _mm256_cvttpd_epi32(_mm256_loadu_pd(p + i));
    const __m128i x1 = _mm256_cvttpd_epi32(_mm256_loadu_pd(p + i + 4));
    _mm_stream_si128(reinterpret_cast<__m128i*>(q + i), _mm_packs_epi32(x0, x1));
  }
  _mm_sfence();
  for (; i < cnt; ++i) q[i] = static_cast<int16_t>(p[i]);
}

template <class F>
static double timed(int T, F&& f) {
  double best = 1e30;
  for (int rep = 0; rep < 5; ++rep) {
    std::vector<std::thread> th;
    const auto t0 = std::chrono::steady_clock::now();
    for (int t = 0; t < T; ++t) th.emplace_back([&, t] { f(t); });
    for (auto& x : th) x.join();
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    best = std::min(best, ms);
  }
  return best;
}

int main(int argc, char** argv) {
  const size_t n = argc > 1 ? std::atoll(argv[1]) : 10000;
  const size_t cnt = n * n;
  std::vector<double> a(cnt);
  for (size_t i = 0; i < cnt; ++i) a[i] = static_cast<double>((i * 2654435761u) % 30000);
  int16_t* q = static_cast<int16_t*>(std::aligned_alloc(64, (cnt * 2 + 63) / 64 * 64));
  for (size_t i = 0; i < cnt; ++i) q[i] = 0;
  const int hw = static_cast<int>(std::thread::hardware_concurrency());
  std::printf("hardware_concurrency %d, matrix %zu x %zu fp64 = %.0f MB\n", hw, n, n, cnt * 8 / 1e6);
  volatile double sink = 0;
  for (int T : {1, 2, 4, 8, 12, 16, 24, 32}) {
    if (T > 2 * hw) break;
    std::vector<double> part(T);
    const double ms_r = timed(T, [&](int t) {
      const size_t a0 = cnt * t / T, a1 = cnt * (t + 1) / T;
      part[t] = sum_slice(a.data() + a0, a1 - a0);
    });
    for (double x : part) sink = sink + x;
    const double ms_n = timed(T, [&](int t) {
      const size_t a0 = cnt * t / T / 8 * 8, a1 = t + 1 == T ? cnt : cnt * (t + 1) / T / 8 * 8;
      narrow_slice(a.data() + a0, q + a0, a1 - a0);
    });
    std::vector<int> okv(T);
    const double ms_l = timed(T, [&](int t) {
      const size_t a0 = cnt * t / T / 8 * 8, a1 = t + 1 == T ? cnt : cnt * (t + 1) / T / 8 * 8;
      okv[t] = lsapgpu::narrow_to_i16(a.data() + a0, q + a0, a1 - a0);
    });
    std::printf("threads %2d  read %7.2f ms  %6.1f GB/s   read+narrow-write %7.2f ms  %6.1f GB/s   library narrow %7.2f ms  %6.1f GB/s (ok %d)\n",
                T, ms_r, cnt * 8 / ms_r / 1e6, ms_n, cnt * 8 / ms_n / 1e6, ms_l, cnt * 8 / ms_l / 1e6, okv[0]);
  }
  std::free(q);
  return sink == 12345.0;
}
