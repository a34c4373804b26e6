// Micro-benchmark: HBM -> smem row streaming with cp.async.bulk (one producer
// thread per CTA, a ring of B row slots, consumers only wait + release).
// Measures the rate the pair scan's staging can reach per (row bytes, depth).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(c)); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory"); }
__device__ __forceinline__ void cp(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s32(d)), "l"(s), "r"(n), "r"(s32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(s32(b)), "r"(ph) : "memory");
}

__global__ void stream(const unsigned char* src, int64_t nrows, uint32_t row, int B, int per_cta, int pieces, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)(sm + (size_t)B * row);
  uint64_t* empty = full + 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) { for (int k = 0; k < B; ++k) { init(&full[k], 1); init(&empty[k], NW); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  unsigned long long acc = 0;
  if (warp == NW) {
    if (lane == 0)
      for (int q = 0; q < per_cta; ++q) {
        const int b = q % B;
        if (q >= B) wait(&empty[b], ((q / B) - 1) & 1);
        const uint64_t r = (uint64_t)(blockIdx.x * 7919ull + q * 104729ull) % nrows;
        expect(&full[b], row);
        const uint32_t piece = row / pieces;
        for (int k = 0; k < pieces; ++k) cp(sm + (size_t)b * row + k * piece, src + r * row + k * piece, piece, &full[b]);
      }
  } else {
    for (int q = 0; q < per_cta; ++q) {
      const int b = q % B;
      wait(&full[b], (q / B) & 1);
      acc += sm[(size_t)b * row + threadIdx.x * 4];
      __syncwarp();
      if (lane == 0) arrive(&empty[b]);
    }
  }
  if (acc == 123456789ull) *sink = acc;
}

int main() {
  const size_t bytes = 4ull << 30;
  unsigned char* src; cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (uint32_t row : {5120u, 10240u, 20480u, 40960u})
    for (int B : {2, 3, 4, 6, 8}) for (int pieces : {1, 4}) {
      if ((size_t)B * row > 200 * 1024) continue;
      const int64_t nrows = bytes / row;
      const int per_cta = (int)((2ull << 30) / row / sms);
      const size_t smem = (size_t)B * row + 256;
      for (int it = 0; it < 2; ++it) {
        cudaEventRecord(e0);
        stream<<<sms, 512, smem>>>(src, nrows, row, B, per_cta, pieces, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double gb = (double)per_cta * sms * row / 1e9;
      printf("row %6u B %d pieces %d in-flight/SM %6.0f KB : %7.1f GB/s  %s\n", row, B, pieces, (B - 1) * row / 1024.0, gb / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
