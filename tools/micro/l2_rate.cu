// Micro-benchmark: L2-hit vs HBM streaming rate into SMs, for TMA bulk
// copies into a shared-memory ring and for plain 16-byte loads.  Sizes the
// position-stream (tau / acur / entries) traffic of the long-row scan, which
// every item re-reads from L2.
#include <cstdio>
#include <cstdint>
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
__global__ void tma_stream(const unsigned char* src, int64_t nrows, uint32_t piece, int B, int per_cta, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)(sm + (size_t)B * piece);
  uint64_t* empty = full + 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) { for (int k = 0; k < B; ++k) { init(&full[k], 1); init(&empty[k], NW); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  unsigned long long acc = 0;
  if (warp == NW) {
    if (lane == 0)
      for (int q = 0; q < per_cta; ++q) {
        const int b = q % B;
        if (q >= B) wait(&empty[b], ((q / B) - 1) & 1);
        expect(&full[b], piece);
        const uint64_t r = (uint64_t)(blockIdx.x * 7919ull + q * 104729ull) % nrows;
        cp(sm + (size_t)b * piece, src + r * piece, piece, &full[b]);
      }
  } else {
    for (int q = 0; q < per_cta; ++q) {
      const int b = q % B;
      wait(&full[b], (q / B) & 1);
      acc += sm[(size_t)b * piece + threadIdx.x * 4];
      __syncwarp();
      if (lane == 0) arrive(&empty[b]);
    }
  }
  if (acc == 123456789ull) *sink = acc;
}
__global__ void ldg_stream(const uint4* src, int64_t nvec, int64_t per_thread, unsigned long long* sink) {
  uint32_t acc = 0;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
#pragma unroll 8
  for (int64_t k = 0; k < per_thread; ++k) {
    const uint4 v = __ldcg(src + (i % nvec));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
    i += stride;
  }
  if (acc == 0x12345678u) *sink = acc;
}
int main() {
  const size_t bytes = 4ull << 30;
  unsigned char* src; cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (size_t foot : {16ull << 20, 48ull << 20, 96ull << 20, 4ull << 30})
    for (uint32_t piece : {8192u, 16384u, 32768u})
      for (int B : {4, 8}) {
        const size_t smem = (size_t)B * piece + 512;
        if (smem > 200 * 1024) continue;
        const int64_t nrows = foot / piece;
        const int per_cta = (int)((8ull << 30) / piece / sms);
        float ms = 0;
        for (int it = 0; it < 3; ++it) {
          cudaEventRecord(e0);
          tma_stream<<<sms, 512, smem>>>(src, nrows, piece, B, per_cta, sink);
          cudaEventRecord(e1); cudaEventSynchronize(e1);
          cudaEventElapsedTime(&ms, e0, e1);
        }
        const double gb = (double)per_cta * sms * piece / 1e9;
        printf("tma  foot %5zu MB piece %6u B %d : %8.1f GB/s %s\n", foot >> 20, piece, B, gb / (ms * 1e-3),
               cudaGetErrorString(cudaGetLastError()));
        fflush(stdout);
      }
  for (size_t foot : {16ull << 20, 48ull << 20, 96ull << 20, 4ull << 30})
    for (int per_sm : {4, 8}) {
      const int grid = sms * per_sm;
      const int64_t nvec = foot / 16;
      const int64_t per_thread = (int64_t)((8ull << 30) / 16 / ((size_t)grid * 256));
      float ms = 0;
      for (int it = 0; it < 3; ++it) {
        cudaEventRecord(e0);
        ldg_stream<<<grid, 256>>>((const uint4*)src, nvec, per_thread, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      const double gb = (double)per_thread * grid * 256 * 16 / 1e9;
      printf("ldg  foot %5zu MB ctas/SM %d : %8.1f GB/s %s\n", foot >> 20, per_sm, gb / (ms * 1e-3),
             cudaGetErrorString(cudaGetLastError()));
      fflush(stdout);
    }
  return 0;
}
