// Micro-benchmark: TMA bulk-copy rate with copies issued by 1 or several lanes
// of a producer warp (does the per-SM copy rate scale with issuing lanes?).
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
// each stage = `pieces` copies of `piece` bytes, issued by `lanes` lanes
__global__ void stream(const unsigned char* src, int64_t nrows, uint32_t piece, int pieces, int lanes, int B, int per_cta, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const uint32_t stage = piece * pieces;
  uint64_t* full = (uint64_t*)(sm + (size_t)B * stage);
  uint64_t* empty = full + 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) { for (int k = 0; k < B; ++k) { init(&full[k], 1); init(&empty[k], NW); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  unsigned long long acc = 0;
  if (warp == NW) {
    for (int q = 0; q < per_cta; ++q) {
      const int b = q % B;
      if (q >= B) wait(&empty[b], ((q / B) - 1) & 1);
      if (lane == 0) expect(&full[b], stage);
      __syncwarp();
      for (int k = lane; lane < lanes && k < pieces; k += lanes) {
        const uint64_t r = (uint64_t)(blockIdx.x * 7919ull + q * 104729ull + k * 31ull) % nrows;
        cp(sm + (size_t)b * stage + (size_t)k * piece, src + r * piece, piece, &full[b]);
      }
      __syncwarp();
    }
  } else {
    for (int q = 0; q < per_cta; ++q) {
      const int b = q % B;
      wait(&full[b], (q / B) & 1);
      acc += sm[(size_t)b * stage + threadIdx.x * 4];
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
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (uint32_t piece : {4096u, 8192u, 16384u, 32768u})
    for (int lanes : {1, 4, 32}) for (int B : {2, 4}) {
      const int pieces = (int)(49152 / piece);  // 48 KB stages
      const size_t smem = (size_t)B * piece * pieces + 256;
      if (smem > 200 * 1024) continue;
      const int64_t nrows = bytes / piece;
      const int per_cta = (int)((2ull << 30) / (piece * pieces) / sms);
      for (int it = 0; it < 2; ++it) {
        cudaEventRecord(e0);
        stream<<<sms, 512, smem>>>(src, nrows, piece, pieces, lanes, B, per_cta, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double gb = (double)per_cta * sms * piece * pieces / 1e9;
      fflush(stdout);
      printf("piece %6u x%2d lanes %2d B %d : %7.1f GB/s  %.2f Mcopies/s/SM %s\n", piece, pieces, lanes, B, gb / (ms * 1e-3),
             (double)per_cta * pieces / (ms * 1e-3) / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
