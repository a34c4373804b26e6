// Microbenchmark: cost of grid-wide (cooperative) and cluster barriers on B200.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void grid_sync_loop(int iters, int* sink) {
  cg::grid_group g = cg::this_grid();
  int acc = 0;
  for (int k = 0; k < iters; ++k) { acc += k; g.sync(); }
  if (acc == -1) *sink = acc;
}

__global__ void __cluster_dims__(16, 1, 1) cluster_sync_loop16(int iters, int* sink) {
  cg::cluster_group c = cg::this_cluster();
  int acc = 0;
  for (int k = 0; k < iters; ++k) { acc += k; c.sync(); }
  if (acc == -1) *sink = acc;
}
__global__ void __cluster_dims__(8, 1, 1) cluster_sync_loop8(int iters, int* sink) {
  cg::cluster_group c = cg::this_cluster();
  int acc = 0;
  for (int k = 0; k < iters; ++k) { acc += k; c.sync(); }
  if (acc == -1) *sink = acc;
}

__global__ void empty_kernel(int* sink) { if (threadIdx.x == 12345) *sink = 1; }

int main() {
  int* sink; cudaMalloc(&sink, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int bpsm : {1, 2}) for (int th : {256, 1024}) {
    if (bpsm * th > 2048) continue;
    int iters = 2000;
    void* args[] = {&iters, &sink};
    dim3 grid(sms * bpsm), block(th);
    cudaLaunchCooperativeKernel((void*)grid_sync_loop, grid, block, args, 0, 0);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)grid_sync_loop, grid, block, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid.sync  grid=%d block=%d : %.3f us/sync (%s)\n", sms*bpsm, th, ms*1e3/iters, cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(cluster_sync_loop16, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int th : {256, 1024}) {
    int iters = 20000;
    cluster_sync_loop16<<<16, th>>>(iters, sink); cudaDeviceSynchronize();
    cudaEventRecord(a); cluster_sync_loop16<<<16, th>>>(iters, sink); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("cluster16.sync block=%d : %.3f us/sync (%s)\n", th, ms*1e3/iters, cudaGetErrorString(cudaGetLastError()));
    cluster_sync_loop8<<<8, th>>>(iters, sink); cudaDeviceSynchronize();
    cudaEventRecord(a); cluster_sync_loop8<<<8, th>>>(iters, sink); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("cluster8.sync  block=%d : %.3f us/sync (%s)\n", th, ms*1e3/iters, cudaGetErrorString(cudaGetLastError()));
  }
  // graph of back-to-back empty kernels: launch overhead per node
  cudaStream_t s; cudaStreamCreate(&s);
  cudaGraph_t gr; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int k = 0; k < 200; ++k) empty_kernel<<<1, 32, 0, s>>>(sink);
  cudaStreamEndCapture(s, &gr); cudaGraphInstantiate(&ge, gr, 0);
  cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
  cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("graph: %.3f us per dependent empty kernel node\n", ms * 1e3 / 200);
  cudaEventRecord(a, s); for (int k = 0; k < 200; ++k) empty_kernel<<<1, 32, 0, s>>>(sink); cudaEventRecord(b, s); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("stream: %.3f us per dependent empty kernel launch\n", ms * 1e3 / 200);
  return 0;
}
