// graph_rebuild_memcheck.cu -- minimal reproducer for a compute-sanitizer
// memcheck report seen on the solver's graph mode: a kernel inside a
// conditional WHILE node reads a 248-byte control block, the graph is
// destroyed and rebuilt, and memcheck reports the (valid) read as "out of
// bounds ... inside the nearest allocation" in the rebuilt graph.  Nothing
// but the graph API and one cudaMalloc is involved.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o graph_rebuild_memcheck graph_rebuild_memcheck.cu
//   compute-sanitizer --tool memcheck ./graph_rebuild_memcheck [cluster]
#include <cstdio>
#include <cstring>

#include <cuda_runtime.h>

struct Ctl {
  int iter;
  int sum;
  int pad[60];
};

__global__ void body(Ctl* c, cudaGraphConditionalHandle h) {
  const int v = c->iter;  // every thread reads the control block
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    c->sum += v;
    c->iter = v + 1;
    if (v + 1 >= 3) cudaGraphSetConditional(h, 0);
  }
}

__global__ void __cluster_dims__(2, 1, 1) body_cluster(Ctl* c, cudaGraphConditionalHandle h) {
  const int v = c->iter;
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    c->sum += v;
    c->iter = v + 1;
    if (v + 1 >= 3) cudaGraphSetConditional(h, 0);
  }
}

int main(int argc, char** argv) {
  const bool cluster = argc > 1 && std::strcmp(argv[1], "cluster") == 0;
  Ctl* c = nullptr;
  cudaMalloc(&c, sizeof(Ctl));
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int rep = 0; rep < 3; ++rep) {
    cudaGraph_t g;
    cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    cudaGraphAddNode(&node, g, nullptr, 0, &p);
    cudaGraph_t bg = p.conditional.phGraph_out[0];
    cudaStreamBeginCaptureToGraph(s, bg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (cluster)
      body_cluster<<<2, 64, 0, s>>>(c, h);
    else
      body<<<2, 64, 0, s>>>(c, h);
    cudaStreamEndCapture(s, &bg);
    cudaGraphExec_t e;
    cudaGraphInstantiate(&e, g, 0);
    cudaMemsetAsync(c, 0, sizeof(Ctl), s);
    cudaGraphLaunch(e, s);
    cudaStreamSynchronize(s);
    Ctl h_c;
    cudaMemcpy(&h_c, c, sizeof(Ctl), cudaMemcpyDeviceToHost);
    std::printf("build %d: iter %d sum %d (%s)\n", rep, h_c.iter, h_c.sum, cudaGetErrorString(cudaGetLastError()));
    cudaGraphExecDestroy(e);
    cudaGraphDestroy(g);
  }
  cudaFree(c);
  return 0;
}
