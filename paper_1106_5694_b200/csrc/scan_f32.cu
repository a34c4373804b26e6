// Pair-scan instantiations for float storage, key mode 2: the streaming
// kernel (scan_kernel.cuh) and the resident-state kernel (scan_resident.cuh).
#include "scan_big.cuh"
#include "scan_cluster.cuh"

namespace lsapgpu {
template cudaError_t launch_scan_typed<float, 2>(const DevState&, const ScanPlan&, int, cudaStream_t);
template cudaError_t launch_scan_res_typed<float, 2>(const DevState&, const ScanPlan&, int, cudaStream_t);
template cudaError_t launch_scan_big_typed<float, 2>(const DevState&, const ScanPlan&, int, cudaStream_t);
template cudaError_t launch_scan_cl_typed<float, 2>(const DevState&, const ScanPlan&, int, cudaStream_t);
}  // namespace lsapgpu

namespace lsapgpu {
namespace {
template <int CS>
int cl_active_t(size_t smem) {
  auto k = scan_detail::pair_scan_cl_kernel<float, scan_detail::kFloat, CS>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  if (CS > 8 && cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS);
  cfg.blockDim = dim3(scan_detail::kClThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, k, &cfg) != cudaSuccess) clusters = 0;
  cudaGetLastError();
  return clusters;
}
}  // namespace

// Clusters of CS cluster-kernel CTAs with `smem` dynamic bytes resident at once.
int cl_active_clusters(int CS, size_t smem) {
  switch (CS) {
    case 2: return cl_active_t<2>(smem);
    case 4: return cl_active_t<4>(smem);
    default: return 0;
  }
}
}  // namespace lsapgpu
