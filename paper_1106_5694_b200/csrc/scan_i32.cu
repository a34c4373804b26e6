// Pair-scan instantiations for int32_t storage, key mode 1: the streaming
// kernel (scan_kernel.cuh) and the resident-state kernel (scan_resident.cuh).
#include "scan_resident.cuh"

namespace lsapgpu {
template cudaError_t launch_scan_typed<int32_t, 1>(const DevState&, const ScanPlan&, int, cudaStream_t);
template cudaError_t launch_scan_res_typed<int32_t, 1>(const DevState&, const ScanPlan&, int, cudaStream_t);
}  // namespace lsapgpu
