// Pair-scan instantiations for float storage, key mode 2: the streaming
// kernel (scan_kernel.cuh) and the resident-state kernel (scan_resident.cuh).
#include "scan_resident.cuh"

namespace lsapgpu {
template cudaError_t launch_scan_typed<float, 2>(const DevState&, const ScanPlan&, int, cudaStream_t);
template cudaError_t launch_scan_res_typed<float, 2>(const DevState&, const ScanPlan&, int, cudaStream_t);
}  // namespace lsapgpu
