// Pair-scan instantiations for int16_t storage, key mode 0: the streaming
// kernel (scan_kernel.cuh) and the resident-state kernel (scan_resident.cuh).
#include "scan_resident.cuh"

namespace lsapgpu {
template cudaError_t launch_scan_typed<int16_t, 0>(const DevState&, const ScanPlan&, int, cudaStream_t);
template cudaError_t launch_scan_res_typed<int16_t, 0>(const DevState&, const ScanPlan&, int, cudaStream_t);
}  // namespace lsapgpu
