// Quantized-filter pair scan (scan_filter.cuh), every storage type.
#include "scan_filter.cuh"

namespace lsapgpu {
template cudaError_t launch_scan_filter_typed<int16_t>(const DevState&, const ScanPlan&, int, cudaStream_t);
template cudaError_t launch_scan_filter_typed<int32_t>(const DevState&, const ScanPlan&, int, cudaStream_t);
template cudaError_t launch_scan_filter_typed<float>(const DevState&, const ScanPlan&, int, cudaStream_t);
template cudaError_t launch_scan_filter_typed<double>(const DevState&, const ScanPlan&, int, cudaStream_t);
}  // namespace lsapgpu
