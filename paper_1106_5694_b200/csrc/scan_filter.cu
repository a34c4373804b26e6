// Quantized-filter pair scan (scan_filter.cuh): float storage.
#include "scan_filter.cuh"

namespace lsapgpu {
template cudaError_t launch_scan_filter_typed<float>(const DevState&, const ScanPlan&, int, cudaStream_t);
}  // namespace lsapgpu
