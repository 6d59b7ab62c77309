// igemm_inst_d.cu -- explicit instantiations of the fused GEMM for s = 21..32.
#include "igemm_kernel.cuh"

namespace ozimmu {
namespace gemm_detail {
template cudaError_t launch_t<21>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<22>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<23>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<24>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<25>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<26>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<27>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<28>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<29>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<30>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<31>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<32>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
}  // namespace gemm_detail
}  // namespace ozimmu
