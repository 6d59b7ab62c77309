// igemm_inst_a.cu -- explicit instantiations of the fused GEMM for s = 1..8.
#include "igemm_kernel.cuh"

namespace ozimmu {
namespace gemm_detail {
template cudaError_t launch_t<1>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<2>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<3>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<4>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<5>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<6>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<7>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<8>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
}  // namespace gemm_detail
}  // namespace ozimmu
