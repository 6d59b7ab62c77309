// igemm_inst_b.cu -- explicit instantiations of the fused GEMM for s = 9..12.
#include "igemm_kernel.cuh"

namespace ozimmu {
namespace gemm_detail {
template cudaError_t launch_t<9>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<10>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<11>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<12>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
}  // namespace gemm_detail
}  // namespace ozimmu
