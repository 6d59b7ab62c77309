// igemm_inst_e.cu -- explicit instantiations of the fused GEMM with N_c = 32 for s = 1..10
// (small problems, plan_gemm picks them when the default tiles fill only a few waves).
#include "igemm_kernel.cuh"

namespace ozimmu {
namespace gemm_detail {
template cudaError_t launch_t<1, 32>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<2, 32>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<3, 32>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<4, 32>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<5, 32>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<6, 32>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<7, 32>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<8, 32>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<9, 32>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<10, 32>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
}  // namespace gemm_detail
}  // namespace ozimmu
