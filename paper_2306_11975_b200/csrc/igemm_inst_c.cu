// igemm_inst_c.cu -- explicit instantiations of the fused GEMM for s = 13..20.
#include "igemm_kernel.cuh"

namespace ozimmu {
namespace gemm_detail {
template cudaError_t launch_t<13>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<14>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<15>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<16>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<17>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<18>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<19>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
template cudaError_t launch_t<20>(const GemmArgs &, const GemmPlan &, EpiMode, cudaStream_t);
}  // namespace gemm_detail
}  // namespace ozimmu
