// tools/launch_probe.cu -- fixed costs of a launch like k_oz_gemm's (development tool):
// empty kernel with 0 / 227 KB dynamic SMEM, with/without a 2-CTA cluster, with a TMEM
// alloc/dealloc; back-to-back launches alternating with a small-SMEM kernel (as the slicing
// kernels do), CUDA-event timed.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2306_11975_b200/csrc/ptx.cuh"
using namespace ozimmu;

__global__ void k_small(int *p) { if (threadIdx.x == 0 && p) p[blockIdx.x] = 1; }
__global__ void __launch_bounds__(224, 1) k_big(int *p, int tmem) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t slot;
    if (tmem) {
        if (threadIdx.x / 32 == 0) { ptx::tmem_alloc(&slot, 512); ptx::tmem_relinquish(); }
        __syncthreads();
        if (threadIdx.x / 32 == 0) ptx::tmem_dealloc(slot, 512);
    }
    if (threadIdx.x == 0 && p) p[blockIdx.x] = (int)(size_t)smem & 1;
}

int main() {
    int *d;
    cudaMalloc(&d, 4096 * sizeof(int));
    cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Cfg { const char *name; int smem; int cl; int tmem; int alt; };
    Cfg cfgs[] = {{"big0_smem", 0, 1, 0, 0}, {"big227_smem", 220 * 1024, 1, 0, 0},
                  {"big227_alt_small", 220 * 1024, 1, 0, 1}, {"big227_cl2", 220 * 1024, 2, 0, 0},
                  {"big227_cl2_tmem", 220 * 1024, 2, 1, 0}, {"big227_cl2_tmem_alt", 220 * 1024, 2, 1, 1}};
    for (auto &c : cfgs) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            for (int i = 0; i < 200; ++i) {
                if (c.alt) k_small<<<128, 256>>>(d);
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(148);
                cfg.blockDim = dim3(224);
                cfg.dynamicSmemBytes = c.smem;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = c.cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, k_big, d, c.tmem);
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("%-22s %7.2f us per iteration (%s)\n", c.name, ms * 1e3 / 200,
                            cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
