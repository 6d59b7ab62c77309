// tools/mma_bench.cu -- microbenchmark of tcgen05.mma.kind::i8 issue/throughput for the
// N mixes the Ozaki kernel uses (development tool, not part of the product).
// One CTA per SM, operands resident in SMEM (zeros), one thread issues MMAs back to back.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2306_11975_b200/csrc/ptx.cuh"

using namespace ozimmu;

__global__ void __launch_bounds__(128, 1) k_bench(const int *ns, int nn, int rounds, long long *cycles,
                                                  int mode) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32;
    // mode 0/1: zeros; mode >= 2: pseudo-random bytes (the Ozaki digit planes are ~uniform
    // in [-127, 127], which toggles the MAC array and changes power, not cycles)
    for (int i = threadIdx.x; i < 168 * 1024 / 16; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 97u;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        reinterpret_cast<int4 *>(smem)[i] = mode >= 2 ? make_int4(h, h * 3u + 1u, h * 7u + 5u, h ^ 0xdeadbeefu)
                                                   : make_int4(0, 0, 0, 0);
    }
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    if (warp == 0) { ptx::tmem_alloc(&tslot, 512); ptx::tmem_relinquish(); }
    asm volatile("fence.proxy.async.shared::cta;");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 1) {
        if (ptx::elect_one()) {
            // mode 3: A rotates over a 7-tile ring (16 KB each) and B sits after it, with the
            // s = 9 window offsets (as in k_oz_gemm); modes 0-2: fixed addresses
            const uint32_t a0 = ptx::smem_u32(smem);
            const uint32_t b = mode == 3 ? a0 + 7 * 16384 : a0 + 16384;
            long long t0 = clock64();
            for (int r = 0; r < rounds; ++r) {
                for (int i = 0; i < nn; ++i) {
                    const int N = ns[i];
                    for (int ks = 0; ks < 4; ++ks) {
                        const uint32_t a = mode == 3 ? a0 + (uint32_t)(((r * nn + i) % 7) * 16384) : a0;
                        const uint32_t boff = mode == 3 ? (uint32_t)((i % 9) * 48 * 128) : 0u;
                        uint64_t ad = ptx::smem_desc_kmajor<128>(a + ks * 32);
                        uint64_t bd = ptx::smem_desc_kmajor<128>(b + boff + ks * 32);
                        uint32_t col = mode == 0 ? 0u : (uint32_t)((i % 2) * 256);
                        ptx::mma_i8(tmem + col, ad, bd, ptx::idesc_i8(128, N), 1u);
                    }
                }
            }
            ptx::mma_commit(&bar);
            ptx::mbar_wait(&bar, 0);
            long long t1 = clock64();
            if (blockIdx.x == 0) cycles[0] = t1 - t0;
        }
        __syncwarp();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

int main() {
    std::vector<std::pair<const char *, std::vector<int>>> mixes = {
        {"N256x8", {256, 256, 256, 256, 256, 256, 256, 256}},
        {"N128x8", {128, 128, 128, 128, 128, 128, 128, 128}},
        {"N64x8", {64, 64, 64, 64, 64, 64, 64, 64}},
        {"N48x8", {48, 48, 48, 48, 48, 48, 48, 48}},
        {"s9nc48", {240, 192, 240, 144, 240, 96, 240, 48, 240, 192, 144, 96, 48}},
        {"s9bal", {240, 192, 192, 192, 192, 144, 144, 144, 240, 192, 144, 96, 48}},
        {"N96x8", {96, 96, 96, 96, 96, 96, 96, 96}},
        {"N144x8", {144, 144, 144, 144, 144, 144, 144, 144}},
        {"s9nc32", {256, 32, 256, 224, 192, 160, 128, 96, 64, 32}},
        {"s7nc64", {256, 192, 256, 128, 256, 64, 256, 192, 128, 64}},
    };
    int *d_ns;
    long long *d_cyc;
    cudaMalloc(&d_ns, 64 * sizeof(int));
    cudaMalloc(&d_cyc, sizeof(long long));
    cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int mode = 2; mode < 4; ++mode)
        for (auto &mx : mixes) {
            cudaMemcpy(d_ns, mx.second.data(), mx.second.size() * sizeof(int), cudaMemcpyHostToDevice);
            long long ntot = 0;
            for (int n : mx.second) ntot += n;
            const int rounds = 2000;
            k_bench<<<sms, 128, 200 * 1024>>>(d_ns, (int)mx.second.size(), rounds, d_cyc, mode);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k_bench<<<sms, 128, 200 * 1024>>>(d_ns, (int)mx.second.size(), rounds, d_cyc, mode);
            cudaEventRecord(e1);
            cudaError_t err = cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            long long cyc = 0;
            cudaMemcpy(&cyc, d_cyc, sizeof(cyc), cudaMemcpyDeviceToHost);
            double macs = (double)rounds * 4 * 128.0 * 32 * ntot;  // per SM
            printf("%-8s mode=%d  %s  MAC/clk/SM=%.0f (peak 8192)  chip TOPS=%.0f  clk=%.0f MHz\n",
                   mx.first, mode, cudaGetErrorString(err), macs / cyc, 2 * macs * sms / (ms * 1e-3) / 1e12,
                   cyc / (ms * 1e-3) / 1e6);
        }
    return 0;
}
