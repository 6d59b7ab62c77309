// tools/issue_bench.cu -- what limits the tensor-pipe utilisation of k_oz_gemm's MMA issue
// (development tool, not part of the product).  One CTA per SM, 192 threads like
// k_oz_gemm, operands resident in SMEM (random bytes, no TMA), the s = 9 / NC = 48 window
// issue sequence of k_oz_gemm (ascending or interleaved slice order), with toggles:
//   bit 0 (1)  : per-A-tile mbarrier round trip: the issuer waits a_full[slot] (made ready
//                by a "producer" warp after the slot's commit, as the TMA producer would)
//   bit 1 (2)  : the 4 "epilogue" warps poll an mbarrier (try_wait loop) the whole time
//   bit 2 (4)  : interleaved slice order (1, s, 2, s-1, ...)
//   bit 3 (8)  : issuer = one lane (else elect.sync per tile)
//   bit 4 (16) : producer uses nanosleep backoff in its wait
//   bit 5 (32) : epilogue polls with nanosleep backoff
//   bit 6 (64) : (tile_sync) wait only before even tiles (stages of two slices)
//   bit 7 (128): two issuer warps (5 and 0) taking alternate tiles (elect per tile)
//   bit 8 (256): issuer waits with mbarrier.test_wait spin instead of try_wait
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/issue_bench tools/issue_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2306_11975_b200/csrc/ptx.cuh"

using namespace ozimmu;
constexpr int S = 9, NC = 48, KKB = 128, STAGES = 7;

__device__ __forceinline__ bool try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                 "selp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(ptx::smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void wait_test(uint64_t *bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                     "selp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(ptx::smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void wait_backoff(uint64_t *bar, uint32_t parity) {
    while (!try_wait(bar, parity)) __nanosleep(64);
}

__device__ __forceinline__ int slice_p(int i, bool inter) {
    return !inter ? i + 1 : ((i & 1) == 0 ? i / 2 + 1 : S - i / 2);
}

__global__ void __launch_bounds__(192, 1) k_issue(int kblocks, int flags, long long *cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t a_full[STAGES], a_empty[STAGES], done_bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (STAGES * 16384 + 2 * S * NC * KKB) / 16; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 97u;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        reinterpret_cast<int4 *>(smem)[i] = make_int4(h, h * 3u + 1u, h * 7u + 5u, h ^ 0xdeadbeefu);
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) { ptx::mbar_init(&a_full[i], 1); ptx::mbar_init(&a_empty[i], 1); }
        ptx::mbar_init(&done_bar, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) { ptx::tmem_alloc(&tslot, 512); ptx::tmem_relinquish(); }
    asm volatile("fence.proxy.async.shared::cta;");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    const bool tile_sync = flags & 1, epi_poll = flags & 2, inter = flags & 4, one_lane = flags & 8;
    const uint32_t smA = ptx::smem_u32(smem), smB = smA + STAGES * 16384;
    if (warp == 4) {  // producer: re-arm a_full[slot] once the slot's MMAs committed
        if (tile_sync && lane == 0) {
            int as = 0; uint32_t aph = 0;
            const long long total = (long long)kblocks * S;
            for (long long t = 0; t < total; ++t) {
                if (flags & 16) wait_backoff(&a_empty[as], aph ^ 1);
                else ptx::mbar_wait(&a_empty[as], aph ^ 1);
                ptx::mbar_arrive(&a_full[as]);
                if (++as == STAGES) { as = 0; aph ^= 1; }
            }
        }
    } else if (warp == 5) {
        constexpr int kMaxBlk = 256 / NC;
        auto issue = [&](int p, uint64_t ad, uint64_t bd) {
            const int L = S + 1 - p;
            for (int j0 = 0; j0 < L; j0 += kMaxBlk) {
                const int nbk = (L - j0) < kMaxBlk ? (L - j0) : kMaxBlk;
                ptx::mma_i8(tmem + (uint32_t)(j0 * NC), ad, bd + (uint64_t)((j0 * NC * KKB) >> 4),
                            ptx::idesc_i8(128, (uint32_t)(nbk * NC)), 1u);
            }
        };
        const uint64_t adesc_base = ptx::smem_desc_kmajor<KKB>(smA);
        const uint64_t bdesc0 = ptx::smem_desc_kmajor<KKB>(smB);
        long long t0 = clock64();
        if (one_lane) {
            if (lane == 0) {
                int as = 0; uint32_t aph = 0;
                for (int kb = 0; kb < kblocks; ++kb) {
#pragma unroll
                    for (int i = 0; i < S; ++i) {
                        const int p = slice_p(i, inter);
                        if (tile_sync) ptx::mbar_wait(&a_full[as], aph);
                        ptx::tc_fence_after();
                        const uint64_t ad = adesc_base + (uint64_t)((as * 16384) >> 4);
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            issue(p, ad + ks * 2, bdesc0 + (uint64_t)(((p - 1) * NC * KKB + ks * 32) >> 4));
                        ptx::mma_commit(&a_empty[as]);
                        if (++as == STAGES) { as = 0; aph ^= 1; }
                    }
                }
                ptx::mma_commit(&done_bar);
            }
            __syncwarp();
        } else {
            int as = 0; uint32_t aph = 0;
            const bool two = flags & 128;
            for (int kb = 0; kb < kblocks; ++kb) {
#pragma unroll
                for (int i = 0; i < S; ++i) {
                    const int p = slice_p(i, inter);
                    const bool mine = !two || (((kb * S + i) & 1) == 0);
                    if (tile_sync && mine && (!(flags & 64) || (i & 1) == 0)) {
                        if (flags & 256) wait_test(&a_full[as], aph);
                        else ptx::mbar_wait(&a_full[as], aph);
                    }
                    ptx::tc_fence_after();
                    if (mine && ptx::elect_one()) {
                        const uint64_t ad = adesc_base + (uint64_t)((as * 16384) >> 4);
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            issue(p, ad + ks * 2, bdesc0 + (uint64_t)(((p - 1) * NC * KKB + ks * 32) >> 4));
                        ptx::mma_commit(&a_empty[as]);
                    }
                    __syncwarp();
                    if (++as == STAGES) { as = 0; aph ^= 1; }
                }
            }
            if (ptx::elect_one()) ptx::mma_commit(&done_bar);
            __syncwarp();
        }
        ptx::mbar_wait(&done_bar, 0);
        long long t1 = clock64();
        if (lane == 0) cycles[blockIdx.x] = t1 - t0;
    } else if (warp == 0 && (flags & 128)) {  // second issuer: odd tiles
        constexpr int kMaxBlk = 256 / NC;
        auto issue = [&](int p, uint64_t ad, uint64_t bd) {
            const int L = S + 1 - p;
            for (int j0 = 0; j0 < L; j0 += kMaxBlk) {
                const int nbk = (L - j0) < kMaxBlk ? (L - j0) : kMaxBlk;
                ptx::mma_i8(tmem + (uint32_t)(j0 * NC), ad, bd + (uint64_t)((j0 * NC * KKB) >> 4),
                            ptx::idesc_i8(128, (uint32_t)(nbk * NC)), 1u);
            }
        };
        const uint64_t adesc_base = ptx::smem_desc_kmajor<KKB>(smA);
        const uint64_t bdesc0 = ptx::smem_desc_kmajor<KKB>(smB);
        int as = 0; uint32_t aph = 0;
        for (int kb = 0; kb < kblocks; ++kb) {
#pragma unroll
            for (int i = 0; i < S; ++i) {
                const int p = slice_p(i, inter);
                const bool mine = ((kb * S + i) & 1) == 1;
                if (tile_sync && mine) ptx::mbar_wait(&a_full[as], aph);
                ptx::tc_fence_after();
                if (mine && ptx::elect_one()) {
                    const uint64_t ad = adesc_base + (uint64_t)((as * 16384) >> 4);
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks)
                        issue(p, ad + ks * 2, bdesc0 + (uint64_t)(((p - 1) * NC * KKB + ks * 32) >> 4));
                    ptx::mma_commit(&a_empty[as]);
                }
                __syncwarp();
                if (++as == STAGES) { as = 0; aph ^= 1; }
            }
        }
    } else {  // "epilogue" warps
        if (epi_poll) {
            if (flags & 32) wait_backoff(&done_bar, 0);
            else ptx::mbar_wait(&done_bar, 0);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long *d_cyc;
    cudaMalloc(&d_cyc, sms * sizeof(long long));
    const int smem = STAGES * 16384 + 2 * S * NC * KKB + 1024;
    cudaFuncSetAttribute(k_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int kblocks = 2000;
    const int flag_sets[] = {0, 1, 5, 1 | 64, 5 | 64, 1 | 128, 5 | 128, 1 | 256, 1 | 16, 3, 0 | 128};
    for (int flags : flag_sets) {
        k_issue<<<sms, 192, smem>>>(kblocks, flags, d_cyc);
        cudaError_t err = cudaDeviceSynchronize();
        long long cyc[1024];
        cudaMemcpy(cyc, d_cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < sms; ++i) avg += cyc[i];
        avg /= sms;
        const double macs = (double)kblocks * 4 * 128.0 * 32 * (S * (S + 1) / 2) * NC;
        printf("flags=%2d tile_sync=%d epi_poll=%d inter=%d one_lane=%d prod_backoff=%d epi_backoff=%d  %s  MAC/clk/SM=%.0f  util=%.3f\n",
               flags, flags & 1, (flags >> 1) & 1, (flags >> 2) & 1, (flags >> 3) & 1, (flags >> 4) & 1,
               (flags >> 5) & 1, cudaGetErrorString(err), macs / avg, macs / avg / 8192);
    }
    return 0;
}
