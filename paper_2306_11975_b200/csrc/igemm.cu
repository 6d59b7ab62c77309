// igemm.cu -- A4 + A5 of the Ozaki scheme on sm_100a in ONE persistent kernel:
//   INT8 x INT8 -> INT32 slice-pair GEMMs on tcgen05 tensor cores (Alg. 3 line 6)
//   + the FP64 accumulation / scaling epilogue (Alg. 3 line 7),
// replacing the paper's cublasGemmEx-per-pair + separate FP64 accumulation kernel
// (whose accumulation pass was HBM-bound at ~90% of DRAM BW).
//
// Design:
//  * Output tile = 128 rows x NC columns of C, one CTA per SM (persistent, grouped raster,
//    soft per-wave grid barrier so CTAs sharing operands stream K through L2 together).
//  * K is processed in k-blocks of 128 bytes (one 128B-swizzle row).  Per k-block ONE 3-D
//    TMA box brings all s B-slice tiles of the NC columns (B planes are stored in reversed
//    slice order q -> s-q) into the B ring, and the s A-slice tiles (128 x 128 B each) flow
//    one by one through a deeper A ring.
//  * Operand sharing: for A-slice p, its partners B^(1..s+1-p) are the contiguous
//    "window" of reversed B blocks [p-1, s-1]; tcgen05.mma instructions with
//    N = (s+1-p) NC (split into <= 256-wide pieces) multiply A^(p) by the whole window,
//    and window block j lands in TMEM column block j, which always holds level g = s+1-j.
//    So TMEM accumulates the exact per-level sums L_g directly: each A and B slice tile
//    is loaded once per k-block and every pair i+j <= s+1 is covered.
//  * INT32 budget: a level has <= s pairs, so K is processed in chunks with
//    s * k_chunk * (2^w-1)^2 <= 2^31-1; between chunks the epilogue drains TMEM into exact
//    int64 partial sums (per-CTA global scratch).
//  * Epilogue (4 warps, TMEM lane quarter = warp % 4): L_g -> FP64 in the canonical
//    order g = s+1 .. 2 (reading A6), ldexp by E_A+E_B (A7), alpha/beta (A8), NaN rows (A9),
//    coalesced column-major stores of C.
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "internal.h"
#include "ptx.cuh"

namespace ozimmu {
namespace {

constexpr int kThreads = 192;  // warps 0-3 epilogue, 4 TMA producer, 5 MMA issuer
constexpr int kBlockM = 128;
constexpr int kKB = 128;       // K bytes per k-block = one 128B swizzle row
constexpr int kGroupM = 8;     // grouped raster: 8 row-blocks per group

struct KParams {
    int64_t m, n, k_pad;
    int s, w;
    int64_t num_k_blocks, chunk_blocks;
    int k_chunks;
    int64_t tiles_m, tiles_n, num_tiles;
    int a_stages, b_stages;
    uint32_t a_stage_bytes, b_stage_bytes;
    uint32_t tmem_cols;
    int mode;
    double alpha, beta;
    const int32_t *EA, *EB;
    double *C;
    int64_t ldc;
    void *out;
    int64_t *scratch;
    unsigned int *wave_counter;  // soft grid barrier between tile waves (may be null)
    int64_t full_waves;          // waves in which every CTA has a tile
};

__device__ __forceinline__ void tile_coords(int64_t t, const KParams &P, int64_t &mb,
                                            int64_t &nb) {
    const int64_t per_group = (int64_t)kGroupM * P.tiles_n;
    const int64_t g = t / per_group;
    const int64_t r = t % per_group;
    const int64_t gm0 = g * kGroupM;
    int64_t gsz = P.tiles_m - gm0;
    gsz = gsz < kGroupM ? gsz : kGroupM;
    mb = gm0 + r % gsz;
    nb = r / gsz;
}

// 2^e as a double for e in the normal range (exact).
__device__ __forceinline__ double pow2(int e) {
    return __longlong_as_double(static_cast<long long>(1023 + e) << 52);
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned int ld_acquire(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Soft barrier: CTAs of the persistent grid start tile-wave `wave` together, so that the
// CTAs sharing A row-blocks / B column-blocks stream the same K range through L2 at the
// same time.  Bounded wait: never a deadlock if some CTAs are not co-resident.
__device__ __forceinline__ void wave_sync(const KParams &P, int64_t wave) {
    if (!P.wave_counter || wave >= P.full_waves) return;
    atomicAdd(P.wave_counter, 1u);
    const unsigned int target = (unsigned int)((wave + 1) * gridDim.x);
    const uint64_t t0 = globaltimer();
    while (ld_acquire(P.wave_counter) < target) {
        if (globaltimer() - t0 > 200000ull) break;  // 200 us cap
        __nanosleep(256);
    }
}

template <int NC>
__global__ void __launch_bounds__(kThreads, 1)
    k_oz_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const KParams P) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    // [B ring: b_stages x (s x NC x 128)] [A ring: a_stages x (128 x 128)] [barriers]
    uint8_t *smB = smem;
    uint8_t *smA = smem + (size_t)P.b_stages * P.b_stage_bytes;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smA + (size_t)P.a_stages * P.a_stage_bytes);
    uint64_t *b_full = bars;
    uint64_t *b_empty = b_full + P.b_stages;
    uint64_t *a_full = b_empty + P.b_stages;
    uint64_t *a_empty = a_full + P.a_stages;
    uint64_t *tmem_full = a_empty + P.a_stages;
    uint64_t *tmem_empty = tmem_full + 1;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 1);

    const uint32_t warp = ptx::warp_id();
    const uint32_t lane = ptx::lane_id();
    const int s = P.s;

    if (warp == 5 && lane == 0) {
        for (int i = 0; i < P.b_stages; ++i) {
            ptx::mbar_init(&b_full[i], 1);
            ptx::mbar_init(&b_empty[i], 1);
        }
        for (int i = 0; i < P.a_stages; ++i) {
            ptx::mbar_init(&a_full[i], 1);
            ptx::mbar_init(&a_empty[i], 1);
        }
        ptx::mbar_init(tmem_full, 1);
        ptx::mbar_init(tmem_empty, 4 * 32);
        ptx::fence_mbar_init();
        ptx::fence_proxy_async();
    }
    if (warp == 4 && lane == 0) {
        ptx::tma_prefetch_desc(&tmA);
        ptx::tma_prefetch_desc(&tmB);
    }
    if (warp == 0) {
        ptx::tmem_alloc(tmem_slot, P.tmem_cols);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 4) {
        // ===================== TMA producer =====================
        if (ptx::elect_one()) {
            int bs = 0, as = 0;
            uint32_t bph = 0, aph = 0;
            int64_t wave = 0;
            const uint32_t b_tx = (uint32_t)(s * NC * kKB), a_tx = (uint32_t)(kBlockM * kKB);
            for (int64_t t = blockIdx.x; t < P.num_tiles; t += gridDim.x, ++wave) {
                int64_t mb, nb;
                tile_coords(t, P, mb, nb);
                wave_sync(P, wave);
                for (int64_t kb = 0; kb < P.num_k_blocks; ++kb) {
                    ptx::mbar_wait(&b_empty[bs], bph ^ 1);
                    ptx::mbar_arrive_expect_tx(&b_full[bs], b_tx);
                    ptx::tma_load_3d(&tmB, &b_full[bs], smB + (size_t)bs * P.b_stage_bytes,
                                     (int32_t)(kb * kKB), (int32_t)(nb * NC), 0,
                                     ptx::kEvictNormal);
                    if (++bs == P.b_stages) { bs = 0; bph ^= 1; }
                    for (int p = 0; p < s; ++p) {
                        ptx::mbar_wait(&a_empty[as], aph ^ 1);
                        ptx::mbar_arrive_expect_tx(&a_full[as], a_tx);
                        ptx::tma_load_3d(&tmA, &a_full[as], smA + (size_t)as * P.a_stage_bytes,
                                         (int32_t)(kb * kKB), (int32_t)(mb * kBlockM), p,
                                         ptx::kEvictNormal);
                        if (++as == P.a_stages) { as = 0; aph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 5) {
        // ===================== MMA issuer =====================
        constexpr int kMaxBlk = 256 / NC;  // window blocks per instruction (N <= 256)
        int bs = 0, as = 0;
        uint32_t bph = 0, aph = 0;
        uint32_t acc_iter = 0;
        for (int64_t t = blockIdx.x; t < P.num_tiles; t += gridDim.x) {
            for (int c = 0; c < P.k_chunks; ++c, ++acc_iter) {
                ptx::mbar_wait(tmem_empty, (acc_iter & 1) ^ 1);
                ptx::tc_fence_after();
                const int64_t kb0 = (int64_t)c * P.chunk_blocks;
                int64_t kb1 = kb0 + P.chunk_blocks;
                kb1 = kb1 < P.num_k_blocks ? kb1 : P.num_k_blocks;
                for (int64_t kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&b_full[bs], bph);
                    const uint32_t bBase = ptx::smem_u32(smB + (size_t)bs * P.b_stage_bytes);
                    for (int p = 1; p <= s; ++p) {
                        ptx::mbar_wait(&a_full[as], aph);
                        ptx::tc_fence_after();
                        if (ptx::elect_one()) {
                            const uint32_t aBase =
                                ptx::smem_u32(smA + (size_t)as * P.a_stage_bytes);
                            const int L = s + 1 - p;  // window: partners q = 1..L
#pragma unroll
                            for (int ks = 0; ks < kKB / 32; ++ks) {
                                const uint64_t adesc =
                                    ptx::smem_desc_kmajor<kKB>(aBase + (uint32_t)(ks * 32));
                                const uint32_t acc = (kb == kb0 && ks == 0 && p == 1) ? 0u : 1u;
                                for (int j0 = 0; j0 < L; j0 += kMaxBlk) {
                                    const int nbk = (L - j0) < kMaxBlk ? (L - j0) : kMaxBlk;
                                    const uint64_t bdesc = ptx::smem_desc_kmajor<kKB>(
                                        bBase + (uint32_t)((p - 1 + j0) * NC * kKB + ks * 32));
                                    ptx::mma_i8(tmem_base + (uint32_t)(j0 * NC), adesc, bdesc,
                                                ptx::idesc_i8(kBlockM, (uint32_t)(nbk * NC)),
                                                acc);
                                }
                            }
                            ptx::mma_commit(&a_empty[as]);  // A slot free when these finish
                        }
                        __syncwarp();
                        if (++as == P.a_stages) { as = 0; aph ^= 1; }
                    }
                    if (ptx::elect_one()) ptx::mma_commit(&b_empty[bs]);
                    __syncwarp();
                    if (++bs == P.b_stages) { bs = 0; bph ^= 1; }
                }
                if (ptx::elect_one()) ptx::mma_commit(tmem_full);  // chunk accumulated
                __syncwarp();
            }
        }
    } else {
        // ===================== epilogue (warps 0-3) =====================
        const uint32_t row_local = warp * 32 + lane;
        const uint32_t lane_addr = (warp * 32) << 16;
        int64_t *scr = P.scratch ? P.scratch + (int64_t)blockIdx.x * s * NC * kBlockM : nullptr;
        uint32_t acc_iter = 0;
        for (int64_t t = blockIdx.x; t < P.num_tiles; t += gridDim.x) {
            int64_t mb, nb;
            tile_coords(t, P, mb, nb);
            const int64_t row = mb * kBlockM + row_local;
            const bool row_ok = row < P.m;
            const int32_t ea = (P.mode == EPI_DGEMM && row_ok) ? P.EA[row] : 0;
            for (int c = 0; c < P.k_chunks; ++c, ++acc_iter) {
                ptx::mbar_wait(tmem_full, acc_iter & 1);
                ptx::tc_fence_after();
                const bool first = c == 0, last = c == P.k_chunks - 1;
#pragma unroll 1
                for (int cg = 0; cg < NC / 8; ++cg) {
                    double acc[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) acc[i] = 0.0;
#pragma unroll 1
                    for (int j = 0; j < s; ++j) {  // level g = s+1-j, descending g
                        __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge first
                        uint32_t v[8];
                        ptx::tmem_ld_x8(tmem_base + lane_addr + (uint32_t)(j * NC + cg * 8), v);
                        ptx::tmem_ld_wait();
                        int64_t Lg[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) Lg[i] = (int64_t)(int32_t)v[i];
                        if (scr) {
                            int64_t *sp = scr + ((int64_t)(j * NC + cg * 8) * kBlockM) + row_local;
                            if (!first) {
#pragma unroll
                                for (int i = 0; i < 8; ++i) Lg[i] += sp[i * kBlockM];
                            }
                            if (!last) {
#pragma unroll
                                for (int i = 0; i < 8; ++i) sp[i * kBlockM] = Lg[i];
                            }
                        }
                        if (!last) continue;
                        if (P.mode == EPI_DGEMM) {
                            const double sc = pow2(-P.w * (s + 1 - j));
#pragma unroll
                            for (int i = 0; i < 8; ++i)
                                acc[i] = __dadd_rn(acc[i], __dmul_rn((double)Lg[i], sc));
                        } else if (row_ok) {
#pragma unroll
                            for (int i = 0; i < 8; ++i) {
                                const int64_t col = nb * NC + cg * 8 + i;
                                if (col >= P.n) continue;
                                if (P.mode == EPI_LEVELS_I64) {
                                    const int gi = s - 1 - j;  // g - 2
                                    static_cast<int64_t *>(P.out)[(int64_t)gi * P.m * P.n + row +
                                                                  col * P.m] = Lg[i];
                                } else {
                                    static_cast<int32_t *>(P.out)[row + col * P.m] = (int32_t)Lg[i];
                                }
                            }
                        }
                    }
                    if (last && P.mode == EPI_DGEMM && row_ok) {
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int64_t col = nb * NC + cg * 8 + i;
                            if (col >= P.n) continue;
                            const int32_t eb = P.EB[col];
                            double X;
                            if (ea == kExpNonFinite || eb == kExpNonFinite)
                                X = __longlong_as_double(0x7ff8000000000000ll);
                            else
                                X = ldexp(acc[i], ea + eb);
                            double *cp = P.C + row + col * P.ldc;
                            double r;
                            if (P.beta == 0.0) r = __dmul_rn(P.alpha, X);
                            else r = __fma_rn(P.alpha, X, __dmul_rn(P.beta, *cp));
                            *cp = r;
                        }
                    }
                }
                ptx::tc_fence_before();
                ptx::mbar_arrive(tmem_empty);
            }
        }
    }
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, P.tmem_cols);
    }
#endif
}

// ---- host side -----------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                    const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                    const cuuint32_t *, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    }
    return fn;
}

// 3-D map over planes [s][rows][k_pad] (int8, K contiguous), 128B swizzle, box
// (128 B of K, box_rows rows, box_s slices).
bool make_map(CUtensorMap *map, const int8_t *base, int64_t k_pad, int64_t rows, int s,
              uint32_t box_rows, uint32_t box_s) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)k_pad, (cuuint64_t)rows, (cuuint64_t)s};
    cuuint64_t strides[2] = {(cuuint64_t)k_pad, (cuuint64_t)(k_pad * rows)};
    cuuint32_t box[3] = {(cuuint32_t)kKB, box_rows, box_s};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t *>(base), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int NC>
cudaError_t launch_t(const GemmArgs &a, const GemmPlan &p, EpiMode mode, cudaStream_t st) {
    CUtensorMap tmA, tmB;
    if (!make_map(&tmA, a.a_planes, a.k_pad, a.m, a.s, kBlockM, 1)) return cudaErrorInvalidValue;
    if (!make_map(&tmB, a.b_planes, a.k_pad, a.n, a.s, NC, (uint32_t)a.s))
        return cudaErrorInvalidValue;
    KParams P;
    P.m = a.m;
    P.n = a.n;
    P.k_pad = a.k_pad;
    P.s = a.s;
    P.w = a.w;
    P.num_k_blocks = p.num_k_blocks;
    P.chunk_blocks = p.chunk_blocks;
    P.k_chunks = p.k_chunks;
    P.tiles_m = ceil_div(a.m, kBlockM);
    P.tiles_n = ceil_div(a.n, NC);
    P.num_tiles = P.tiles_m * P.tiles_n;
    P.a_stages = p.a_stages;
    P.b_stages = p.b_stages;
    P.a_stage_bytes = (uint32_t)(kBlockM * kKB);
    P.b_stage_bytes = (uint32_t)(a.s * NC * kKB);
    P.tmem_cols = (uint32_t)p.tmem_cols;
    P.mode = mode;
    P.alpha = a.alpha;
    P.beta = a.beta;
    P.EA = a.EA;
    P.EB = a.EB;
    P.C = a.C;
    P.ldc = a.ldc;
    P.out = a.out;
    P.scratch = p.k_chunks > 1 ? a.chunk_scratch : nullptr;
    P.wave_counter = a.wave_counter;
    P.full_waves = P.num_tiles / p.grid;
    if (P.wave_counter) {
        cudaError_t e = cudaMemsetAsync(P.wave_counter, 0, sizeof(unsigned int), st);
        if (e != cudaSuccess) return e;
    }
    auto kern = k_oz_gemm<NC>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
    if (e != cudaSuccess) return e;
    kern<<<p.grid, kThreads, p.smem_bytes, st>>>(tmA, tmB, P);
    return cudaGetLastError();
}

}  // namespace

bool plan_gemm(int s, int w, int64_t m, int64_t n, int64_t k_pad, int num_sms, GemmPlan *p) {
    if (s < 1 || w < 1) return false;
    // N_c: largest tile with s * N_c TMEM columns <= 512 (one INT32 column per level)
    int nc = 0;
    for (int cand : {64, 48, 32, 16})
        if (s * cand <= 512) { nc = cand; break; }
    if (!nc) return false;
    const size_t smem_budget = 232448 - 2048;  // 227 KB opt-in max minus barriers/alignment
    const size_t b_stage = (size_t)s * nc * kKB;
    const size_t a_stage = (size_t)kBlockM * kKB;
    const int b_stages = 2;
    if (b_stages * b_stage + 2 * a_stage > smem_budget) return false;
    int a_stages = (int)((smem_budget - b_stages * b_stage) / a_stage);
    if (a_stages > 12) a_stages = 12;
    // INT32 budget per accumulator: (#pairs <= s) * k_chunk * (2^w - 1)^2 <= 2^31 - 1
    const int64_t d = ((int64_t)1 << w) - 1;
    const int64_t kmax = (int64_t)2147483647 / ((int64_t)s * d * d);
    const int64_t cb = kmax / kKB;
    if (cb < 1) return false;
    p->tile_n = nc;
    p->k_block = kKB;
    p->a_stages = a_stages;
    p->b_stages = b_stages;
    p->stages = a_stages;
    p->num_k_blocks = ceil_div(k_pad, kKB);
    p->chunk_blocks = cb;
    p->k_chunks = (int)ceil_div(p->num_k_blocks, cb);
    if (p->k_chunks < 1) p->k_chunks = 1;
    const int64_t tiles = ceil_div(m, kBlockM) * ceil_div(n, nc);
    p->grid = (int)(tiles < num_sms ? tiles : num_sms);
    if (p->grid < 1) p->grid = 1;
    p->smem_bytes = 1024 /*align slack*/ + b_stage * b_stages + a_stage * a_stages +
                    8 * (2 * b_stages + 2 * a_stages + 2) + 16;
    int cols = 32;
    while (cols < s * nc) cols <<= 1;
    p->tmem_cols = cols;
    return true;
}

size_t chunk_scratch_bytes(const GemmPlan &p, int s) {
    if (p.k_chunks <= 1) return 0;
    return (size_t)p.grid * s * p.tile_n * kBlockM * sizeof(int64_t);
}

cudaError_t launch_gemm(const GemmArgs &a, const GemmPlan &p, EpiMode mode, cudaStream_t st,
                        int *launches) {
    if (a.m <= 0 || a.n <= 0) return cudaSuccess;
    cudaError_t e;
    switch (p.tile_n) {
    case 64: e = launch_t<64>(a, p, mode, st); break;
    case 48: e = launch_t<48>(a, p, mode, st); break;
    case 32: e = launch_t<32>(a, p, mode, st); break;
    case 16: e = launch_t<16>(a, p, mode, st); break;
    default: return cudaErrorInvalidValue;
    }
    ++*launches;
    return e;
}

}  // namespace ozimmu
