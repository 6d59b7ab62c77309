// igemm_kernel.cuh -- the fused tcgen05 Ozaki GEMM kernel template (see igemm.cu).
#pragma once
// Included by igemm.cu (plan + dispatch) and by igemm_inst_*.cu, which hold the explicit
// instantiations of launch_t<S> (split so nvcc compiles the 32 kernels in parallel).
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "internal.h"
#include "ptx.cuh"

namespace ozimmu {
namespace gemm_detail {

constexpr int kThreads = 224;  // warps 0-3 epilogue, 4 TMA producer, 5 and 6 MMA issuers
constexpr int kBlockM = 128;
constexpr int kKB = 128;       // K bytes per k-block = one 128B swizzle row
constexpr int kGroupM = 8;     // grouped raster: 8 row-blocks per group

struct KParams {
    int64_t m, n, k_pad;
    int s, w;
    int64_t num_k_blocks, chunk_blocks;
    int k_chunks;
    int64_t tiles_m, tiles_n, num_tiles;
    // work units: one per cluster of cl = clm x cln CTAs, which takes row blocks
    // (clm i .. clm i + clm-1) x column tiles (cln j .. cln j + cln-1); the CTAs of a row
    // block share its A tiles (TMA multicast), the CTAs of a column tile share its B tiles
    int cl, clm, cln;
    int64_t units_m, units_n, num_units;
    int a_stages, b_stages;
    uint32_t a_stage_bytes, b_stage_bytes;
    uint32_t tmem_cols;
    int mode;
    double alpha, beta;
    double alpha_im, beta_im;
    const int32_t *EA, *EB;
    double *C;
    int64_t ldc;
    BatchMap c_rows, c_cols;     // stacked batches (C element units)
    void *out;
    int64_t *scratch;
    unsigned int *wave_counter;  // soft grid barrier between tile waves (may be null)
    int64_t full_waves;          // waves in which every CTA has a tile
    int wave_lag;                // waves a CTA may run ahead of the slowest one (0 = lockstep)
    int ksync;                   // extra soft barriers every `ksync` k-blocks (0 = per tile only)
    long long *stats;            // optional per-CTA stall counters (kStatSlots per CTA) or null
    int G;                       // pairs per INT32 accumulator (sub-group size)
    int T;                       // accumulator regions (sub-groups) per level, 1 or 2
    uint32_t region_col[2];      // TMEM column of region t (region t holds levels j < s - tG)
    // stream-K schedule (small problems, k_chunks == 1): cluster c of the G clusters takes the
    // kb-units [c W / G, (c+1) W / G) of W = num_units x num_k_blocks, so the last partial wave
    // disappears; a unit split between clusters leaves exact int32 partial level sums in
    // sk_part and the last cluster to finish it (sk_count) adds them and runs the epilogue.
    int sk;
    int64_t sk_total;            // W
    int *sk_count;               // [num_units][cl] arrivals (zeroed before the launch)
    int32_t *sk_part;            // [G][2 slots][cl][used_cols][128] partial level sums
    uint32_t used_cols;          // TMEM columns holding level sums
    // accumulator buffers: 2 = the level sums of consecutive tiles alternate between two TMEM
    // regions acc_stride columns apart, so the MMAs of tile t+1 run while the epilogue drains
    // tile t (short K: the drain is a large part of a tile); 1 = one region (the epilogue
    // releases it level by level as soon as every level has been read)
    int nacc;
    uint32_t acc_stride;
};

// ---- work schedule -------------------------------------------------------------------------
// Data-parallel: units u = c, c + G, .. (G = clusters in the grid), every unit over the whole
// K.  Stream-K: the contiguous kb-range of cluster c, cut into segments at unit boundaries;
// only a cluster's first and last segment can be a partial unit (slots 0 and 1).
__device__ __forceinline__ int64_t sk_begin(const KParams &P, int64_t c, int64_t G) {
    return c * P.sk_total / G;
}
// the cluster whose kb-range holds kb-unit g
__device__ __forceinline__ int64_t sk_owner(const KParams &P, int64_t g, int64_t G) {
    int64_t c = g * G / P.sk_total;
    while (c + 1 < G && sk_begin(P, c + 1, G) <= g) ++c;
    while (c > 0 && sk_begin(P, c, G) > g) --c;
    return c;
}
struct WorkIter {
    int64_t u, kb0, kb1;  // current unit and its k-block range
    bool first;           // first segment of this cluster (stream-K partial slot 0)
    int64_t g, ge;        // stream-K cursor / end (kb-units)
    __device__ __forceinline__ void start(const KParams &P) {
        const int64_t G = gridDim.x / P.cl, c = blockIdx.x / P.cl;
        first = true;
        if (P.sk) {
            g = sk_begin(P, c, G);
            ge = sk_begin(P, c + 1, G);
            seg(P);
        } else {
            u = c;
            kb0 = 0;
            kb1 = P.num_k_blocks;
        }
    }
    __device__ __forceinline__ void seg(const KParams &P) {
        u = g / P.num_k_blocks;
        kb0 = g - u * P.num_k_blocks;
        kb1 = kb0 + (ge - g);
        if (kb1 > P.num_k_blocks) kb1 = P.num_k_blocks;
    }
    __device__ __forceinline__ bool valid(const KParams &P) const {
        return P.sk ? g < ge : u < P.num_units;
    }
    __device__ __forceinline__ bool full(const KParams &P) const {
        return kb0 == 0 && kb1 == P.num_k_blocks;
    }
    __device__ __forceinline__ void next(const KParams &P) {
        first = false;
        if (P.sk) {
            g += kb1 - kb0;
            if (g < ge) seg(P);
        } else {
            u += gridDim.x / P.cl;
        }
    }
};

// N_c (output columns per tile) as a function of s: the largest of {64, 48, 32, 16} with
// s * N_c <= 512 TMEM columns.
__host__ __device__ constexpr int nc_for(int S) {
    return S * 64 <= 512 ? 64 : (S * 48 <= 512 ? 48 : (S * 32 <= 512 ? 32 : 16));
}

// Order in which the s A-slice tiles of a k-block are loaded and consumed: p = 1, s, 2,
// s-1, ... (long and short windows alternate, so the two MMA issuers get similar work; the
// ascending order measured the same).  The level sums are exact integers, so the order of
// the MMAs into TMEM does not change any result.
// L2 cache policy of the operand loads (TMA .L2::cache_hint)
#ifndef OZ_A_HINT
#define OZ_A_HINT ptx::kEvictNormal
#endif
#ifndef OZ_B_HINT
#define OZ_B_HINT ptx::kEvictNormal
#endif
#ifndef OZ_KSNAKE
#define OZ_KSNAKE 1
#endif
#ifndef OZ_SLICE_ORDER
#define OZ_SLICE_ORDER 1
#endif
__host__ __device__ constexpr int slice_p(int S, int i) {
    return OZ_SLICE_ORDER == 0 ? i + 1 : ((i & 1) == 0 ? i / 2 + 1 : S - i / 2);
}

// stall-counter slots (development instrumentation, OZIMMU_STATS=1)
enum : int { ST_TOTAL = 0, ST_MMA_WAIT_B, ST_MMA_WAIT_A, ST_MMA_WAIT_TMEM, ST_PROD_WAVE,
             ST_PROD_WAIT_A, ST_PROD_WAIT_B, ST_EPI_BUSY, ST_EPI_TMEM, ST_EPI_STORE,
             ST_MMA_FIRST_A, ST_MMA_B_TILE0, ST_MMA_NS, ST_KERNEL_NS, kStatSlots = 14 };

// Grouped raster over units (kGroupM row blocks per group); rank = CTA rank in the cluster
// (rank = rm * cln + rn).  mb / nb may reach tiles_m / tiles_n: a dummy tile (operands
// zero-filled by TMA, no stores).
__device__ __forceinline__ void tile_coords(int64_t u, const KParams &P, uint32_t rank,
                                            int64_t &mb, int64_t &nb) {
    const int64_t GM = kGroupM / P.clm;  // unit rows per group
    const int64_t per_group = GM * P.units_n;
    const int64_t g = u / per_group;
    const int64_t r = u % per_group;
    const int64_t gm0 = g * GM;
    int64_t gsz = P.units_m - gm0;
    gsz = gsz < GM ? gsz : GM;
    mb = (gm0 + r % gsz) * P.clm + (int64_t)(rank / (uint32_t)P.cln);
    nb = (r / gsz) * P.cln + (int64_t)(rank % (uint32_t)P.cln);
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
__device__ __forceinline__ void wave_sync(const KParams &P, int64_t wave, int64_t bidx) {
    if (!P.wave_counter || wave >= P.full_waves) return;
    atomicAdd(P.wave_counter, 1u);
    if (bidx < P.wave_lag) return;
    const unsigned int target = (unsigned int)((bidx + 1 - P.wave_lag) * gridDim.x);
    const uint64_t t0 = globaltimer();
    while (ld_acquire(P.wave_counter) < target) {
        if (globaltimer() - t0 > 200000ull) break;  // 200 us cap
        __nanosleep(256);
    }
}

// X = acc 2^e with ldexp semantics (reading A7): exact power-of-two multiply in range.
__device__ __forceinline__ double scale_x(double acc, int32_t ea, int32_t eb) {
    if (ea == kExpNonFinite || eb == kExpNonFinite) return __longlong_as_double(0x7ff8000000000000ll);
    const int e = ea + eb;
    if (e >= -1022 && e <= 1023) return __dmul_rn(acc, pow2(e));  // one rounding, 2^e exact
    return ldexp(acc, e);
}
// z = a x for complex a, x (ZGEMM reading A16): re = fma(ar, xr, -(ai xi)), im = fma(ar, xi, ai xr)
__device__ __forceinline__ void cmul(double ar, double ai, double xr, double xi, double &zr,
                                     double &zi) {
    zr = __fma_rn(ar, xr, -__dmul_rn(ai, xi));
    zi = __fma_rn(ar, xi, __dmul_rn(ai, xr));
}

// Offset of row `row` / column `col` of C (in C elements) under a stacked-batch map.
__device__ __forceinline__ int64_t c_row_off(const BatchMap &b, int64_t row) {
    if (!b.per_item) return row;
    const int64_t it = row / b.per_item;
    return it * b.stride + (row - it * b.per_item);
}
__device__ __forceinline__ int64_t c_col_off(const BatchMap &b, int64_t col, int64_t ldc) {
    if (!b.per_item) return col * ldc;
    const uint32_t it = static_cast<uint32_t>(col) / static_cast<uint32_t>(b.per_item);
    return (int64_t)it * b.stride + (col - (int64_t)it * b.per_item) * ldc;
}

// Final output of one row (this thread) of the tile: real C (reading A8) or complex C.
template <int NC>
__device__ __forceinline__ void store_row(const KParams &P, const double (&acc)[NC],
                                          const int32_t *ebt, int32_t ea, int64_t row,
                                          int64_t nb) {
    const int64_t roff = c_row_off(P.c_rows, row);
    if (P.mode == EPI_DGEMM) {
        double *crow = P.C + roff;
        // Fast path (every full tile in practice): all NC columns inside C, no stacked-batch
        // column map, and every scale 2^(E_A + E_B) a normal double -- then X = acc 2^e is
        // one exact multiply and the loop has no per-element branches.  Same operations as
        // the general path below, so the same bits.
        if ((nb + 1) * NC <= P.n && !P.c_cols.per_item && ea != kExpNonFinite) {
            bool ok = true;
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                const long long e = (long long)ea + ebt[i];  // no int overflow on the marker
                ok &= ebt[i] != kExpNonFinite && e >= -1022 && e <= 1023;
            }
            if (ok) {
                double *cp = crow + (nb * NC) * P.ldc;
                if (P.beta == 0.0) {
#pragma unroll
                    for (int i = 0; i < NC; ++i)
                        cp[i * P.ldc] = __dmul_rn(P.alpha, __dmul_rn(acc[i], pow2(ea + ebt[i])));
                } else {
#pragma unroll
                    for (int i = 0; i < NC; ++i) {
                        const double X = __dmul_rn(acc[i], pow2(ea + ebt[i]));
                        cp[i * P.ldc] = __fma_rn(P.alpha, X, __dmul_rn(P.beta, cp[i * P.ldc]));
                    }
                }
                return;
            }
        }
#pragma unroll
        for (int i = 0; i < NC; ++i) {
            const int64_t col = nb * NC + i;
            if (col >= P.n) break;
            const double X = scale_x(acc[i], ea, ebt[i]);
            double *cp = crow + c_col_off(P.c_cols, col, P.ldc);
            *cp = P.beta == 0.0 ? __dmul_rn(P.alpha, X)
                                : __fma_rn(P.alpha, X, __dmul_rn(P.beta, *cp));
        }
    } else {  // EPI_ZGEMM: columns (2j, 2j+1) = (Re, Im) of complex column j
        const bool beta0 = P.beta == 0.0 && P.beta_im == 0.0;
        // Fast path (full tiles with normal scales, as for DGEMM): the same operations without
        // per-element range checks -- X = acc 2^e is one exact multiply -- so the same bits.
        if ((nb + 1) * NC <= P.n && !P.c_cols.per_item && ea != kExpNonFinite) {
            bool ok = true;
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                const long long e = (long long)ea + ebt[i];
                ok &= ebt[i] != kExpNonFinite && e >= -1022 && e <= 1023;
            }
            if (ok) {
                double2 *cp = reinterpret_cast<double2 *>(P.C) + roff + (nb * NC >> 1) * P.ldc;
#pragma unroll
                for (int i = 0; i < NC; i += 2) {
                    const double xr = __dmul_rn(acc[i], pow2(ea + ebt[i]));
                    const double xi = __dmul_rn(acc[i + 1], pow2(ea + ebt[i + 1]));
                    double tr, ti;
                    cmul(P.alpha, P.alpha_im, xr, xi, tr, ti);
                    if (!beta0) {
                        const double2 c = cp[(i >> 1) * P.ldc];
                        double ur, ui;
                        cmul(P.beta, P.beta_im, c.x, c.y, ur, ui);
                        tr = __dadd_rn(tr, ur);
                        ti = __dadd_rn(ti, ui);
                    }
                    cp[(i >> 1) * P.ldc] = make_double2(tr, ti);
                }
                return;
            }
        }
#pragma unroll
        for (int i = 0; i < NC; i += 2) {
            const int64_t col = nb * NC + i;
            if (col >= P.n) break;
            const double xr = scale_x(acc[i], ea, ebt[i]);
            const double xi = scale_x(acc[i + 1], ea, ebt[i + 1]);
            double tr, ti;
            cmul(P.alpha, P.alpha_im, xr, xi, tr, ti);
            double2 *cp = reinterpret_cast<double2 *>(P.C) + roff + c_col_off(P.c_cols, col >> 1, P.ldc);
            if (!beta0) {
                const double2 c = *cp;
                double ur, ui;
                cmul(P.beta, P.beta_im, c.x, c.y, ur, ui);
                tr = __dadd_rn(tr, ur);
                ti = __dadd_rn(ti, ui);
            }
            *cp = make_double2(tr, ti);
        }
    }
}

template <int S, int NCV = nc_for(S)>
__global__ void __launch_bounds__(kThreads, 1)
    k_oz_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const KParams P) {
    constexpr int NC = NCV;  // output columns per tile (nc_for(S), or 32 for small problems)
#ifndef OZ_PIPE_DRAIN
#define OZ_PIPE_DRAIN 1
#endif
    // epilogue drain with the next level's TMEM loads in flight: N_c = 32 only (measured: 1024^3
    // GEMM 52.3 -> 51.2 us, 2048^3 257.6 -> 254.7 us; at N_c = 48 the second buffer spills and
    // 16384^3 loses ~0.5 %)
    constexpr bool kPipeDrain = OZ_PIPE_DRAIN && NC <= 32;
    __shared__ int32_t eb_s[2][64];  // column exponents of the current tile (double-buffered)
    __shared__ int sk_old;           // stream-K: arrivals before this CTA's part of a unit
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
    uint64_t *tmem_full = a_empty + P.a_stages;   // [2]: one per accumulator buffer
    uint64_t *tmem_empty = tmem_full + 2;         // [2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);

    const uint32_t warp = ptx::warp_id();
    const uint32_t lane = ptx::lane_id();
    constexpr int s = S;
    const uint32_t rank = P.cl > 1 ? ptx::cluster_ctarank() : 0u;
    const uint32_t rm = rank / (uint32_t)P.cln, rn = rank % (uint32_t)P.cln;
    // multicast groups: CTAs sharing this CTA's row block (A) / column tile (B)
    const uint16_t amask = (uint16_t)(((1u << P.cln) - 1u) << (rm * P.cln));
    uint16_t bmask = 0;
    for (int j = 0; j < P.clm; ++j) bmask |= (uint16_t)(1u << (j * P.cln + rn));

    if (warp == 5 && lane == 0) {
        for (int i = 0; i < P.b_stages; ++i) {
            ptx::mbar_init(&b_full[i], 1);
            ptx::mbar_init(&b_empty[i], 2 * P.clm);  // both MMA issuers of each CTA sharing it
        }
        for (int i = 0; i < P.a_stages; ++i) {
            ptx::mbar_init(&a_full[i], 1);
            ptx::mbar_init(&a_empty[i], (uint32_t)P.cln);  // the MMAs of each CTA sharing it
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tmem_full[i], 2);  // committed by both MMA issuers
            ptx::mbar_init(&tmem_empty[i], 4 * 32);
        }
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
    if (P.cl > 1) ptx::cluster_sync();  // peers' barriers initialised before any multicast
    else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // Programmatic dependent launch (launch_t): the set-up above may overlap the tail of the
    // previous kernel on the stream (the slicing); nothing below reads global memory before
    // that kernel has completed and its writes are visible.
    asm volatile("griddepcontrol.wait;" ::: "memory");


    if (warp == 4) {
        // ===================== TMA producer =====================
        if (ptx::elect_one()) {
            int bs = 0, as = 0;
            uint32_t bph = 0, aph = 0;
            int64_t wave = 0, bidx = 0;  // tile wave, soft-barrier instance
            long long st_w = 0, st_pa = 0, st_pb = 0;
            const uint32_t b_tx = (uint32_t)(s * NC * kKB), a_tx = (uint32_t)(kBlockM * kKB);
            WorkIter it;
            for (it.start(P); it.valid(P); it.next(P), ++wave) {
                int64_t mb, nb;
                tile_coords(it.u, P, rank, mb, nb);
                long long c0 = P.stats ? clock64() : 0;
                wave_sync(P, wave, bidx++);
                if (P.stats) st_w += clock64() - c0;
                // K snake: odd waves walk K backwards, so a wave starts on the k-blocks the
                // previous wave (same A row blocks) touched last, still in L2.  The INT32
                // sums are order-independent; K chunks (int64 partials) keep the forward order.
                const bool rev = OZ_KSNAKE && !P.sk && P.k_chunks == 1 && (wave & 1);
                auto kmap = [&](int64_t kb) { return rev ? P.num_k_blocks - 1 - kb : kb; };
                for (int64_t kb = it.kb0; kb < it.kb1; ++kb) {
                    const int64_t kx = kmap(kb);
                    if (P.ksync && kb > 0 && kb % P.ksync == 0) {
                        long long c3 = P.stats ? clock64() : 0;
                        wave_sync(P, wave, bidx++);
                        if (P.stats) st_w += clock64() - c3;
                    }
                    long long c1 = P.stats ? clock64() : 0;
                    ptx::mbar_wait(&b_empty[bs], bph ^ 1);
                    if (P.stats) st_pb += clock64() - c1;
                    ptx::mbar_arrive_expect_tx(&b_full[bs], b_tx);
                    if (P.clm == 1) {
                        ptx::tma_load_3d(&tmB, &b_full[bs], smB + (size_t)bs * P.b_stage_bytes,
                                         (int32_t)(kx * kKB), (int32_t)(nb * NC), 0, OZ_B_HINT);
                    } else {  // this CTA's NC/clm columns of every slice, to its column group
                        const int part = NC / P.clm;
#pragma unroll 1
                        for (int z = 0; z < S; ++z)
                            ptx::tma_load_3d_mc(&tmB, &b_full[bs],
                                                smB + (size_t)bs * P.b_stage_bytes +
                                                    (size_t)(z * NC + (int)rm * part) * kKB,
                                                (int32_t)(kx * kKB),
                                                (int32_t)(nb * NC + (int)rm * part), z, bmask,
                                                OZ_B_HINT);
                    }
                    if (++bs == P.b_stages) { bs = 0; bph ^= 1; }
#pragma unroll 1
                    for (int i = 0; i < S; ++i) {
                        long long c2 = P.stats ? clock64() : 0;
                        ptx::mbar_wait(&a_empty[as], aph ^ 1);
                        if (P.stats) st_pa += clock64() - c2;
                        ptx::mbar_arrive_expect_tx(&a_full[as], a_tx);
                        if (P.cln > 1) {  // this CTA's rows of the tile, to its row group
                            const int part = kBlockM / P.cln;
                            ptx::tma_load_3d_mc(&tmA, &a_full[as],
                                                smA + (size_t)as * P.a_stage_bytes +
                                                    (size_t)rn * part * kKB,
                                                (int32_t)(kx * kKB),
                                                (int32_t)(mb * kBlockM + (int)rn * part),
                                                slice_p(S, i) - 1, amask, OZ_A_HINT);
                        }
                        else
                            ptx::tma_load_3d(&tmA, &a_full[as], smA + (size_t)as * P.a_stage_bytes,
                                             (int32_t)(kx * kKB), (int32_t)(mb * kBlockM),
                                             slice_p(S, i) - 1, OZ_A_HINT);
                        if (++as == P.a_stages) { as = 0; aph ^= 1; }
                    }
                }
            }
            if (P.cl > 1) {
                // drain: every slot released by all CTAs sharing it, so no multicast arrive
                // is still in flight towards a peer when the cluster exits
                for (int i = 0; i < P.a_stages; ++i) {
                    ptx::mbar_wait(&a_empty[as], aph ^ 1);
                    if (++as == P.a_stages) { as = 0; aph ^= 1; }
                }
                for (int i = 0; i < P.b_stages; ++i) {
                    ptx::mbar_wait(&b_empty[bs], bph ^ 1);
                    if (++bs == P.b_stages) { bs = 0; bph ^= 1; }
                }
            }
            if (P.stats) {
                long long *st = P.stats + (int64_t)blockIdx.x * kStatSlots;
                st[ST_PROD_WAVE] = st_w;
                st[ST_PROD_WAIT_A] = st_pa;
                st[ST_PROD_WAIT_B] = st_pb;
            }
        }
    } else if (warp == 5 || warp == 6) {
        // ===================== MMA issuers (two warps) =====================
        // The A-slice tiles of the ring alternate between warps 5 and 6 (tile t -> warp
        // 5 + (t & 1)): while one warp waits on its tile's mbarrier and builds descriptors,
        // the other's MMAs keep the tensor pipe fed (one issuer leaves ~15% of the pipe idle
        // on the per-tile wait latency; tools/issue_bench.cu).  Every MMA accumulates
        // (the epilogue zeroes TMEM before releasing it), so the interleaving of the two
        // warps' MMAs cannot change the exact integer level sums.  b_empty and tmem_full
        // take one commit from each warp.
        constexpr int kMaxBlk = 256 / NC;  // window blocks per instruction (N <= 256)
        const uint32_t me = warp - 5;
        // TMEM column of A-slice p's window: region t(p) = (p-1)/G (INT32 sub-group)
        uint32_t pcol0[S + 1], pcol[S + 1];
#pragma unroll
        for (int p = 1; p <= S; ++p) pcol0[p] = tmem_base + P.region_col[(p - 1) / P.G];
        int bs = 0, as = 0;
        uint32_t bph = 0, aph = 0, tpar = 0;
        uint32_t acc_iter = 0;
        long long st_b = 0, st_b0 = 0, st_a = 0, st_t = 0, st_af = 0, t_begin = clock64();
        const uint64_t ns_begin = globaltimer();
        const uint64_t adesc_base = ptx::smem_desc_kmajor<kKB>(ptx::smem_u32(smA));
        const uint64_t bdesc_base = ptx::smem_desc_kmajor<kKB>(ptx::smem_u32(smB));

        // MMAs of A-slice p for one k-step against its window [0, L), split into the fewest
        // instructions of N <= 256 with block counts as equal as possible: an M = 128,
        // K = 32 i8 MMA costs about max(N/2, ~58) cycles (tools/mma_bench.cu), so 6 blocks
        // go as 3 + 3 rather than 5 + 1.
        auto issue = [&](int p, uint64_t ad, uint64_t bd) {
            const int L = S + 1 - p;
            const int pieces = (L + kMaxBlk - 1) / kMaxBlk;
            int j0 = 0;
#pragma unroll
            for (int q = 0; q < pieces; ++q) {
                const int nbk = L / pieces + (q < L % pieces ? 1 : 0);
                ptx::mma_i8(pcol[p] + (uint32_t)(j0 * NC), ad, bd + (uint64_t)((j0 * NC * kKB) >> 4),
                            ptx::idesc_i8(kBlockM, (uint32_t)(nbk * NC)), 1u);
                j0 += nbk;
            }
        };

        WorkIter it;
        for (it.start(P); it.valid(P); it.next(P)) {
            for (int c = 0; c < P.k_chunks; ++c, ++acc_iter) {
                int64_t kb0 = (int64_t)c * P.chunk_blocks;
                int64_t kb1 = kb0 + P.chunk_blocks;
                kb1 = kb1 < P.num_k_blocks ? kb1 : P.num_k_blocks;
                if (P.sk) {  // stream-K (k_chunks == 1): this cluster's k-blocks of the unit
                    kb0 = it.kb0;
                    kb1 = it.kb1;
                }
                // the epilogue has read and zeroed accumulator buffer `ab` (its use acc_iter / nacc)
                const uint32_t ab = P.nacc > 1 ? (acc_iter & 1u) : 0u;
                const uint32_t acc_ph = P.nacc > 1 ? ((acc_iter >> 1) & 1u) : (acc_iter & 1u);
#pragma unroll
                for (int p = 1; p <= S; ++p) pcol[p] = pcol0[p] + ab * P.acc_stride;
                {
                    long long c0 = P.stats ? clock64() : 0;
                    ptx::mbar_wait(&tmem_empty[ab], acc_ph);
                    if (P.stats) st_t += clock64() - c0;
                    ptx::tc_fence_after();
                }
                for (int64_t kb = kb0; kb < kb1; ++kb) {
                    long long c1 = P.stats ? clock64() : 0;
                    ptx::mbar_wait(&b_full[bs], bph);
                    if (P.stats) {
                        if (kb == 0) st_b0 += clock64() - c1;
                        else st_b += clock64() - c1;
                    }
                    const uint64_t bdesc0 = bdesc_base + ((bs * P.b_stage_bytes) >> 4);
#pragma unroll
                    for (int i = 0; i < S; ++i) {
                        const int p = slice_p(S, i);
                        // tile parity: tpar flips every tile (S is folded in by the counter).
                        // a_stages is even, so ring slot `as` always holds tiles of the same
                        // parity: each slot has ONE consumer warp, which waits on every phase
                        // of it in order (with an odd ring a warp would skip the other warp's
                        // phases of a slot and a parity wait could then pass on a phase that
                        // has not completed).
                        if (((tpar + (uint32_t)i) & 1u) == me) {
                            long long c2 = P.stats ? clock64() : 0;
                            ptx::mbar_wait(&a_full[as], aph);
                            if (P.stats) {
                                if (kb == kb0) st_af += clock64() - c2;
                                else st_a += clock64() - c2;
                            }
                            ptx::tc_fence_after();
                            if (ptx::elect_one()) {
                                const uint64_t adesc0 = adesc_base + ((as * P.a_stage_bytes) >> 4);
#pragma unroll
                                for (int ks = 0; ks < kKB / 32; ++ks)
                                    issue(p, adesc0 + (uint64_t)(ks * 2),
                                          bdesc0 + (uint64_t)(((p - 1) * NC * kKB + ks * 32) >> 4));
                                if (P.cln > 1) ptx::mma_commit_mc(&a_empty[as], amask);
                                else ptx::mma_commit(&a_empty[as]);
                            }
                            __syncwarp();
                        }
                        if (++as == P.a_stages) { as = 0; aph ^= 1; }
                    }
                    tpar += (uint32_t)S;
                    if (ptx::elect_one()) {
                        if (P.clm > 1) ptx::mma_commit_mc(&b_empty[bs], bmask);
                        else ptx::mma_commit(&b_empty[bs]);
                    }
                    __syncwarp();
                    if (++bs == P.b_stages) { bs = 0; bph ^= 1; }
                }
                if (ptx::elect_one()) ptx::mma_commit(&tmem_full[ab]);  // period accumulated
                __syncwarp();
            }
        }
        if (P.stats && lane == 0 && me == 0) {
            long long *st = P.stats + (int64_t)blockIdx.x * kStatSlots;
            st[ST_TOTAL] = clock64() - t_begin;
            st[ST_MMA_NS] = (long long)(globaltimer() - ns_begin);  // with ST_TOTAL: the SM clock
            st[ST_MMA_WAIT_B] = st_b;
            st[ST_MMA_WAIT_A] = st_a;
            st[ST_MMA_WAIT_TMEM] = st_t;
            st[ST_MMA_FIRST_A] = st_af;
            st[ST_MMA_B_TILE0] = st_b0;
        }
    } else {
        // ===================== epilogue (warps 0-3) =====================
        // Thread = one row of the tile (TMEM lane).  Level-major: level j (g = s+1-j) of all
        // NC columns is read from TMEM (both INT32 sub-group regions) and combined in FP64 in
        // the canonical order g = s+1 .. 2 (reading A6).  The accumulator is released to the
        // next period's MMAs as soon as every level has been read; the scaling (A7),
        // alpha/beta (A8), NaN rows/cols (A9) and the stores of C then overlap those MMAs.
        const uint32_t row_local = warp * 32 + lane;
        const uint32_t lane_addr = (warp * 32) << 16;
        const uint32_t tmem_base0 = tmem_base;
        int64_t *scr = P.scratch ? P.scratch + (int64_t)blockIdx.x * s * NC * kBlockM : nullptr;
        const int T = P.T;
        const int G = P.G;
        constexpr int kCH = NC < 32 ? NC : 32;  // columns per TMEM read batch
        // The MMA issuers only accumulate: this warp zeroes its 32 TMEM lanes of every column
        // it reads (after reading them) and, once, before the first period.
        {
            const uint32_t used = (uint32_t)(S * NC) + (T > 1 ? (uint32_t)((S - G) * NC) : 0u);
            for (int b = 0; b < P.nacc; ++b)
                for (uint32_t c = 0; c < used; c += 16)
                    ptx::tmem_st_zero_x16(tmem_base + b * P.acc_stride + lane_addr + c);
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            for (int b = 0; b < P.nacc; ++b) ptx::mbar_arrive(&tmem_empty[b]);  // buffers zeroed
        }
        uint32_t acc_iter = 0, tile_iter = 0;
        long long st_e = 0, st_et = 0, st_es = 0;
        WorkIter it;
        for (it.start(P); it.valid(P); it.next(P)) {
            const int64_t u = it.u;
            int64_t mb, nb;
            tile_coords(u, P, rank, mb, nb);
            const int64_t row = mb * kBlockM + row_local;
            const bool row_ok = row < P.m;
            const bool fp_out = P.mode == EPI_DGEMM || P.mode == EPI_ZGEMM;
            const int32_t ea = (fp_out && row_ok) ? P.EA[row] : 0;
            // stage this tile's column exponents in shared memory while the MMAs run
            int32_t *ebt = eb_s[tile_iter & 1];
            if (fp_out && row_local < (uint32_t)NC) {
                const int64_t col = nb * NC + row_local;
                ebt[row_local] = col < P.n ? P.EB[col] : 0;
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            ++tile_iter;
            for (int c = 0; c < P.k_chunks; ++c, ++acc_iter) {
                const uint32_t ab = P.nacc > 1 ? (acc_iter & 1u) : 0u;
                const uint32_t acc_ph = P.nacc > 1 ? ((acc_iter >> 1) & 1u) : (acc_iter & 1u);
                const uint32_t tmem_base = tmem_base0 + ab * P.acc_stride;  // this period's buffer
                ptx::mbar_wait(&tmem_full[ab], acc_ph);
                ptx::tc_fence_after();
                long long ce = P.stats ? clock64() : 0;
                const bool first = c == 0, last = c == P.k_chunks - 1;
                if (P.sk && !it.full(P)) {
                    // ------------- stream-K: this cluster holds k-blocks [kb0, kb1) -------------
                    // The parts of a unit come from consecutive clusters and are combined as exact
                    // integers (the same L_g as one CTA over the whole K, so the same C).  A part
                    // that finds every other part already parked (the usual case: the other
                    // clusters open their ranges with this unit) is the last: it adds the parked
                    // int32 partials into its own TMEM accumulators and falls through to the
                    // normal epilogue.  Otherwise it parks its partial and counts its arrival; the
                    // last arrival does the same, the others zero and release TMEM.
                    const int64_t NG = gridDim.x / P.cl, cidx = blockIdx.x / P.cl;
                    const int64_t nkb = P.num_k_blocks;
                    const int64_t cf = sk_owner(P, u * nkb, NG), cl_ = sk_owner(P, u * nkb + nkb - 1, NG);
                    const int np = (int)(cl_ - cf + 1);
                    const int slot_f = sk_begin(P, cf, NG) == u * nkb ? 0 : 1;
                    // partial layout [slot][row][used_cols] int32: each thread writes and reads
                    // its own row with 16-byte accesses
                    auto part = [&](int64_t cc, int slot) {
                        return P.sk_part + ((cc * 2 + slot) * P.cl + rank) * (int64_t)P.used_cols *
                                               kBlockM + (int64_t)row_local * P.used_cols;
                    };
                    int *cnt = P.sk_count + u * P.cl + rank;
                    if (row_local == 0) sk_old = (int)ld_acquire(reinterpret_cast<const unsigned int *>(cnt));
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    bool last_part = sk_old == np - 1;  // every other part is parked
                    asm volatile("bar.sync 1, 128;" ::: "memory");  // sk_old is reused
                    if (!last_part) {  // park this part (TMEM untouched until the count is known)
                        int32_t *mine = part(cidx, it.first ? 0 : 1);
                        for (uint32_t col = 0; col < P.used_cols; col += 16) {
                            uint32_t v[16];
                            __syncwarp();
                            ptx::tmem_ld_x16(tmem_base + lane_addr + col, v);
                            ptx::tmem_ld_wait();
                            int4 *dst = reinterpret_cast<int4 *>(mine + col);
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                dst[q] = make_int4((int)v[4 * q], (int)v[4 * q + 1], (int)v[4 * q + 2],
                                                   (int)v[4 * q + 3]);
                        }
                        __threadfence();
                        asm volatile("bar.sync 1, 128;" ::: "memory");
                        if (row_local == 0) sk_old = atomicAdd(cnt, 1);
                        asm volatile("bar.sync 1, 128;" ::: "memory");
                        last_part = sk_old == np - 1;
                        asm volatile("bar.sync 1, 128;" ::: "memory");
                        if (!last_part) {  // another part finishes the unit: zero and release TMEM
                            for (uint32_t col = 0; col < P.used_cols; col += 16)
                                ptx::tmem_st_zero_x16(tmem_base + lane_addr + col);
                            ptx::tmem_st_wait();
                            ptx::tc_fence_before();
                            ptx::mbar_arrive(&tmem_empty[ab]);
                            if (P.stats) st_e += clock64() - ce;
                            continue;
                        }
                    }
                    // last part: TMEM += every other parked part, column block by column block
                    // (region totals stay within the INT32 budget of the whole K)
                    __threadfence();
                    for (uint32_t col = 0; col < P.used_cols; col += 32) {  // used_cols % 16 == 0
                        const bool two = col + 16 < P.used_cols;
                        uint32_t v[32];
                        __syncwarp();
                        ptx::tmem_ld_x16(tmem_base + lane_addr + col, v);
                        if (two) ptx::tmem_ld_x16(tmem_base + lane_addr + col + 16, v + 16);
                        ptx::tmem_ld_wait();
                        for (int64_t cc = cf; cc <= cl_; ++cc) {
                            if (cc == cidx) continue;
                            const int4 *q0 = reinterpret_cast<const int4 *>(
                                part(cc, cc == cf ? slot_f : 0) + col);
                            int4 x[8];
#pragma unroll
                            for (int q = 0; q < 8; ++q)
                                x[q] = (q < 4 || two) ? __ldcg(q0 + q) : make_int4(0, 0, 0, 0);
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                v[4 * q] += (uint32_t)x[q].x;
                                v[4 * q + 1] += (uint32_t)x[q].y;
                                v[4 * q + 2] += (uint32_t)x[q].z;
                                v[4 * q + 3] += (uint32_t)x[q].w;
                            }
                        }
                        ptx::tmem_st_x16(tmem_base + lane_addr + col, v);
                        if (two) ptx::tmem_st_x16(tmem_base + lane_addr + col + 16, v + 16);
                    }
                    ptx::tmem_st_wait();
                    // fall through: the unit's complete level sums are in TMEM
                }
                if (fp_out && !scr) {
                    // ---------------- fast path: one period, FP64 result ----------------
                    double acc[NC];
#pragma unroll
                    for (int i = 0; i < NC; ++i) acc[i] = 0.0;
                    // levels held in two INT32 regions first (T = 2: j < S - G), one at a time
                    const int j_two = T > 1 ? S - G : 0;
#pragma unroll 1
                    for (int j = 0; j < (kPipeDrain ? j_two : S); ++j) {  // level g = s+1-j
                        const double sc = pow2(-P.w * (S + 1 - j));
                        const bool two = T > 1 && j < S - G;
#pragma unroll
                        for (int c0 = 0; c0 < NC; c0 += kCH) {
                            uint32_t v[kCH], v2[kCH];
                            __syncwarp();
#pragma unroll
                            for (int c16 = 0; c16 < kCH; c16 += 16)
                                if (c0 + c16 < NC)
                                    ptx::tmem_ld_x16(tmem_base + lane_addr + (uint32_t)(j * NC + c0 + c16),
                                                     &v[c16]);
                            if (two) {
#pragma unroll
                                for (int c16 = 0; c16 < kCH; c16 += 16)
                                    if (c0 + c16 < NC)
                                        ptx::tmem_ld_x16(tmem_base + lane_addr + P.region_col[1] +
                                                             (uint32_t)(j * NC + c0 + c16), &v2[c16]);
                                ptx::tmem_ld_wait();
#pragma unroll
                                for (int c16 = 0; c16 < kCH; c16 += 16)
                                    if (c0 + c16 < NC) {
                                        ptx::tmem_st_zero_x16(tmem_base + lane_addr + (uint32_t)(j * NC + c0 + c16));
                                        ptx::tmem_st_zero_x16(tmem_base + lane_addr + P.region_col[1] +
                                                              (uint32_t)(j * NC + c0 + c16));
                                    }
                                // acc += L_g 2^(-wg): the product is exact, so the fma rounds
                                // once like the oracle's add; both INT32 parts and their sum
                                // are exact in binary64.
#pragma unroll
                                for (int ii = 0; ii < kCH; ++ii)
                                    if (c0 + ii < NC)
                                        acc[c0 + ii] = __fma_rn(__dadd_rn((double)(int32_t)v[ii],
                                                                          (double)(int32_t)v2[ii]),
                                                                sc, acc[c0 + ii]);
                            } else {
                                ptx::tmem_ld_wait();
#pragma unroll
                                for (int c16 = 0; c16 < kCH; c16 += 16)
                                    if (c0 + c16 < NC)
                                        ptx::tmem_st_zero_x16(tmem_base + lane_addr + (uint32_t)(j * NC + c0 + c16));
#pragma unroll
                                for (int ii = 0; ii < kCH; ++ii)
                                    if (c0 + ii < NC)
                                        acc[c0 + ii] = __fma_rn((double)(int32_t)v[ii], sc, acc[c0 + ii]);
                            }
                        }
                    }
                    if constexpr (kPipeDrain) {
                        // the remaining levels (one region each) with the TMEM loads of level j+1
                        // in flight while level j is zeroed and accumulated (two register
                        // buffers): the drain is bound by the load latency otherwise, the FP64
                        // work per level being short (same operations in the same order)
                        uint32_t va[NC], vb[NC];
                        auto load_lvl = [&](int j, uint32_t (&v)[NC]) {
                            __syncwarp();
#pragma unroll
                            for (int c16 = 0; c16 < NC; c16 += 16)
                                ptx::tmem_ld_x16(tmem_base + lane_addr + (uint32_t)(j * NC + c16), &v[c16]);
                        };
                        auto use_lvl = [&](int j, const uint32_t (&v)[NC]) {
#pragma unroll
                            for (int c16 = 0; c16 < NC; c16 += 16)
                                ptx::tmem_st_zero_x16(tmem_base + lane_addr + (uint32_t)(j * NC + c16));
                            const double sc = pow2(-P.w * (S + 1 - j));
#pragma unroll
                            for (int ii = 0; ii < NC; ++ii)
                                acc[ii] = __fma_rn((double)(int32_t)v[ii], sc, acc[ii]);
                        };
                        if (j_two < S) load_lvl(j_two, va);
#pragma unroll 1
                        for (int j = j_two; j < S; j += 2) {
                            ptx::tmem_ld_wait();  // level j (va)
                            if (j + 1 < S) load_lvl(j + 1, vb);
                            use_lvl(j, va);
                            if (j + 1 >= S) break;
                            ptx::tmem_ld_wait();  // level j+1 (vb)
                            if (j + 2 < S) load_lvl(j + 2, va);
                            use_lvl(j + 1, vb);
                        }
                    }
                    ptx::tmem_st_wait();
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(&tmem_empty[ab]);  // accumulator read and zeroed: next period may start
                    if (P.stats) st_et += clock64() - ce;
                    long long cs0 = P.stats ? clock64() : 0;
                    if (row_ok) store_row<NC>(P, acc, ebt, ea, row, nb);
                    if (P.stats) {
                        st_es += clock64() - cs0;
                        st_e += clock64() - ce;
                    }
                    continue;
                }
                // ---------------- general path: K-chunk partials / debug outputs ----------------
                // K-chunk partial sums live in per-CTA int64 scratch, row-major [row][s N_c], so
                // each thread moves 16 consecutive values of its row with 16-byte accesses (all
                // in flight together): a chunk boundary costs a few memory round trips per
                // level, not one per value.
                int64_t *scr_row = scr ? scr + (int64_t)row_local * (S * NC) : nullptr;
                if (scr && !last) {
                    // drain this K chunk: partial (+)= level sums, TMEM zeroed for the next chunk
#pragma unroll 1
                    for (int j = 0; j < S; ++j) {
                        const bool two = T > 1 && j < S - G;
#pragma unroll
                        for (int c0 = 0; c0 < NC; c0 += 16) {
                            const uint32_t col = (uint32_t)(j * NC + c0);
                            uint32_t v[16], v2[16];
                            __syncwarp();
                            ptx::tmem_ld_x16(tmem_base + lane_addr + col, v);
                            if (two) ptx::tmem_ld_x16(tmem_base + lane_addr + P.region_col[1] + col, v2);
                            ptx::tmem_ld_wait();
                            ptx::tmem_st_zero_x16(tmem_base + lane_addr + col);
                            if (two) ptx::tmem_st_zero_x16(tmem_base + lane_addr + P.region_col[1] + col);
                            longlong2 *sp = reinterpret_cast<longlong2 *>(scr_row + col);
                            longlong2 o[8];
#pragma unroll
                            for (int q = 0; q < 8; ++q) o[q] = first ? make_longlong2(0, 0) : sp[q];
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                o[q].x += (long long)(int32_t)v[2 * q] + (two ? (int32_t)v2[2 * q] : 0);
                                o[q].y += (long long)(int32_t)v[2 * q + 1] + (two ? (int32_t)v2[2 * q + 1] : 0);
                                sp[q] = o[q];
                            }
                        }
                    }
                    ptx::tmem_st_wait();
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(&tmem_empty[ab]);
                    if (P.stats) st_e += clock64() - ce;
                    continue;
                }
                double acc[NC];
#pragma unroll
                for (int i = 0; i < NC; ++i) acc[i] = 0.0;
#pragma unroll 1
                for (int j = 0; j < S; ++j) {
                    const bool two = T > 1 && j < S - G;
                    const double sc = pow2(-P.w * (S + 1 - j));
#pragma unroll
                    for (int c0 = 0; c0 < NC; c0 += 16) {
                        const uint32_t col = (uint32_t)(j * NC + c0);
                        uint32_t v[16], v2[16];
                        __syncwarp();
                        ptx::tmem_ld_x16(tmem_base + lane_addr + col, v);
                        if (two) ptx::tmem_ld_x16(tmem_base + lane_addr + P.region_col[1] + col, v2);
                        ptx::tmem_ld_wait();
                        ptx::tmem_st_zero_x16(tmem_base + lane_addr + col);
                        if (two) ptx::tmem_st_zero_x16(tmem_base + lane_addr + P.region_col[1] + col);
                        longlong2 o[8];
                        if (scr && !first) {  // last chunk: the earlier chunks' partials
                            const longlong2 *sp = reinterpret_cast<const longlong2 *>(scr_row + col);
#pragma unroll
                            for (int q = 0; q < 8; ++q) o[q] = sp[q];
                        } else {
#pragma unroll
                            for (int q = 0; q < 8; ++q) o[q] = make_longlong2(0, 0);
                        }
#pragma unroll
                        for (int ii = 0; ii < 16; ++ii) {
                            const int i = c0 + ii;
                            int64_t Lg = (int64_t)(int32_t)v[ii];
                            if (two) Lg += (int64_t)(int32_t)v2[ii];
                            Lg += (ii & 1) ? o[ii >> 1].y : o[ii >> 1].x;
                            if (fp_out) {
                                acc[i] = __fma_rn((double)Lg, sc, acc[i]);
                            } else if (row_ok) {
                                const int64_t colg = nb * NC + i;
                                if (colg < P.n) {
                                    if (P.mode == EPI_LEVELS_I64)
                                        static_cast<int64_t *>(P.out)[(int64_t)(S - 1 - j) * P.m * P.n +
                                                                      row + colg * P.m] = Lg;
                                    else
                                        static_cast<int32_t *>(P.out)[row + colg * P.m] = (int32_t)Lg;
                                }
                            }
                        }
                    }
                }
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                ptx::mbar_arrive(&tmem_empty[ab]);
                if (last && fp_out && row_ok) store_row<NC>(P, acc, ebt, ea, row, nb);
                if (P.stats) st_e += clock64() - ce;
            }
        }
        if (P.stats && warp == 0 && lane == 0) {
            P.stats[(int64_t)blockIdx.x * kStatSlots + ST_EPI_BUSY] = st_e;
            P.stats[(int64_t)blockIdx.x * kStatSlots + ST_EPI_TMEM] = st_et;
            P.stats[(int64_t)blockIdx.x * kStatSlots + ST_EPI_STORE] = st_es;
        }
    }
    if (P.cl > 1) ptx::cluster_sync();
    else __syncthreads();
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

inline PFN_encodeTiled get_encode() {
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
// plane_rows (>= rows, 0 = rows): rows per plane in memory, so a window of rows of a larger
// buffer (a column chunk of a B-slice buffer) can be addressed in place.
inline bool make_map(CUtensorMap *map, const int8_t *base, int64_t k_pad, int64_t rows, int s,
              uint32_t box_rows, uint32_t box_s, int64_t plane_rows = 0) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    if (plane_rows < rows) plane_rows = rows;
    cuuint64_t dims[3] = {(cuuint64_t)k_pad, (cuuint64_t)rows, (cuuint64_t)s};
    cuuint64_t strides[2] = {(cuuint64_t)k_pad, (cuuint64_t)(k_pad * plane_rows)};
    cuuint32_t box[3] = {(cuuint32_t)kKB, box_rows, box_s};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t *>(base), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int S, int NCV = nc_for(S)>
cudaError_t launch_t(const GemmArgs &a, const GemmPlan &p, EpiMode mode, cudaStream_t st) {
    constexpr int NC = NCV;
    auto kern = k_oz_gemm<S, NCV>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
    if (e != cudaSuccess) return e;
    // CTA pairs (clusters of 2) sharing the A tiles by TMA multicast: each CTA loads half of
    // every A-slice tile and multicasts it to both, halving the A bytes per SM from L2 (the
    // larger operand stream: 128 rows x s slices per k-block vs NC x s for B).  Measured at
    // 16384^3, s = 9: +1.7% (less L2 traffic -> more clock under the power cap).  Pairs take
    // column tiles (2j, 2j+1); an odd column-tile count leaves one dummy tile per row block,
    // so pairs are used only when that waste is small.  OZIMMU_CLUSTER=1 forces single CTAs;
    // OZIMMU_CLUSTER=4 takes 2 x 2 clusters (B tiles multicast down the row-block pair too).
#ifndef OZ_CLUSTER_DEFAULT
#define OZ_CLUSTER_DEFAULT 2
#endif
    static const int cl_env =
        getenv("OZIMMU_CLUSTER") ? atoi(getenv("OZIMMU_CLUSTER")) : OZ_CLUSTER_DEFAULT;
    const int64_t tiles_m = ceil_div(a.m, kBlockM), tiles_n = ceil_div(a.n, NC);
    // a dimension is split over the cluster only when the dummy tiles it leaves are few
    auto splits = [](int64_t tiles) { return tiles >= 2 && (tiles % 2 == 0 || tiles >= 32); };
    int clm = 1, cln = 1;
    if (cl_env >= 2 && splits(tiles_n)) cln = 2;
    if (cl_env >= 4 && cln == 2 && splits(tiles_m)) clm = 2;
    // experiments: OZIMMU_CLUSTER_N / _M set the cluster shape directly (e.g. 4 x 1: A tiles
    // multicast to four CTAs of a row block)
    static const int cln_env = getenv("OZIMMU_CLUSTER_N") ? atoi(getenv("OZIMMU_CLUSTER_N")) : 0;
    static const int clm_env = getenv("OZIMMU_CLUSTER_M") ? atoi(getenv("OZIMMU_CLUSTER_M")) : 0;
    if (cln_env == 1 || cln_env == 2 || cln_env == 4) cln = cln_env;
    if (clm_env == 1 || clm_env == 2) clm = clm_env;
    if (clm * cln > 4) clm = 1;
    int cl = clm * cln;
    if (p.grid < cl) clm = cln = cl = 1;
    int grid = p.grid;
    cudaLaunchAttribute attr[1];
    if (cl > 1) {
        int dev = 0;
        cudaGetDevice(&dev);
        static int maxc_cache[64][33][5];
        int &maxc = maxc_cache[dev & 63][S][cl];
        if (maxc == 0) {
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3((unsigned)(p.grid / cl * cl));
            q.blockDim = dim3(kThreads);
            q.dynamicSmemBytes = p.smem_bytes;
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = cl;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            q.attrs = attr;
            q.numAttrs = 1;
            if (cudaOccupancyMaxActiveClusters(&maxc, kern, &q) != cudaSuccess || maxc < 1) {
                cudaGetLastError();
                maxc = -1;
            }
        }
        const int64_t units = ceil_div(tiles_m, clm) * ceil_div(tiles_n, cln);
        if (maxc < 1) {
            clm = cln = cl = 1;
        } else {
            int64_t c = maxc < p.grid / cl ? maxc : p.grid / cl;
            if (!p.sk) c = c < units ? c : units;  // stream-K: clusters share units' K loops
            grid = (int)(cl * c);
        }
    }
    CUtensorMap tmA, tmB;
    if (!make_map(&tmA, a.a_planes, a.k_pad, a.m, a.s, (uint32_t)(kBlockM / cln), 1,
                  a.a_plane_rows))
        return cudaErrorInvalidValue;
    // B: one box of all s slices, or (clm > 1) one box of NC/clm columns per slice
    if (!make_map(&tmB, a.b_planes, a.k_pad, a.n, a.s, (uint32_t)(NC / clm),
                  clm == 1 ? (uint32_t)a.s : 1u, a.b_plane_rows))
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
    P.alpha_im = a.alpha_im;
    P.beta_im = a.beta_im;
    P.EA = a.EA;
    P.EB = a.EB;
    P.C = a.C;
    P.ldc = a.ldc;
    P.c_rows = a.c_rows;
    P.c_cols = a.c_cols;
    P.out = a.out;
    P.scratch = p.k_chunks > 1 ? a.chunk_scratch : nullptr;
    P.wave_counter = a.wave_counter;
    P.sk = (p.sk && p.k_chunks == 1 && a.chunk_scratch) ? 1 : 0;
    P.sk_total = 0;
    P.sk_count = nullptr;
    P.sk_part = nullptr;
    P.used_cols = (uint32_t)((p.T == 2 ? 2 * S - p.G : S) * NC);
    P.nacc = p.nacc;
    P.acc_stride = (uint32_t)(p.tmem_cols / 2);
    P.stats = a.stats;
    P.G = p.G;
    P.T = p.T;
    P.region_col[0] = 0;
    P.region_col[1] = (uint32_t)(S * NC);
    P.cl = cl;
    P.clm = clm;
    P.cln = cln;
    P.units_m = ceil_div(P.tiles_m, clm);
    P.units_n = ceil_div(P.tiles_n, cln);
    P.num_units = P.units_m * P.units_n;
    P.full_waves = P.num_units / (grid / cl);
    static const int lag_env = getenv("OZIMMU_WAVE_LAG") ? atoi(getenv("OZIMMU_WAVE_LAG")) : 0;
    P.wave_lag = lag_env > 0 ? lag_env : 0;
    static const int ksync_env = getenv("OZIMMU_KSYNC") ? atoi(getenv("OZIMMU_KSYNC")) : 0;
    P.ksync = ksync_env > 0 ? ksync_env : 0;
    if (P.sk) {
        // stream-K: no per-wave barrier (no waves); counters zeroed, partials in the scratch
        P.wave_counter = nullptr;
        P.sk_total = P.num_units * P.num_k_blocks;
        P.sk_count = reinterpret_cast<int *>(a.chunk_scratch);
        const size_t cnt = sk_counters_bytes(P.num_units * cl);
        P.sk_part = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(a.chunk_scratch) + cnt);
        e = cudaMemsetAsync(P.sk_count, 0, cnt, st);
        if (e != cudaSuccess) return e;
    }
    if (P.wave_counter && !a.counter_zeroed) {
        e = cudaMemsetAsync(P.wave_counter, 0, sizeof(unsigned int), st);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = p.smem_bytes;
    cfg.stream = st;
    cudaLaunchAttribute la[2];
    int na = 0;
    if (cl > 1) {
        la[na].id = cudaLaunchAttributeClusterDimension;
        la[na].val.clusterDim.x = cl;
        la[na].val.clusterDim.y = 1;
        la[na].val.clusterDim.z = 1;
        ++na;
    }
    // programmatic dependent launch: CTAs may start their set-up (barriers, TMEM, descriptor
    // prefetch) while the previous kernel drains; k_oz_gemm waits (griddepcontrol.wait) before
    // its first global access.  OZIMMU_NO_PDL=1 turns it off (experiments).
    static const bool no_pdl = getenv("OZIMMU_NO_PDL") != nullptr;
    if (!no_pdl) {
        la[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        la[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = na ? la : nullptr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, tmA, tmB, P);
}

}  // namespace gemm_detail
}  // namespace ozimmu
