// split.cu -- A2 (exponent scan) + A3 (slicing) of the Ozaki scheme on sm_100a.
//
// SplitInt, Alg. 4: per row of op(A) / column of op(B) a shared
// power-of-two scale 2^E (E = frexp exponent of the max |x|, reading A3), then
// s signed INT8 digits d_p = sgn(x) * (floor(|x| 2^(w p - E)) mod 2^w) (readings
// A4/A5).  The paper's implementation "uses bit operations to cut the mantissa"
// (P:530); so do we: everything below is integer arithmetic on the IEEE-754 bit
// pattern, |x| = M * 2^e0 with M the (sub)normal significand.
//
// HBM-bound: read 8 B/element (16 B when the rows are strided and need a separate
// exponent pass), write s B/element.  128-bit loads, 64-bit stores, grids sized
// in multiples of the SM count.
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace ozimmu {
namespace {

// E-candidate of one element: frexp exponent of |x| (x != 0), kExpNonFinite for
// NaN/Inf, kKeyEmpty for +-0.  max() over a vector gives its E (or a marker).
__device__ __forceinline__ int32_t exp_key(double x) {
    const uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
    const int be = static_cast<int>((u >> 52) & 0x7FF);
    const uint64_t fr = u & ((1ull << 52) - 1);
    if (be == 0x7FF) return kExpNonFinite;
    if (be != 0) return be - 1022;                  // |x| in [2^(be-1023), 2^(be-1022))
    if (fr != 0) return -1010 - __clzll(fr);         // subnormal: floor(log2|x|) + 1
    return kKeyEmpty;
}

__device__ __forceinline__ int32_t key_to_exp(int32_t key) {
    return key == kKeyEmpty ? 0 : key;  // all-zero vector: E = 0 (reading A11)
}

// s digits of x (scale 2^E, width w) packed into out[p] byte `lane` (little endian).
// Only called with E finite and |x| < 2^E.
template <int MAXS>
__device__ __forceinline__ void digits_of(double x, int32_t E, int s, int w, int lane,
                                          uint64_t (&out)[MAXS]) {
    const uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
    const int be = static_cast<int>((u >> 52) & 0x7FF);
    const uint64_t fr = u & ((1ull << 52) - 1);
    const bool neg = (u >> 63) != 0;
    const uint64_t M = be ? (fr | (1ull << 52)) : fr;  // |x| = M 2^e0
    const int e0 = be ? be - 1075 : -1074;
    const int t0 = e0 - E;                              // sh_p = t0 + w p
    const uint64_t mask = (1ull << w) - 1;
#pragma unroll
    for (int p = 0; p < MAXS; ++p) {
        if (p < s) {
            const int sh = t0 + w * (p + 1);
            uint64_t v;
            if (sh >= 0) v = sh >= 64 ? 0 : (M << sh);
            else v = (-sh) >= 64 ? 0 : (M >> (-sh));
            int d = static_cast<int>(v & mask);
            d = neg ? -d : d;
            out[p] |= static_cast<uint64_t>(static_cast<uint8_t>(static_cast<int8_t>(d)))
                      << (8 * lane);
        }
    }
}

// ---------------------------------------------------------------------------------
// Contiguous vectors (row of op(A) with transA = T, column of op(B) with transB = N):
// TPR threads per vector, one pass for the exponent (max reduction), one pass for
// the digits (the second read of a <= 128 KB row hits L2).
// ---------------------------------------------------------------------------------
template <int TPR, int MAXS>
__global__ void __launch_bounds__(256) k_split_contig(const double *__restrict__ M, int64_t ld,
                                                      int64_t rows, int64_t kdim, int64_t k_pad,
                                                      int s, int w, int reverse,
                                                      int8_t *__restrict__ planes,
                                                      int64_t plane_stride, int32_t *__restrict__ E) {
    constexpr int VPB = 256 / TPR;  // vectors per block
    __shared__ int32_t red[256 / 32];
    const int sub = threadIdx.x / TPR;
    const int t = threadIdx.x % TPR;
    const int64_t r = static_cast<int64_t>(blockIdx.x) * VPB + sub;
    const bool active = r < rows;
    const double *v = M + (active ? r : 0) * ld;
    const bool al16 = ((reinterpret_cast<uintptr_t>(v) & 15) == 0);
    const int64_t nchunk = k_pad / 8;

    // ---- pass 1: E = max exponent key ----
    int32_t key = kKeyEmpty;
    if (active) {
        for (int64_t c = t; c < nchunk; c += TPR) {
            const int64_t l0 = c * 8;
            double x[8];
            if (al16 && l0 + 8 <= kdim) {
                const double2 *q = reinterpret_cast<const double2 *>(v + l0);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    double2 d2 = __ldg(q + i);
                    x[2 * i] = d2.x;
                    x[2 * i + 1] = d2.y;
                }
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) x[i] = (l0 + i < kdim) ? __ldg(v + l0 + i) : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) key = max(key, exp_key(x[i]));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffff, key, o));
    if (TPR > 32) {
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = key;
        __syncthreads();
        key = red[0];
#pragma unroll
        for (int i = 1; i < TPR / 32; ++i) key = max(key, red[i]);
    }
    if (!active) return;
    const int32_t Ev = key_to_exp(key);
    if (t == 0) E[r] = Ev;
    const bool bad = Ev == kExpNonFinite;

    // ---- pass 2: digits ----
    for (int64_t c = t; c < nchunk; c += TPR) {
        const int64_t l0 = c * 8;
        uint64_t out[MAXS];
#pragma unroll
        for (int p = 0; p < MAXS; ++p) out[p] = 0;
        if (!bad) {
            double x[8];
            if (al16 && l0 + 8 <= kdim) {
                const double2 *q = reinterpret_cast<const double2 *>(v + l0);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    double2 d2 = __ldg(q + i);
                    x[2 * i] = d2.x;
                    x[2 * i + 1] = d2.y;
                }
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) x[i] = (l0 + i < kdim) ? __ldg(v + l0 + i) : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (x[i] != 0.0) digits_of<MAXS>(x[i], Ev, s, w, i, out);
        }
#pragma unroll
        for (int p = 0; p < MAXS; ++p) {
            if (p < s) {
                const int pidx = reverse ? (s - 1 - p) : p;
                *reinterpret_cast<uint64_t *>(planes + pidx * plane_stride + r * k_pad + l0) = out[p];
            }
        }
    }
}

// ---------------------------------------------------------------------------------
// Strided vectors (row of op(A) with transA = N, column of op(B) with transB = T):
// element l of vector r at M[r + l*ld]; consecutive vectors are consecutive in memory.
// ---------------------------------------------------------------------------------

// Pass 1: one thread per vector, a slice of l per blockIdx.y; atomicMax of the key.
__global__ void __launch_bounds__(256) k_expscan_strided(const double *__restrict__ M, int64_t ld,
                                                         int64_t rows, int64_t kdim, int64_t lchunk,
                                                         int32_t *__restrict__ keys) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
    if (r >= rows) return;
    const int64_t l0 = static_cast<int64_t>(blockIdx.y) * lchunk;
    const int64_t l1 = min(kdim, l0 + lchunk);
    int32_t key = kKeyEmpty;
    int64_t l = l0;
    for (; l + 8 <= l1; l += 8) {
        double x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(M + r + (l + i) * ld);
#pragma unroll
        for (int i = 0; i < 8; ++i) key = max(key, exp_key(x[i]));
    }
    for (; l < l1; ++l) key = max(key, exp_key(__ldg(M + r + l * ld)));
    if (key != kKeyEmpty) atomicMax(keys + r, key);
}

// Pass 2: 64 vectors x 64 elements per block, transposed through shared memory.
template <int MAXS>
__global__ void __launch_bounds__(256) k_split_strided(const double *__restrict__ M, int64_t ld,
                                                       int64_t rows, int64_t kdim, int64_t k_pad,
                                                       int s, int w, int reverse,
                                                       const int32_t *__restrict__ keys,
                                                       int8_t *__restrict__ planes,
                                                       int64_t plane_stride,
                                                       int32_t *__restrict__ E) {
    __shared__ double tile[64][65];  // [l][r]
    __shared__ int32_t exps[64];
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 64;
    const int64_t l0 = static_cast<int64_t>(blockIdx.y) * 64;
    const int tid = threadIdx.x;
    if (tid < 64) {
        const int64_t r = r0 + tid;
        int32_t e = 0;
        if (r < rows) {
            e = key_to_exp(keys[r]);
            if (blockIdx.y == 0) E[r] = e;
        }
        exps[tid] = e;
    }
    // coalesced load: warp reads 32 consecutive vectors at one l
#pragma unroll 4
    for (int i = 0; i < 16; ++i) {
        const int rr = tid & 63;
        const int ll = (tid >> 6) + 4 * i;
        const int64_t r = r0 + rr, l = l0 + ll;
        tile[ll][rr] = (r < rows && l < kdim) ? __ldg(M + r + l * ld) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int task = tid; task < 512; task += 256) {
        const int rr = task & 63;
        const int l8 = task >> 6;  // 0..7
        const int64_t r = r0 + rr;
        const int64_t lb = l0 + l8 * 8;
        if (r >= rows || lb >= k_pad) continue;
        const int32_t Ev = exps[rr];
        uint64_t out[MAXS];
#pragma unroll
        for (int p = 0; p < MAXS; ++p) out[p] = 0;
        if (Ev != kExpNonFinite) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const double x = tile[l8 * 8 + i][rr];
                if (x != 0.0) digits_of<MAXS>(x, Ev, s, w, i, out);
            }
        }
#pragma unroll
        for (int p = 0; p < MAXS; ++p) {
            if (p < s) {
                const int pidx = reverse ? (s - 1 - p) : p;
                *reinterpret_cast<uint64_t *>(planes + pidx * plane_stride + r * k_pad + lb) = out[p];
            }
        }
    }
}

template <int MAXS>
cudaError_t launch_split_t(const double *M, int64_t ld, bool contiguous, int64_t rows,
                           int64_t kdim, int64_t k_pad, int s, int w, bool reverse,
                           int8_t *planes, int64_t plane_stride, int32_t *E,
                           int32_t *key_scratch, int num_sms, cudaStream_t st, int *launches) {
    if (contiguous) {
        if (k_pad >= 2048) {
            const int64_t blocks = rows;
            k_split_contig<256, MAXS><<<(unsigned)blocks, 256, 0, st>>>(
                M, ld, rows, kdim, k_pad, s, w, reverse, planes, plane_stride, E);
        } else {
            const int64_t blocks = ceil_div(rows, 8);
            k_split_contig<32, MAXS><<<(unsigned)blocks, 256, 0, st>>>(
                M, ld, rows, kdim, k_pad, s, w, reverse, planes, plane_stride, E);
        }
        ++*launches;
        return cudaGetLastError();
    }
    // strided: exponent scan then transposing slice
    cudaError_t e = cudaMemsetAsync(key_scratch, 0x80, sizeof(int32_t) * rows, st);
    if (e != cudaSuccess) return e;
    const int64_t rblocks = ceil_div(rows, 256);
    int64_t ysplit = ceil_div(4 * (int64_t)num_sms, rblocks);
    ysplit = ysplit < 1 ? 1 : ysplit;
    int64_t lchunk = round_up(ceil_div(kdim, ysplit), 8);
    if (lchunk < 64) lchunk = 64;
    ysplit = ceil_div(kdim, lchunk);
    if (ysplit < 1) ysplit = 1;
    k_expscan_strided<<<dim3((unsigned)rblocks, (unsigned)ysplit), 256, 0, st>>>(
        M, ld, rows, kdim, lchunk, key_scratch);
    ++*launches;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    k_split_strided<MAXS><<<dim3((unsigned)ceil_div(rows, 64), (unsigned)ceil_div(k_pad, 64)), 256,
                            0, st>>>(M, ld, rows, kdim, k_pad, s, w, reverse, key_scratch, planes,
                                     plane_stride, E);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_split(const double *M, int64_t ld, bool contiguous, int64_t rows, int64_t kdim,
                         int64_t k_pad, int s, int w, bool reverse, int8_t *planes,
                         int64_t plane_stride, int32_t *E, int32_t *key_scratch, int num_sms,
                         cudaStream_t st, int *launches) {
    if (rows <= 0) return cudaSuccess;
    if (s <= 8)
        return launch_split_t<8>(M, ld, contiguous, rows, kdim, k_pad, s, w, reverse, planes,
                                 plane_stride, E, key_scratch, num_sms, st, launches);
    if (s <= 16)
        return launch_split_t<16>(M, ld, contiguous, rows, kdim, k_pad, s, w, reverse, planes,
                                  plane_stride, E, key_scratch, num_sms, st, launches);
    return launch_split_t<32>(M, ld, contiguous, rows, kdim, k_pad, s, w, reverse, planes,
                              plane_stride, E, key_scratch, num_sms, st, launches);
}

}  // namespace ozimmu
