// auto.cu -- NEXT row f2: INT8-AUTO split selection (Discussion P:713-734).
//
// "Before a GEMM computation, we check all the elements of the input matrices and
// determine the appropriate number of splits ... so that the average mantissa loss in the
// splitting process is equal to or smaller than a threshold T".  Reading A17:
// for a nonzero finite x in a vector with exponent E, the significant bits of |x|/2^E sit
// at positions lead = E - ilogb(x) .. t_last = lead + vlen - 1 (vlen: bits from the MSB to
// the last 1 of the significand); s slices of w bits keep positions 1..s*w, so
//     loss_s(x) = min(vlen, max(0, t_last - s*w)).
// These kernels accumulate, for s = 1..s_max, the exact integer sum of loss_s over the
// nonzero finite elements of the rows of op(A) / columns of op(B), plus their count; the
// host then picks the smallest s whose mean loss is <= T for both operands.
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace ozimmu {
namespace {

constexpr int kMaxS = 32;

__device__ __forceinline__ int32_t exp_key_a(double x) {  // as split.cu's exp_key
    const uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
    const int be = static_cast<int>((u >> 52) & 0x7FF);
    const uint64_t fr = u & ((1ull << 52) - 1);
    if (be == 0x7FF) return kExpNonFinite;
    if (be != 0) return be - 1022;
    if (fr != 0) return -1010 - __clzll(fr);
    return kKeyEmpty;
}

// (t_last, vlen) of a nonzero finite x relative to the vector exponent E.
__device__ __forceinline__ void bit_span(double x, int32_t E, int &t_last, int &vlen) {
    const uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
    const int be = static_cast<int>((u >> 52) & 0x7FF);
    const uint64_t fr = u & ((1ull << 52) - 1);
    const uint64_t M = be ? (fr | (1ull << 52)) : fr;   // |x| = M 2^e0, M != 0
    const int e0 = be ? be - 1075 : -1074;
    const int msb = 63 - __clzll(M);                     // ilogb(x) = e0 + msb
    const int tz = __ffsll(static_cast<long long>(M)) - 1;
    vlen = msb - tz + 1;
    t_last = E - (e0 + tz);                              // position of the lowest set bit
}

template <int S_MAX>
__device__ __forceinline__ void add_loss(double x, int32_t E, int w, int s_max,
                                         uint32_t (&acc)[S_MAX], uint32_t &cnt) {
    if (x == 0.0) return;
    int t_last, vlen;
    bit_span(x, E, t_last, vlen);
    ++cnt;
#pragma unroll
    for (int s = 1; s <= S_MAX; ++s) {
        if (s > s_max) break;
        int over = t_last - s * w;
        over = over < 0 ? 0 : (over > vlen ? vlen : over);
        acc[s - 1] += (uint32_t)over;
    }
}

// Block-reduce the per-thread sums and add them to out[0..s_max) (int64) and out[kMaxS].
template <int S_MAX>
__device__ __forceinline__ void flush(const uint32_t (&acc)[S_MAX], uint32_t cnt, int s_max,
                                      unsigned long long *out) {
    __shared__ unsigned long long red[S_MAX + 1];
    if (threadIdx.x <= S_MAX) red[threadIdx.x] = 0;
    __syncthreads();
#pragma unroll
    for (int s = 0; s < S_MAX; ++s) {
        if (s >= s_max) break;
        unsigned long long v = acc[s];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&red[s], v);
    }
    unsigned long long c = cnt;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffff, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&red[S_MAX], c);
    __syncthreads();
    if (threadIdx.x < (unsigned)s_max && red[threadIdx.x]) atomicAdd(&out[threadIdx.x], red[threadIdx.x]);
    if (threadIdx.x == 0 && red[S_MAX]) atomicAdd(&out[kMaxS], red[S_MAX]);
}

// Contiguous vectors: one 256-thread block per vector; pass 1 exponent, pass 2 losses.
__global__ void __launch_bounds__(256) k_loss_contig(const double *__restrict__ M, int64_t ld,
                                                     int64_t rows, int64_t kdim, int w, int s_max,
                                                     unsigned long long *__restrict__ out) {
    __shared__ int32_t kred[8];
    const int64_t r = blockIdx.x;
    const double *v = M + r * ld;
    int32_t key = kKeyEmpty;
    for (int64_t l = threadIdx.x; l < kdim; l += 256) key = max(key, exp_key_a(__ldg(v + l)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffff, key, o));
    if ((threadIdx.x & 31) == 0) kred[threadIdx.x >> 5] = key;
    __syncthreads();
    key = kred[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) key = max(key, kred[i]);
    uint32_t acc[kMaxS];
#pragma unroll
    for (int s = 0; s < kMaxS; ++s) acc[s] = 0;
    uint32_t cnt = 0;
    if (key != kExpNonFinite && key != kKeyEmpty) {  // non-finite / zero vectors: no loss
        for (int64_t l = threadIdx.x; l < kdim; l += 256) add_loss<kMaxS>(__ldg(v + l), key, w, s_max, acc, cnt);
    }
    flush<kMaxS>(acc, cnt, s_max, out);
}

// Strided vectors (element l of vector r at M[r + l ld]; complex: the (re, im) pair at
// 2 (r + l ld)): one thread per vector and a slice of l per blockIdx.y; the exponent comes
// from keys.
template <int CPX>
__global__ void __launch_bounds__(256) k_loss_strided(const double *__restrict__ M, int64_t ld,
                                                      int64_t rows, int64_t kdim, int64_t lchunk,
                                                      const int32_t *__restrict__ keys, int w,
                                                      int s_max, unsigned long long *__restrict__ out) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
    uint32_t acc[kMaxS];
#pragma unroll
    for (int s = 0; s < kMaxS; ++s) acc[s] = 0;
    uint32_t cnt = 0;
    if (r < rows) {
        const int32_t key = keys[r];
        if (key != kExpNonFinite && key != kKeyEmpty) {
            const int64_t l0 = static_cast<int64_t>(blockIdx.y) * lchunk;
            const int64_t l1 = min(kdim, l0 + lchunk);
            for (int64_t l = l0; l < l1; ++l) {
                if (CPX) {
                    const double2 z = __ldg(reinterpret_cast<const double2 *>(M) + r + l * ld);
                    add_loss<kMaxS>(z.x, key, w, s_max, acc, cnt);
                    add_loss<kMaxS>(z.y, key, w, s_max, acc, cnt);
                } else {
                    add_loss<kMaxS>(__ldg(M + r + l * ld), key, w, s_max, acc, cnt);
                }
            }
        }
    }
    flush<kMaxS>(acc, cnt, s_max, out);
}

template <int CPX>
__global__ void k_expscan_strided_a(const double *__restrict__ M, int64_t ld, int64_t rows,
                                    int64_t kdim, int64_t lchunk, int32_t *__restrict__ keys) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
    if (r >= rows) return;
    const int64_t l0 = static_cast<int64_t>(blockIdx.y) * lchunk;
    const int64_t l1 = min(kdim, l0 + lchunk);
    int32_t key = kKeyEmpty;
    for (int64_t l = l0; l < l1; ++l) {
        if (CPX) {
            const double2 z = __ldg(reinterpret_cast<const double2 *>(M) + r + l * ld);
            key = max(key, max(exp_key_a(z.x), exp_key_a(z.y)));
        } else {
            key = max(key, exp_key_a(__ldg(M + r + l * ld)));
        }
    }
    if (key != kKeyEmpty) atomicMax(keys + r, key);
}

}  // namespace

// out: device uint64 [kMaxS + 1] (loss sums for s = 1..s_max, then the nonzero count),
// accumulated (caller zeroes it).  key_scratch: int32 [rows] (strided case).  cpx: the
// vectors are complex (kdim counts complex elements in the strided case, doubles in the
// contiguous one; the loss depends only on the magnitudes, so rows of A-hat / columns of
// B-hat of reading A16 have the statistics of their complex vectors).
cudaError_t launch_mantissa_loss(const double *M, int64_t ld, bool contiguous, int64_t rows,
                                 int64_t kdim, int w, int s_max, unsigned long long *out,
                                 int32_t *key_scratch, int num_sms, cudaStream_t st,
                                 int *launches, int cpx) {
    if (rows <= 0 || kdim <= 0) return cudaSuccess;
    if (s_max < 1 || s_max > kMaxS) return cudaErrorInvalidValue;
    if (contiguous) {
        k_loss_contig<<<(unsigned)rows, 256, 0, st>>>(M, ld, rows, kdim, w, s_max, out);
        ++*launches;
        return cudaGetLastError();
    }
    cudaError_t e = cudaMemsetAsync(key_scratch, 0x80, sizeof(int32_t) * rows, st);
    if (e != cudaSuccess) return e;
    const int64_t rblocks = ceil_div(rows, 256);
    int64_t ysplit = ceil_div(4 * (int64_t)num_sms, rblocks);
    if (ysplit < 1) ysplit = 1;
    int64_t lchunk = ceil_div(kdim, ysplit);
    if (lchunk < 64) lchunk = 64;
    ysplit = ceil_div(kdim, lchunk);
    if (cpx)
        k_expscan_strided_a<1><<<dim3((unsigned)rblocks, (unsigned)ysplit), 256, 0, st>>>(
            M, ld, rows, kdim, lchunk, key_scratch);
    else
        k_expscan_strided_a<0><<<dim3((unsigned)rblocks, (unsigned)ysplit), 256, 0, st>>>(
            M, ld, rows, kdim, lchunk, key_scratch);
    ++*launches;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (cpx)
        k_loss_strided<1><<<dim3((unsigned)rblocks, (unsigned)ysplit), 256, 0, st>>>(
            M, ld, rows, kdim, lchunk, key_scratch, w, s_max, out);
    else
        k_loss_strided<0><<<dim3((unsigned)rblocks, (unsigned)ysplit), 256, 0, st>>>(
            M, ld, rows, kdim, lchunk, key_scratch, w, s_max, out);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace ozimmu
