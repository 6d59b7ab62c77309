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
//
// Evaluation (exact, no loop over s per element).  With l = t_last - vlen,
//     loss_s(x) = max(0, t_last - s w) - max(0, l - s w)
// (min(max(0, a), v) = max(0, a) - max(0, a - v) for v >= 0), and for an integer y,
// max(0, y - s w) > 0 exactly for 1 <= s <= q(y) = (y - 1) div w (y >= 1), so
//     sum_x loss_s(x) = F(s),  F(s) = sum_{y: q(y) >= s} c_y y  -  s w sum_{y: q(y) >= s} c_y
// over the multiset of y = t_last (c = +1) and y = l (c = -1).  Each thread bins its
// elements by q' = min(q, s_max) into a signed count and a signed sum held in its own
// shared-memory column; suffix sums over q' give its F(s) for every s.
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

// L2 eviction priority of the two passes over a contiguous vector (as split.cu): the exponent
// pass keeps the vector in L2 for the statistics pass, which reads it for the last time.
__device__ __forceinline__ uint64_t l2_pol(bool keep) {
    uint64_t p;
    if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ldg_pol(const double *q, uint64_t pol) {
    double r;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(q), "l"(pol));
    return r;
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

// Per-thread histogram columns in dynamic shared memory:
//   cnt[q' - 1][tid], ysum[q' - 1][tid] (int32, q' = 1..s_max), then the division table
//   qtab[y - 1] = min((y - 1) div w, s_max) for y - 1 in [0, s_max w].
struct LossHist {
    int32_t *cnt, *ysum;
    const uint8_t *qtab;
    int w, s_max, lim;
    uint32_t nnz;

    __device__ __forceinline__ void bin(int y, int c) {
        if (y <= w) return;  // q(y) = 0: no s >= 1 sees it
        const int q = qtab[min(y - 1, lim)];
        const int i = (q - 1) * blockDim.x + threadIdx.x;
        cnt[i] += c;
        ysum[i] += c * y;
    }
    __device__ __forceinline__ void add(double x, int32_t E) {
        if (x == 0.0) return;
        int t_last, vlen;
        bit_span(x, E, t_last, vlen);
        ++nnz;
        bin(t_last, 1);
        bin(t_last - vlen, -1);
    }
};

__device__ __forceinline__ LossHist hist_init(int w, int s_max) {
    extern __shared__ int32_t sh[];
    LossHist H;
    H.cnt = sh;
    H.ysum = sh + s_max * blockDim.x;
    uint8_t *qt = reinterpret_cast<uint8_t *>(sh + 2 * s_max * blockDim.x);
    H.w = w;
    H.s_max = s_max;
    H.lim = s_max * w;
    H.nnz = 0;
    for (int i = threadIdx.x; i <= H.lim; i += blockDim.x) qt[i] = (uint8_t)min(i / w, s_max);
    for (int q = 0; q < s_max; ++q) {
        H.cnt[q * blockDim.x + threadIdx.x] = 0;
        H.ysum[q * blockDim.x + threadIdx.x] = 0;
    }
    H.qtab = qt;
    __syncthreads();
    return H;
}

size_t hist_smem(int s_max, int threads, int w) {
    return sizeof(int32_t) * 2 * (size_t)s_max * threads + (size_t)(s_max * w + 16);
}

// Suffix sums -> this thread's F(s) for each s, block-reduced into out[0..s_max) (uint64)
// and out[kMaxS] (count of nonzero finite elements).  F(s) of one thread is a sum of
// per-element losses, hence >= 0.
__device__ __forceinline__ void hist_flush(const LossHist &H, unsigned long long *out) {
    __shared__ unsigned long long red[kMaxS + 1];
    if (threadIdx.x <= kMaxS) red[threadIdx.x] = 0;
    __syncthreads();
    long long C = 0, Y = 0;
    for (int q = H.s_max; q >= 1; --q) {
        C += H.cnt[(q - 1) * blockDim.x + threadIdx.x];
        Y += H.ysum[(q - 1) * blockDim.x + threadIdx.x];
        unsigned long long v = (unsigned long long)(Y - (long long)q * H.w * C);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&red[q - 1], v);
    }
    unsigned long long c = H.nnz;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffff, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&red[kMaxS], c);
    __syncthreads();
    if (threadIdx.x < (unsigned)H.s_max && red[threadIdx.x])
        atomicAdd(&out[threadIdx.x], red[threadIdx.x]);
    if (threadIdx.x == 0 && red[kMaxS]) atomicAdd(&out[kMaxS], red[kMaxS]);
}

// Contiguous vectors: persistent 256-thread blocks, one vector at a time (pass 1 its
// exponent, pass 2 the histogram; the second read hits L2); one flush per block.
__global__ void __launch_bounds__(256) k_loss_contig(const double *__restrict__ M, int64_t ld,
                                                     int64_t rows, int64_t kdim, int w, int s_max,
                                                     unsigned long long *__restrict__ out) {
    __shared__ int32_t kred[8];
    LossHist H = hist_init(w, s_max);
    const uint64_t keep = l2_pol(true), strm = l2_pol(false);
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const double *v = M + r * ld;
        int32_t key = kKeyEmpty;
        int64_t l = threadIdx.x;
        for (; l + 3 * 256 < kdim; l += 4 * 256) {
            double x[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = ldg_pol(v + l + i * 256, keep);
#pragma unroll
            for (int i = 0; i < 4; ++i) key = max(key, exp_key_a(x[i]));
        }
        for (; l < kdim; l += 256) key = max(key, exp_key_a(ldg_pol(v + l, keep)));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffff, key, o));
        if ((threadIdx.x & 31) == 0) kred[threadIdx.x >> 5] = key;
        __syncthreads();
        key = kred[0];
#pragma unroll
        for (int i = 1; i < 8; ++i) key = max(key, kred[i]);
        __syncthreads();  // kred is rewritten for the next vector
        if (key == kExpNonFinite || key == kKeyEmpty) continue;  // non-finite / zero: no loss
        l = threadIdx.x;
        for (; l + 3 * 256 < kdim; l += 4 * 256) {
            double x[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = ldg_pol(v + l + i * 256, strm);
#pragma unroll
            for (int i = 0; i < 4; ++i) H.add(x[i], key);
        }
        for (; l < kdim; l += 256) H.add(ldg_pol(v + l, strm), key);
    }
    hist_flush(H, out);
}

// Strided vectors (element l of vector r at M[r + l ld]; complex: the (re, im) pair at
// 2 (r + l ld)): one thread per vector and a slice of l per blockIdx.y; the exponent comes
// from keys (launch_expscan).
template <int CPX>
__global__ void __launch_bounds__(256) k_loss_strided(const double *__restrict__ M, int64_t ld,
                                                      int64_t rows, int64_t kdim, int64_t lchunk,
                                                      const int32_t *__restrict__ keys, int w,
                                                      int s_max, unsigned long long *__restrict__ out) {
    LossHist H = hist_init(w, s_max);
    const int64_t r = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
    const int32_t key = r < rows ? keys[r] : kKeyEmpty;
    if (key != kExpNonFinite && key != kKeyEmpty) {
        const int64_t l0 = static_cast<int64_t>(blockIdx.y) * lchunk;
        const int64_t l1 = min(kdim, l0 + lchunk);
        int64_t l = l0;
        if (CPX) {
            const double2 *Mc = reinterpret_cast<const double2 *>(M);
            for (; l + 4 <= l1; l += 4) {
                double2 z[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) z[i] = __ldg(Mc + r + (l + i) * ld);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    H.add(z[i].x, key);
                    H.add(z[i].y, key);
                }
            }
            for (; l < l1; ++l) {
                const double2 z = __ldg(Mc + r + l * ld);
                H.add(z.x, key);
                H.add(z.y, key);
            }
        } else {
            for (; l + 8 <= l1; l += 8) {
                double x[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) x[i] = __ldg(M + r + (l + i) * ld);
#pragma unroll
                for (int i = 0; i < 8; ++i) H.add(x[i], key);
            }
            for (; l < l1; ++l) H.add(__ldg(M + r + l * ld), key);
        }
    }
    hist_flush(H, out);
}

// ---- accuracy-targeted AUTO (reading A18, Discussion P:713-734) -------------------------
// Per vector v with exponent E (rows of op(A) / columns of op(B)), over its nonzero finite
// elements x, in 32-bit fixed point relative to 2^E:
//     N_t(v) = sum ceil(frac(|x| 2^(wt-E)) 2^32)  (t = 1..s_max),  D(v) = sum floor(|x| 2^(32-E)),
// exact integers (< 2^53: k <= 2^21 terms of <= 2^32), so the sums are order-free;
// rho_v(t) = ((double)N_t / (double)D) 2^(-wt), and rho(t) = max over the vectors (the host
// then takes the smallest s with sum_{t=0..s} rho_A(t) rho_B(s-t) <= tau u sqrt(k)).
// With |x| = M 2^e0 (M the integer significand, e0 its exponent), |x| 2^(wt-E) = M 2^-z,
// z = E - e0 - wt fraction bits: the residual after t digits is the low z bits of M.
template <int W, int SM>  // t = 1..SM (compile time); only t <= s_max are kept
struct ResidAcc {
    // Fast path (every element within 43 bits of its vector's maximum, z0 <= 96 below): the
    // fraction |x| / 2^E is exactly the 96-bit fixed-point V = M 2^(96 - z0) (limbs L0..L2);
    // digit t leaves the bits below position 96 - wt, the 32 just below the cut are the field
    // at bit p = 64 - wt, and the rounding-up ("sticky") bit is "V has a set bit below p".
    // The fields are summed per t in n[t]; the sticky bits are counted once per element in a
    // per-thread shared-memory histogram over T = the number of cuts above V's lowest set bit
    // (the element contributes 1 to N_t for t = 1..T), folded into n[] by flush().
    static constexpr int TMAX = (63 / W) < SM ? (63 / W) : SM;  // cuts with p > 0
    unsigned long long n[SM + 1];  // [0] = D, [t] = N_t (sticky bits after flush())
    uint32_t *hist;                // this thread's column: hist[T * 256], T = 1..TMAX
    double sc;                     // 2^(64 - E): |x| sc is V's top 64 bits plus a fraction
    bool fp;                       // E >= -958: sc is a normal double, the FP route is exact
    int32_t E;
    __device__ __forceinline__ void zero(uint32_t *h, int32_t e) {
#pragma unroll
        for (int t = 0; t <= SM; ++t) n[t] = 0;
        hist = h;
#pragma unroll
        for (int t = 1; t <= TMAX; ++t) hist[t * 256] = 0;
        E = e;
        fp = e >= -958;
        sc = fp ? __longlong_as_double(static_cast<long long>(1023 + 64 - e) << 52) : 0.0;
    }
    __device__ __forceinline__ void flush() {
        uint32_t run = 0;
#pragma unroll
        for (int t = TMAX; t >= 1; --t) {
            run += hist[t * 256];
            n[t] += run;
        }
    }
    __device__ __forceinline__ void add(double x) {
        const uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
        const int be = static_cast<int>((u >> 52) & 0x7FF);
        const uint64_t fr = u & ((1ull << 52) - 1);
        const uint64_t M = be ? (fr | (1ull << 52)) : fr;
        if (M == 0) return;
        const int e0 = be ? be - 1075 : -1074;
        const int z0 = E - e0;  // |x| / 2^E = M 2^-z0
        if (z0 <= 96) {
            uint32_t L[3];
            uint64_t V64;
            if (fp) {
                // |x| 2^(64-E) < 2^64 exactly (power-of-two scaling); its integer part is V's
                // top 64 bits and its fraction (exact: <= 53 significant bits) times 2^32 the
                // low limb, an integer here because no bit of x lies below V's last bit
                const double y = __dmul_rn(fabs(x), sc);
                V64 = __double2ull_rz(y);
                const double r = __dadd_rn(y, -__ull2double_rn(V64));
                L[0] = __double2uint_rz(__dmul_rn(r, 4294967296.0));
            } else {
                const int v = 96 - z0;  // 0..95 (M < 2^53 and |x| < 2^E keep V < 2^96)
                const uint64_t lo = v < 64 ? (M << v) : 0ull;
                const uint64_t hi = v == 0 ? 0ull : (v < 64 ? (M >> (64 - v)) : (M << (v - 64)));
                L[0] = static_cast<uint32_t>(lo);
                V64 = (lo >> 32) | (hi << 32);
            }
            L[1] = static_cast<uint32_t>(V64);
            L[2] = static_cast<uint32_t>(V64 >> 32);
            n[0] += L[2];  // floor(|x| 2^(32-E))
            const int tz = L[0] ? __ffs(static_cast<int>(L[0])) - 1
                                : 31 + __ffsll(static_cast<long long>(V64));
            if (tz < 64 - W) {  // at least one cut above the lowest set bit
                int T = (63 - tz) / W;
                T = T < TMAX ? T : TMAX;
                hist[T * 256] += 1u;
            }
#pragma unroll
            for (int t = 1; t <= SM; ++t) {
                const int p = 64 - W * t;
                uint32_t f;
                if (p >= 0) {
                    const int li = p >> 5, bs = p & 31;
                    const uint32_t hiw = li + 1 < 3 ? L[li + 1] : 0u;
                    f = bs ? __funnelshift_r(L[li], hiw, bs) : L[li];
                } else if (p > -32) {
                    f = (L[0] & ((1u << (32 + p)) - 1u)) << (-p);
                } else {
                    f = 0;
                }
                n[t] += f;
            }
            return;
        }
        // general path (floor(|x| 2^(32-E)) = 0 here: z0 > 96): the residual after t digits is the low z bits of M, z = z0 - wt;
        // ceil of its top 32 bits (z > 32: a shift plus a sticky bit)
#pragma unroll
        for (int t = 1; t <= SM; ++t) {
            const int z = z0 - W * t;
            uint64_t f;
            if (z <= 0) {
                f = 0;
            } else {
                const uint64_t R = z >= 64 ? M : (M & ((1ull << z) - 1));
                if (z <= 32) {
                    f = R << (32 - z);
                } else {
                    const int d = z - 32;
                    const uint64_t hi2 = d >= 64 ? 0ull : (R >> d);
                    const uint64_t lo2 = d >= 64 ? R : (R & ((1ull << d) - 1));
                    f = hi2 + (lo2 != 0 ? 1ull : 0ull);
                }
            }
            n[t] += f;
        }
    }
};

// Contiguous vectors: persistent 256-thread blocks, one vector at a time (pass 1 exponent,
// pass 2 the sums, block-reduced and written to sums[r][0..s_max]).
template <int W, int SM>
__global__ void __launch_bounds__(256) k_resid_contig(const double *__restrict__ M, int64_t ld,
                                                      int64_t rows, int64_t kdim, int s_max,
                                                      unsigned long long *__restrict__ sums,
                                                      int32_t *__restrict__ keys_out) {
    __shared__ uint32_t hist_s[(ResidAcc<W, SM>::TMAX + 1) * 256];  // sticky histograms
    __shared__ int32_t kred[8];
    __shared__ unsigned long long red[8][SM + 1];
    const uint64_t keep = l2_pol(true), strm = l2_pol(false);
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const double *v = M + r * ld;
        int32_t key = kKeyEmpty;
        int64_t l = threadIdx.x;
        for (; l + 3 * 256 < kdim; l += 4 * 256) {
            double x[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = ldg_pol(v + l + i * 256, keep);
#pragma unroll
            for (int i = 0; i < 4; ++i) key = max(key, exp_key_a(x[i]));
        }
        for (; l < kdim; l += 256) key = max(key, exp_key_a(ldg_pol(v + l, keep)));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffff, key, o));
        if ((threadIdx.x & 31) == 0) kred[threadIdx.x >> 5] = key;
        __syncthreads();
        key = kred[0];
#pragma unroll
        for (int i = 1; i < 8; ++i) key = max(key, kred[i]);
        __syncthreads();  // kred is rewritten for the next vector
        if (threadIdx.x == 0) keys_out[r] = key;
        if (key == kExpNonFinite || key == kKeyEmpty) continue;  // skipped vector
        ResidAcc<W, SM> acc;
        acc.zero(hist_s + threadIdx.x, key);
        l = threadIdx.x;
        for (; l + 3 * 256 < kdim; l += 4 * 256) {
            double x[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = ldg_pol(v + l + i * 256, strm);
#pragma unroll
            for (int i = 0; i < 4; ++i) acc.add(x[i]);
        }
        for (; l < kdim; l += 256) acc.add(ldg_pol(v + l, strm));
        acc.flush();
#pragma unroll
        for (int t = 0; t <= SM; ++t) {
            unsigned long long x = acc.n[t];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffff, x, o);
            if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][t] = x;
        }
        __syncthreads();
        if (threadIdx.x <= (unsigned)s_max) {
            unsigned long long x = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) x += red[i][threadIdx.x];
            sums[r * (s_max + 1) + threadIdx.x] = x;
        }
        __syncthreads();
    }
}

// Strided vectors (element l of vector r at M[r + l ld]; complex: the (re, im) pair): one
// thread per vector and a slice of l per blockIdx.y, partial sums added to sums[r][.]
// (zeroed by the caller; integer atomics, so the totals do not depend on the order).
template <int W, int SM, int CPX>
__global__ void __launch_bounds__(256) k_resid_strided(const double *__restrict__ M, int64_t ld,
                                                       int64_t rows, int64_t kdim, int64_t lchunk,
                                                       const int32_t *__restrict__ keys,
                                                       int s_max,
                                                       unsigned long long *__restrict__ sums) {
    __shared__ uint32_t hist_s[(ResidAcc<W, SM>::TMAX + 1) * 256];  // sticky histograms
    const int64_t r = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
    const int32_t key = r < rows ? keys[r] : kKeyEmpty;
    if (key == kExpNonFinite || key == kKeyEmpty) return;
    ResidAcc<W, SM> acc;
    acc.zero(hist_s + threadIdx.x, key);
    const int64_t l0 = static_cast<int64_t>(blockIdx.y) * lchunk;
    const int64_t l1 = min(kdim, l0 + lchunk);
    if (CPX) {
        const double2 *Mc = reinterpret_cast<const double2 *>(M);
        for (int64_t l = l0; l < l1; ++l) {
            const double2 z = __ldg(Mc + r + l * ld);
            acc.add(z.x);
            acc.add(z.y);
        }
    } else {
        int64_t l = l0;
        for (; l + 4 <= l1; l += 4) {
            double x[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = __ldg(M + r + (l + i) * ld);
#pragma unroll
            for (int i = 0; i < 4; ++i) acc.add(x[i]);
        }
        for (; l < l1; ++l) acc.add(__ldg(M + r + l * ld));
    }
    acc.flush();
#pragma unroll
    for (int t = 0; t <= SM; ++t) {
        if (t > s_max) break;
        if (acc.n[t]) atomicAdd(&sums[r * (s_max + 1) + t], acc.n[t]);
    }
}

// rho_v(t) per vector from its sums, max over the vectors into rho_out[0..s_max] (as the bit
// patterns of non-negative doubles, whose unsigned order is their numeric order).
__global__ void k_resid_rho(const unsigned long long *__restrict__ sums, const int32_t *__restrict__ keys,
                            int64_t rows, int w, int s_max, unsigned long long *__restrict__ rho_out) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.y + threadIdx.y;
    const int t = threadIdx.x;
    if (r >= rows || t > s_max) return;
    const int32_t key = keys[r];
    if (key == kExpNonFinite || key == kKeyEmpty) return;
    double rho = 1.0;
    if (t > 0) {
        const double q = __ddiv_rn((double)sums[r * (s_max + 1) + t], (double)sums[r * (s_max + 1)]);
        rho = __dmul_rn(q, __longlong_as_double(static_cast<long long>(1023 - w * t) << 52));
    }
    if (rho > 0.0) atomicMax(&rho_out[t], static_cast<unsigned long long>(__double_as_longlong(rho)));
}

}  // namespace

// Accuracy-targeted AUTO statistics of the vectors of op(M): rho_out (device, s_max + 1 uint64
// holding doubles; max-accumulated, caller zeroes it).  scratch: device uint64
// [rows (s_max + 1)] + int32 [rows] keys.
namespace {
template <int W, int SM>
cudaError_t resid_sums(const double *M, int64_t ld, bool contiguous, int64_t rows, int64_t kdim,
                       int s_max, unsigned long long *sums, int32_t *keys, int num_sms,
                       cudaStream_t st, int *launches, int cpx) {
    if (contiguous) {
        int64_t blocks = 4 * (int64_t)num_sms;
        if (blocks > rows) blocks = rows;
        k_resid_contig<W, SM><<<(unsigned)blocks, 256, 0, st>>>(M, ld, rows, kdim, s_max, sums, keys);
        ++*launches;
        return cudaGetLastError();
    }
    cudaError_t e = cudaMemsetAsync(sums, 0, sizeof(unsigned long long) * rows * (s_max + 1), st);
    if (e != cudaSuccess) return e;
    e = launch_expscan(M, ld, rows, kdim, keys, num_sms, st, launches, cpx);
    if (e != cudaSuccess) return e;
    const int64_t rblocks = ceil_div(rows, 256);
    int64_t ysplit = ceil_div(4 * (int64_t)num_sms, rblocks);
    if (ysplit < 1) ysplit = 1;
    int64_t lchunk = ceil_div(kdim, ysplit);
    if (lchunk < 256) lchunk = 256;
    ysplit = ceil_div(kdim, lchunk);
    if (cpx)
        k_resid_strided<W, SM, 1><<<dim3((unsigned)rblocks, (unsigned)ysplit), 256, 0, st>>>(
            M, ld, rows, kdim, lchunk, keys, s_max, sums);
    else
        k_resid_strided<W, SM, 0><<<dim3((unsigned)rblocks, (unsigned)ysplit), 256, 0, st>>>(
            M, ld, rows, kdim, lchunk, keys, s_max, sums);
    ++*launches;
    return cudaGetLastError();
}

template <int W>
cudaError_t resid_sums_w(const double *M, int64_t ld, bool contiguous, int64_t rows, int64_t kdim,
                         int s_max, unsigned long long *sums, int32_t *keys, int num_sms,
                         cudaStream_t st, int *launches, int cpx) {
    // t = 1..12 covers every decision up to s = 12 (the usual case); larger s_max take the
    // full-width instance
    if (s_max <= 12)
        return resid_sums<W, 12>(M, ld, contiguous, rows, kdim, s_max, sums, keys, num_sms, st,
                                 launches, cpx);
    return resid_sums<W, kMaxS>(M, ld, contiguous, rows, kdim, s_max, sums, keys, num_sms, st,
                                launches, cpx);
}
}  // namespace

// Accuracy-targeted AUTO statistics of the vectors of op(M): rho_out (device, s_max + 1 uint64
// holding doubles; max-accumulated, caller zeroes it).  scratch: device uint64
// [rows (s_max + 1)] + int32 [rows] keys.
cudaError_t launch_trunc_residual(const double *M, int64_t ld, bool contiguous, int64_t rows,
                                  int64_t kdim, int w, int s_max, unsigned long long *rho_out,
                                  void *scratch, int num_sms, cudaStream_t st, int *launches,
                                  int cpx) {
    if (rows <= 0 || kdim <= 0) return cudaSuccess;
    if (s_max < 1 || s_max > kMaxS || w < 5 || w > 7) return cudaErrorInvalidValue;
    unsigned long long *sums = static_cast<unsigned long long *>(scratch);
    int32_t *keys = reinterpret_cast<int32_t *>(sums + rows * (s_max + 1));
    cudaError_t e;
    switch (w) {
    case 7: e = resid_sums_w<7>(M, ld, contiguous, rows, kdim, s_max, sums, keys, num_sms, st, launches, cpx); break;
    case 6: e = resid_sums_w<6>(M, ld, contiguous, rows, kdim, s_max, sums, keys, num_sms, st, launches, cpx); break;
    default: e = resid_sums_w<5>(M, ld, contiguous, rows, kdim, s_max, sums, keys, num_sms, st, launches, cpx); break;
    }
    if (e != cudaSuccess) return e;
    const int ty = 256 / 64;  // 64 threads (t = 0..s_max) x 4 vectors per block
    k_resid_rho<<<(unsigned)ceil_div(rows, ty), dim3(64, ty), 0, st>>>(sums, keys, rows, w, s_max,
                                                                       rho_out);
    ++*launches;
    return cudaGetLastError();
}

size_t trunc_residual_scratch(int64_t rows, int s_max) {
    return sizeof(unsigned long long) * (size_t)rows * (s_max + 1) + sizeof(int32_t) * (size_t)rows;
}

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
    if (s_max < 1 || s_max > kMaxS || w < 1 || w > 7) return cudaErrorInvalidValue;
    // per-thread bins hold int32 sums of y <= 2^12 over <= 2^18 elements per thread
    const size_t smem = hist_smem(s_max, 256, w);
    if (smem > 48 * 1024) {  // s_max > 23: opt in (per device, so on every call; cheap)
        cudaFuncSetAttribute(k_loss_contig, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_loss_strided<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_loss_strided<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    if (contiguous) {
        if (ceil_div(kdim, 256) > (1 << 18)) return cudaErrorInvalidValue;
        int64_t blocks = 4 * (int64_t)num_sms;
        if (blocks > rows) blocks = rows;
        k_loss_contig<<<(unsigned)blocks, 256, smem, st>>>(M, ld, rows, kdim, w, s_max, out);
        ++*launches;
        return cudaGetLastError();
    }
    cudaError_t e = launch_expscan(M, ld, rows, kdim, key_scratch, num_sms, st, launches, cpx);
    if (e != cudaSuccess) return e;
    const int64_t rblocks = ceil_div(rows, 256);
    int64_t ysplit = ceil_div(4 * (int64_t)num_sms, rblocks);
    if (ysplit < 1) ysplit = 1;
    int64_t lchunk = ceil_div(kdim, ysplit);
    if (lchunk < 64) lchunk = 64;
    if (lchunk > (1 << 17)) lchunk = 1 << 17;  // (re, im): 2 elements per step
    ysplit = ceil_div(kdim, lchunk);
    if (cpx)
        k_loss_strided<1><<<dim3((unsigned)rblocks, (unsigned)ysplit), 256, smem, st>>>(
            M, ld, rows, kdim, lchunk, key_scratch, w, s_max, out);
    else
        k_loss_strided<0><<<dim3((unsigned)rblocks, (unsigned)ysplit), 256, smem, st>>>(
            M, ld, rows, kdim, lchunk, key_scratch, w, s_max, out);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace ozimmu
