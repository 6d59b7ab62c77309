// split.cu -- A2 (exponent scan) + A3 (slicing) of the Ozaki scheme on sm_100a.
//
// SplitInt, Alg. 4: per row of op(A) / column of op(B) a shared
// power-of-two scale 2^E (E = frexp exponent of the max |x|, reading A3), then
// s signed INT8 digits d_p = sgn(x) * (floor(|x| 2^(w p - E)) mod 2^w) (readings
// A4/A5).  The paper's implementation "uses bit operations to cut the mantissa"
// (P:530); so do we: everything below is integer arithmetic on the IEEE-754 bit
// pattern, |x| = M * 2^e0 with M the (sub)normal significand.
//
// Digit extraction: per element the fixed-point fraction V = floor(|x| 2^(T - E)),
// T = 32 * ceil(W * S / 32), is built once as 32-bit limbs (a few 64-bit shifts of
// M); digit p is then bits [T - W p, T - W (p-1)) of V -- one funnel shift and a mask
// with compile-time amounts -- and the sign is applied as (d ^ m) - m.
//
// HBM-bound: read 8 B/element (the strided variant reads twice: exponent pass +
// transposing slice pass), write s B/element.  128-bit loads, 64-bit stores.
#include <cstdint>
#include <cstdlib>
#include <cooperative_groups.h>
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

// Start of vector r (units of ld): contiguous vectors r * ld, strided vectors r, or the
// stacked-batch mapping (BatchMap) of either.
__device__ __forceinline__ int64_t vec_off(int64_t r, int64_t ld, int64_t per_item,
                                           int64_t item_stride) {
    if (!per_item) return r * ld;
    const int64_t b = r / per_item;
    return b * item_stride + (r - b * per_item) * ld;
}

// floor(M * 2^sh) mod 2^32 for any integer sh (M < 2^53).
__device__ __forceinline__ uint32_t shifted_limb(uint64_t M, int sh) {
    uint64_t v;
    if (sh >= 0) v = sh >= 64 ? 0ull : (M << sh);
    else v = (-sh) >= 64 ? 0ull : (M >> (-sh));
    return static_cast<uint32_t>(v);
}

template <int W, int S>
struct Digits {
    static constexpr int NL = (W * S + 31) / 32;  // limbs of the fraction window
    static constexpr int T = 32 * NL;             // V = floor(|x| 2^(T - E))
    uint32_t L[NL + 1];
    uint32_t sm;  // 0 or 0xffffffff (sign of x)

    // x finite, |x| < 2^E (x == 0 gives zero limbs)
    __device__ __forceinline__ void init(double x, int32_t E) {
        const uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
        const int be = static_cast<int>((u >> 52) & 0x7FF);
        const uint64_t fr = u & ((1ull << 52) - 1);
        const uint64_t M = be ? (fr | (1ull << 52)) : fr;  // |x| = M 2^e0
        const int e0 = be ? be - 1075 : -1074;
        const int base = e0 - E + T;                         // V = floor(M 2^base)
#pragma unroll
        for (int j = 0; j < NL; ++j) L[j] = shifted_limb(M, base - 32 * j);
        L[NL] = 0;
        sm = (u >> 63) ? 0xffffffffu : 0u;
    }
    // signed digit p (1-based): bits [T - W p, T - W p + W) of V, with the sign of x
    template <int P>
    __device__ __forceinline__ uint32_t digit() const {
        constexpr int t = T - W * P;
        constexpr int li = t / 32, sh = t % 32;
        uint32_t d;
        if (sh + W <= 32) d = (L[li] >> sh) & ((1u << W) - 1);
        else d = __funnelshift_r(L[li], L[li + 1], sh) & ((1u << W) - 1);
        return (d ^ sm) - sm;
    }
};

// pack the low bytes of 4 words
__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    const uint32_t ab = __byte_perm(a, b, 0x0040);
    const uint32_t cd = __byte_perm(c, d, 0x0040);
    return __byte_perm(ab, cd, 0x5410);
}

// Write digit planes p = 1..s of 8 consecutive elements (one 8-byte store per plane).
template <int W, int S, int P = 1>
__device__ __forceinline__ void store_digits(const Digits<W, S> (&dg)[8], int s, int reverse,
                                             int8_t *dst, int64_t plane_stride) {
    if constexpr (P <= S) {
        if (P <= s) {
            uint2 v;
            v.x = pack4(dg[0].template digit<P>(), dg[1].template digit<P>(),
                        dg[2].template digit<P>(), dg[3].template digit<P>());
            v.y = pack4(dg[4].template digit<P>(), dg[5].template digit<P>(),
                        dg[6].template digit<P>(), dg[7].template digit<P>());
            const int pidx = reverse ? (s - P) : (P - 1);
            *reinterpret_cast<uint2 *>(dst + pidx * plane_stride) = v;
            store_digits<W, S, P + 1>(dg, s, reverse, dst, plane_stride);
        }
    }
}

// ---------------------------------------------------------------------------------
// Fast path for W * S <= 96 (s <= 13 at w = 7): the whole fraction window of an element is
// one 64-bit word V = floor(|x| 2^(64 - E)) (W S <= 64), or 96 bits (three limbs), and digit
// p is bits [T - W p, T - W (p-1)) of V (T = 64 or 96).  V is formed in floating point:
// |x| 2^(64-E) is an exact power-of-two scaling (|x| < 2^E, so it is < 2^64; where it would
// underflow the true value is < 1 and both floors are 0), then one truncating conversion to
// u64; the 96-bit window adds the exact fraction times 2^32, truncated, as its low limb.  The digits of 4 elements are produced 4 at a
// time: the 4W-bit field of digits 4g+1 .. 4g+4 is spread over 4 bytes with shifts and
// masks (two levels: 2W-bit halves, then W-bit quarters), and a 4 x 4 byte transpose
// (8 byte permutes) turns the 4 elements' words into 4 plane words holding one element per
// byte.  Signs are applied four bytes at a time on the plane words: for a byte d in
// [0, 127], -d = (0x80 - d) ^ 0x80 (no borrow leaves the byte), selected by a per-byte mask
// of the negative elements (the sign bits replicated by a byte permute).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ double pow2d(int e) {  // 2^e, e in the normal range
    return __longlong_as_double(static_cast<long long>(e + 1023) << 52);
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    return __byte_perm(a, b, sel);
}
// prmt.b32 with the sign-replicate bit of the selector nibbles honoured (__byte_perm masks
// the selector to 3 bits per nibble)
__device__ __forceinline__ uint32_t prmt_sx(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

template <int W, int S>
struct Chunk64 {
    static_assert(W * S <= 96, "fraction window must fit 96 bits");
    // limbs of the fraction window: V = floor(|x| 2^(32 NL - E)); W S <= 64 -> 64 bits (the
    // truncating conversion of |x| 2^(64-E)), else 96 bits (its integer part and the exact
    // fraction times 2^32, truncated: digits reach at most 91 bits below 2^E)
    static constexpr int NL = W * S <= 64 ? 2 : 3;
    static constexpr int NG = (S + 3) / 4;  // digit groups of 4
    uint32_t O[2][S];  // O[h][p-1]: magnitude of digit p of elements 4h .. 4h+3, one per byte
    uint32_t neg[2];   // 0xFF per byte of a negative element (elements 0-3, 4-7)

    // bytes q of the result = digit (4g + nd - q), q < nd (nd = digits in group g)
    template <int Gi>
    __device__ static __forceinline__ uint32_t spread(const uint32_t (&L)[NL]) {
        constexpr int nd = (S - 4 * Gi) < 4 ? (S - 4 * Gi) : 4;
        constexpr int o = 32 * NL - W * (4 * Gi + nd);  // bit offset of the group's field in V
        constexpr int li = o / 32, sh = o % 32;
        uint32_t y;
        if constexpr (li + 1 >= NL) y = L[li] >> sh;
        else if constexpr (sh == 0) y = L[li];
        else y = __funnelshift_r(L[li], L[li + 1], sh);
        constexpr uint32_t m = (1u << W) - 1;
        if constexpr (nd == 4) {
            constexpr uint32_t h2 = (1u << (2 * W)) - 1;
            const uint32_t t = (y & h2) | ((y << (16 - 2 * W)) & (h2 << 16));
            return (t & (m | (m << 16))) | ((t << (8 - W)) & ((m << 8) | (m << 24)));
        } else {
            uint32_t r = y & m;
            if constexpr (nd > 1) r |= (y << (8 - W)) & (m << 8);
            if constexpr (nd > 2) r |= (y << (16 - 2 * W)) & (m << 16);
            return r;
        }
    }

    template <int Gi>
    __device__ __forceinline__ void group(int h, const uint32_t (&L)[4][NL]) {
        if constexpr (Gi < NG) {
            constexpr int nd = (S - 4 * Gi) < 4 ? (S - 4 * Gi) : 4;
            const uint32_t a = spread<Gi>(L[0]), b = spread<Gi>(L[1]);
            const uint32_t c = spread<Gi>(L[2]), d = spread<Gi>(L[3]);
            // 4 x 4 byte transpose: o_q = byte q of (a, b, c, d) = digit 4 Gi + nd - q
            const uint32_t t0 = prmt(a, b, 0x5140), t2 = prmt(c, d, 0x5140);
            O[h][4 * Gi + nd - 1] = prmt(t0, t2, 0x5410);
            if constexpr (nd > 1) O[h][4 * Gi + nd - 2] = prmt(t0, t2, 0x7632);
            if constexpr (nd > 2) {
                const uint32_t t1 = prmt(a, b, 0x7362), t3 = prmt(c, d, 0x7362);
                O[h][4 * Gi + nd - 3] = prmt(t1, t3, 0x5410);
                if constexpr (nd > 3) O[h][4 * Gi] = prmt(t1, t3, 0x7632);
            }
            group<Gi + 1>(h, L);
        }
    }

    // x[] finite, |x| < 2^E (zeros give zero digits)
    __device__ __forceinline__ void init(const double (&x)[8], int32_t E) {
        // 2^(64-E) as one normal double if E >= -958, else as 2^1000 * 2^(64-E-1000)
        const bool small = E < -958;
        const double sc1 = small ? 0x1p1000 : pow2d(64 - E);
        const double sc2 = small ? pow2d(64 - E - 1000) : 1.0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint32_t L[4][NL], sg[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const double xe = x[4 * h + e];
                double y = __dmul_rn(fabs(xe), sc1);
                if (small) y = __dmul_rn(y, sc2);
                const unsigned long long V = __double2ull_rz(y);
                L[e][NL - 1] = static_cast<uint32_t>(V >> 32);
                L[e][NL - 2] = static_cast<uint32_t>(V);
                if constexpr (NL == 3) {
                    // floor(V 2^32 + frac(y) 2^32): V has <= 53 significant bits (exact as a
                    // double), so the fraction y - V and its scaling are exact
                    const double r = __dadd_rn(y, -__ull2double_rn(V));
                    L[e][0] = __double2uint_rz(__dmul_rn(r, 4294967296.0));
                }
                sg[e] = static_cast<uint32_t>(__double2hiint(xe));
            }
            // sign bit of each element replicated over its byte (prmt sign-extend selectors)
            neg[h] = prmt(prmt_sx(sg[0], sg[1], 0x00FB), prmt_sx(sg[2], sg[3], 0xFB00), 0x7610);
            group<0>(h, L);
        }
    }
    // magnitudes of digit P of elements e0 .. e0+3, one per byte
    template <int P>
    __device__ __forceinline__ uint32_t mags(int e0) const {
        return O[e0 >> 2][P - 1];
    }
    // swapped pairs (element 2j <-> 2j+1)
    template <int P>
    __device__ __forceinline__ uint32_t mags_swapped(int e0) const {
        return prmt(O[e0 >> 2][P - 1], 0u, 0x2301);
    }
};

__device__ __forceinline__ void st2_hint(int8_t *dst, uint2 v, uint64_t pol, bool use) {
    if (!use) {
        *reinterpret_cast<uint2 *>(dst) = v;
        return;
    }
    asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;"
                 ::"l"(dst), "r"(v.x), "r"(v.y), "l"(pol) : "memory");
}

__device__ __forceinline__ uint32_t apply_signs(uint32_t w, uint32_t m) {
    const uint32_t n = (0x80808080u - w) ^ 0x80808080u;
    return w ^ ((w ^ n) & m);
}

// digit planes p = 1..s of the 8 elements: one 8-byte store per plane; `m` = sign masks
template <int W, int S, bool SWAP, int P = 1>
__device__ __forceinline__ void store_planes64(const Chunk64<W, S> &c, uint32_t m0, uint32_t m1,
                                               int s, int reverse, int8_t *dst,
                                               int64_t plane_stride, uint64_t spol = 0,
                                               bool suse = false) {
    if constexpr (P <= S) {
        if (P <= s) {
            uint2 v;
            if constexpr (SWAP) {
                v.x = apply_signs(c.template mags_swapped<P>(0), m0);
                v.y = apply_signs(c.template mags_swapped<P>(4), m1);
            } else {
                v.x = apply_signs(c.template mags<P>(0), m0);
                v.y = apply_signs(c.template mags<P>(4), m1);
            }
            // dst = plane of slice P; the next slice's plane is plane_stride further (negative
            // stride for the reversed order, see store64_first)
            st2_hint(dst, v, spol, suse);
            store_planes64<W, S, SWAP, P + 1>(c, m0, m1, s, reverse, dst + plane_stride,
                                              plane_stride, spol, suse);
        }
    }
}

// emit() for Chunk64 (same three operand forms, same signs as below)
template <int W, int S, int CPX>
__device__ __forceinline__ void emit64(const Chunk64<W, S> &c, int s, int reverse, int conj,
                                       int8_t *planes, int64_t r, int64_t l0, int64_t k_pad,
                                       int64_t plane_stride, uint64_t spol = 0,
                                       bool suse = false) {
    constexpr uint32_t kOdd = 0xFF00FF00u, kEven = 0x00FF00FFu;
    // slice 1's plane, and the signed distance to the next slice's plane
    if (reverse) {
        planes += (int64_t)(s - 1) * plane_stride;
        plane_stride = -plane_stride;
    }
    if constexpr (CPX == 0) {
        store_planes64<W, S, false>(c, c.neg[0], c.neg[1], s, reverse, planes + r * k_pad + l0,
                                    plane_stride, spol, suse);
    } else if constexpr (CPX == 1) {
        const uint32_t f = conj ? kOdd : 0u;  // conj: Im negated
        store_planes64<W, S, false>(c, c.neg[0] ^ f, c.neg[1] ^ f, s, reverse,
                                    planes + r * k_pad + l0, plane_stride, spol, suse);
    } else {
        // row 2r = (Re, -Im) (Im := -Im if conj); row 2r+1 = (Im, Re) with the (re, im)
        // swap applied to the masks too
        const uint32_t f0 = conj ? 0u : kOdd;
        store_planes64<W, S, false>(c, c.neg[0] ^ f0, c.neg[1] ^ f0, s, reverse,
                                    planes + (2 * r) * k_pad + l0, plane_stride, spol, suse);
        auto swapb = [](uint32_t m) { return __byte_perm(m, 0, 0x2301); };
        const uint32_t f1 = conj ? kEven : 0u;
        store_planes64<W, S, true>(c, swapb(c.neg[0]) ^ f1, swapb(c.neg[1]) ^ f1, s, reverse,
                                   planes + (2 * r + 1) * k_pad + l0, plane_stride, spol, suse);
    }
}

// Output of one 8-element chunk (elements l0..l0+7 of input vector r) for the three
// operand forms (ZGEMM reading A16, real embedding with interleaved K):
//   CPX 0  real vector                    -> row r
//   CPX 1  complex row of op(A) (re, im)   -> row r, Im negated if conj
//   CPX 2  complex column of op(B)         -> row 2r   = (Re, -Im, ...)
//                                             row 2r+1 = (Im,  Re, ...)   (Im := -Im if conj)
// Sign changes and the (re, im) swap act on the digits (sign-magnitude: digits of -x are
// the negated digits of x), so each input element is digitised once.
template <int W, int S, int CPX>
__device__ __forceinline__ void emit(Digits<W, S> (&dg)[8], int s, int reverse, int conj,
                                     int8_t *planes, int64_t r, int64_t l0, int64_t k_pad,
                                     int64_t plane_stride) {
    if constexpr (CPX == 0) {
        store_digits<W, S>(dg, s, reverse, planes + r * k_pad + l0, plane_stride);
    } else if constexpr (CPX == 1) {
        if (conj) {
#pragma unroll
            for (int i = 1; i < 8; i += 2) dg[i].sm = ~dg[i].sm;
        }
        store_digits<W, S>(dg, s, reverse, planes + r * k_pad + l0, plane_stride);
    } else {
        Digits<W, S> sw[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            sw[i] = dg[i ^ 1];
            if (conj && (i & 1) == 0) sw[i].sm = ~sw[i].sm;  // Im of a conjugated element
        }
        if (!conj) {
#pragma unroll
            for (int i = 1; i < 8; i += 2) dg[i].sm = ~dg[i].sm;  // -Im
        }
        store_digits<W, S>(dg, s, reverse, planes + (2 * r) * k_pad + l0, plane_stride);
        store_digits<W, S>(sw, s, reverse, planes + (2 * r + 1) * k_pad + l0, plane_stride);
    }
}

// L2 eviction priorities (createpolicy + .L2::cache_hint): a first read that will be read again
// (exponent pass) is kept (evict_last), the second read and the plane stores -- touched once
// more only by a later kernel -- go first (evict_first), so a vector's second read finds it
// in L2.  OZIMMU_SPLIT_HINTS=0 turns the hints off (experiments).
enum : int { HINT_NONE = 0, HINT_KEEP = 1, HINT_STREAM = 2 };
__device__ __forceinline__ uint64_t l2_policy(int hint) {
    uint64_t p = 0;
    if (hint == HINT_KEEP)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else if (hint == HINT_STREAM)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double2 ldg2_hint(const double2 *q, uint64_t pol, bool use) {
    if (!use) return __ldg(q);
    double2 r;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(r.x), "=d"(r.y) : "l"(q), "l"(pol));
    return r;
}
__device__ __forceinline__ double ldg1_hint(const double *q, uint64_t pol, bool use) {
    if (!use) return __ldg(q);
    double r;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(q), "l"(pol));
    return r;
}

__device__ __forceinline__ void load8(const double *v, int64_t l0, int64_t kdim, bool al16,
                                      double (&x)[8], uint64_t pol = 0, bool use = false) {
    if (al16 && l0 + 8 <= kdim) {
        const double2 *q = reinterpret_cast<const double2 *>(v + l0);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            double2 d2 = ldg2_hint(q + i, pol, use);
            x[2 * i] = d2.x;
            x[2 * i + 1] = d2.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = (l0 + i < kdim) ? ldg1_hint(v + l0 + i, pol, use) : 0.0;
    }
}

// Exponent key from the running max of the high words |x|_hi (sign cleared): the exponent
// field of the largest |x| is the largest field, so a normal / non-finite maximum decides E
// from its field alone; only an all-subnormal (or zero) set needs the exact key of every
// element (then `exact` is evaluated).
template <typename F>
__device__ __forceinline__ int32_t key_from_hi(uint32_t mx, F exact) {
    if (mx >= 0x7FF00000u) return kExpNonFinite;
    if (mx >= 0x00100000u) return static_cast<int32_t>(mx >> 20) - 1022;
    return exact();
}
__device__ __forceinline__ uint32_t abs_hi(double x) {
    return static_cast<uint32_t>(__double2hiint(x)) & 0x7FFFFFFFu;
}

// Digits of elements l0 .. l0+7 of contiguous vector r (data at v), E = Ev.
template <int W, int S, int CPX>
__device__ __forceinline__ void contig_chunk(const double *v, int64_t l0, int64_t kdim, bool al16,
                                             int32_t Ev, int s, int reverse, int conj,
                                             int8_t *planes, int64_t r, int64_t k_pad,
                                             int64_t plane_stride, uint64_t lpol = 0,
                                             uint64_t spol = 0, bool use = false) {
    const bool bad = Ev == kExpNonFinite;
    double x[8];
    if (!bad) load8(v, l0, kdim, al16, x, lpol, use);
    if constexpr (W * S <= 96) {
        if (bad) {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = 0.0;
        }
        Chunk64<W, S> c;
        c.init(x, bad ? 0 : Ev);
        emit64<W, S, CPX>(c, s, reverse, conj, planes, r, l0, k_pad, plane_stride, spol, use);
    } else {
        Digits<W, S> dg[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) dg[i].init(bad ? 0.0 : x[i], bad ? 0 : Ev);
        emit<W, S, CPX>(dg, s, reverse, conj, planes, r, l0, k_pad, plane_stride);
    }
}

// ---------------------------------------------------------------------------------
// Contiguous vectors (row of op(A) with transA = T, column of op(B) with transB = N):
// TPR threads per vector, one pass for the exponent (max reduction), one pass for
// the digits (the second read of a <= 128 KB row hits L2).
// ---------------------------------------------------------------------------------
// One group of VPB = 256 / TPR contiguous vectors (rb-th group): pass 1 (exponent) and pass 2
// (digits).  Called by every thread of the block (block-uniform rb); red: 8 ints of shared memory.
template <int TPR, int W, int S, int CPX>
__device__ __forceinline__ void contig_group(const double *__restrict__ M, int64_t ld, int64_t rows,
                                             int64_t kdim, int64_t k_pad, int s, int reverse,
                                             int conj, int8_t *__restrict__ planes,
                                             int64_t plane_stride, int32_t *__restrict__ E,
                                             int64_t per_item, int64_t item_stride, int64_t rb,
                                             int32_t *red, uint64_t keep, uint64_t strm, bool use) {
    constexpr int VPB = 256 / TPR;  // vectors per block
    const int sub = threadIdx.x / TPR;
    const int t = threadIdx.x % TPR;
    const int64_t nchunk = k_pad / 8;
    const int64_t r = rb * VPB + sub;
    const bool active = r < rows;
    const double *v = M + vec_off(active ? r : 0, ld, per_item, item_stride);
    const bool al16 = ((reinterpret_cast<uintptr_t>(v) & 15) == 0);

    // ---- pass 1: E = max exponent key ----
    int32_t key = kKeyEmpty;
    if (active) {
        // four chunks' loads in flight per thread (memory parallelism with few blocks per
        // SM, which keeps the vectors in flight -- and so pass 2's re-reads -- in L2); the
        // max of the high words |x|_hi decides E unless everything is subnormal or zero
        uint32_t mx = 0;
        int64_t c = t;
        for (; c + 3 * TPR < nchunk; c += 4 * TPR) {
            double x[4][8];
#pragma unroll
            for (int u = 0; u < 4; ++u) load8(v, (c + u * TPR) * 8, kdim, al16, x[u], keep, use);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int i = 0; i < 8; ++i) mx = max(mx, abs_hi(x[u][i]));
        }
        for (; c < nchunk; c += TPR) {
            double x[8];
            load8(v, c * 8, kdim, al16, x, keep, use);
#pragma unroll
            for (int i = 0; i < 8; ++i) mx = max(mx, abs_hi(x[i]));
        }
        key = key_from_hi(mx, [&]() {  // this thread saw only subnormals / zeros: exact
            int32_t k2 = kKeyEmpty;
            for (int64_t c2 = t; c2 < nchunk; c2 += TPR) {
                double x[8];
                load8(v, c2 * 8, kdim, al16, x);
#pragma unroll
                for (int i = 0; i < 8; ++i) k2 = max(k2, exp_key(x[i]));
            }
            return k2;
        });
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffff, key, o));
    if (TPR > 32) {
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = key;
        __syncthreads();
        key = red[0];
#pragma unroll
        for (int i = 1; i < TPR / 32; ++i) key = max(key, red[i]);
        __syncthreads();  // red[] is rewritten by the next vector
    }
    if (!active) return;
    const int32_t Ev = key_to_exp(key);
    if (t == 0) {
        if (CPX == 2) {
            E[2 * r] = Ev;
            E[2 * r + 1] = Ev;
        } else {
            E[r] = Ev;
        }
    }

    // ---- pass 2: digits ----
    for (int64_t c = t; c < nchunk; c += TPR)
        contig_chunk<W, S, CPX>(v, c * 8, kdim, al16, Ev, s, reverse, conj, planes, r, k_pad,
                                plane_stride, strm, strm, use);
}

template <int TPR, int W, int S, int CPX>
__global__ void __launch_bounds__(256) k_split_contig(const double *__restrict__ M, int64_t ld,
                                                      int64_t rows, int64_t kdim, int64_t k_pad,
                                                      int s, int reverse, int conj,
                                                      int8_t *__restrict__ planes,
                                                      int64_t plane_stride, int32_t *__restrict__ E,
                                                      int64_t per_item, int64_t item_stride,
                                                      int hints) {
    constexpr int VPB = 256 / TPR;  // vectors per block
    // pass 1 keeps the vector in L2 for pass 2, which reads it for the last time; the planes
    // are streamed out (see l2_policy)
    const bool use = hints != 0;
    const uint64_t keep = use ? l2_policy(HINT_KEEP) : 0, strm = use ? l2_policy(HINT_STREAM) : 0;
    __shared__ int32_t red[256 / 32];
    // Persistent blocks (grid sized by the host to a few blocks per SM): the vectors in
    // flight (grid x VPB x 8 k bytes) stay well inside L2, so pass 2 re-reads a vector from
    // L2 instead of HBM.
    for (int64_t rb = blockIdx.x; rb * VPB < rows; rb += gridDim.x)
        contig_group<TPR, W, S, CPX>(M, ld, rows, kdim, k_pad, s, reverse, conj, planes,
                                     plane_stride, E, per_item, item_stride, rb, red, keep, strm,
                                     use);
}

// ---------------------------------------------------------------------------------
// Strided vectors (row of op(A) with transA = N, column of op(B) with transB = T):
// element l of vector r at M[r + l*ld]; consecutive vectors are consecutive in memory.
// ---------------------------------------------------------------------------------

// Pass 1: one thread per vector, a slice of l per blockIdx.y; atomicMax of the key.
template <int CPX>
__global__ void __launch_bounds__(256) k_expscan_strided(const double *__restrict__ M, int64_t ld,
                                                         int64_t rows, int64_t kdim, int64_t lchunk,
                                                         int32_t *__restrict__ keys,
                                                         int64_t per_item, int64_t item_stride) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
    if (r >= rows) return;
    const int64_t ro = vec_off(r, 1, per_item, item_stride);  // element 0 of vector r
    const int64_t l0 = static_cast<int64_t>(blockIdx.y) * lchunk;
    const int64_t l1 = min(kdim, l0 + lchunk);
    int32_t key = kKeyEmpty;
    int64_t l = l0;
    if constexpr (CPX != 0) {  // kdim counts complex elements here; (re, im) pairs: 16-byte loads
        const double2 *Mc = reinterpret_cast<const double2 *>(M);
        for (; l + 4 <= l1; l += 4) {
            double2 x[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = __ldg(Mc + ro + (l + i) * ld);
#pragma unroll
            for (int i = 0; i < 4; ++i) key = max(key, max(exp_key(x[i].x), exp_key(x[i].y)));
        }
        for (; l < l1; ++l) {
            const double2 x = __ldg(Mc + ro + l * ld);
            key = max(key, max(exp_key(x.x), exp_key(x.y)));
        }
        if (key != kKeyEmpty) atomicMax(keys + r, key);
    } else {
    for (; l + 8 <= l1; l += 8) {
        double x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(M + ro + (l + i) * ld);
#pragma unroll
        for (int i = 0; i < 8; ++i) key = max(key, exp_key(x[i]));
    }
    for (; l < l1; ++l) key = max(key, exp_key(__ldg(M + ro + l * ld)));
    if (key != kKeyEmpty) atomicMax(keys + r, key);
    }
}

// Pass 2: 32 vectors x 128 elements per block, transposed through shared memory so that
// both the global reads (32 consecutive vectors at one l) and the plane writes (16 lanes x
// 8 B = 128 contiguous bytes of one vector) are coalesced.  Shared-memory layout: element
// (r, l) -> pair q = l/2 stored at pair slot q ^ ((q >> 2) & 7) ^ (r & 7) of row r, which
// keeps both the column-wise writes and the 16-byte row reads (nearly) conflict-free.
__device__ __forceinline__ int tslot(int r, int l) {
    const int q = l >> 1;
    return 2 * (q ^ ((q >> 2) & 7) ^ (r & 7)) + (l & 1);
}

// One 32-vector x 128-element tile of strided vectors: load (coalesced, transposed through
// shared memory), then digits of 16 8-element chunks per row.  exps[rr] = E of vector r0+rr
// (set and published by the caller before the call's first barrier).
template <int CPX>
__device__ __forceinline__ void strided_tile_load(const double *__restrict__ M, int64_t ld,
                                                  int64_t rows, int64_t kdim, int64_t per_item,
                                                  int64_t item_stride, int64_t r0, int64_t l0,
                                                  double (*tile)[128], uint64_t pol = 0,
                                                  bool use = false) {
    const int tid = threadIdx.x;
    // coalesced load: warp reads 32 consecutive vectors at one l (thread: vector rr,
    // elements lg + 8 it); interior tiles take the unchecked path
    {
        const int rr = tid & 31, lg = tid >> 5;
        const int64_t r = r0 + rr;
        const bool rok = r < rows;
        const int64_t ro = vec_off(rok ? r : 0, 1, per_item, item_stride);
        double *trow = tile[rr];
        if (CPX) {
            // kdim counts doubles (2 per complex element); complex element (r, lc) is the
            // 16-byte pair at 2 (r + lc ld)
            const double2 *q = reinterpret_cast<const double2 *>(M) + ro + (l0 / 2 + lg) * ld;
            const int64_t step = 8 * ld;
            const bool full = rok && l0 + 128 <= kdim;
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const int lc = lg + 8 * it;  // 0..63
                double2 x = make_double2(0.0, 0.0);
                if (full || (rok && l0 + 2 * lc < kdim)) x = ldg2_hint(q, pol, use);
                q += step;
                trow[tslot(rr, 2 * lc)] = x.x;
                trow[tslot(rr, 2 * lc + 1)] = x.y;
            }
        } else {
            const double *q = M + ro + (l0 + lg) * ld;
            const int64_t step = 8 * ld;
            const bool full = rok && l0 + 128 <= kdim;
            double x[16];
#pragma unroll
            for (int it = 0; it < 16; ++it) {
                x[it] = (full || (rok && l0 + lg + 8 * it < kdim)) ? ldg1_hint(q, pol, use) : 0.0;
                q += step;
            }
#pragma unroll
            for (int it = 0; it < 16; ++it) trow[tslot(rr, lg + 8 * it)] = x[it];
        }
    }
}

// Digits of a loaded tile (after a barrier that publishes it and exps[]).
template <int W, int S, int CPX>
__device__ __forceinline__ void strided_tile_digits(int64_t rows, int64_t k_pad, int s,
                                                    int reverse, int conj,
                                                    int8_t *__restrict__ planes,
                                                    int64_t plane_stride, int64_t r0, int64_t l0,
                                                    const double (*tile)[128],
                                                    const int32_t *exps, uint64_t pol = 0,
                                                    bool use = false) {
    const int tid = threadIdx.x;
#pragma unroll 1
    for (int task = tid; task < 512; task += 256) {
        const int c8 = task & 15;  // 8-element chunk of the row
        const int rr = task >> 4;  // 0..31
        const int64_t r = r0 + rr;
        const int64_t lb = l0 + c8 * 8;
        if (r >= rows || lb >= k_pad) continue;
        const int32_t Ev = exps[rr];
        const bool bad = Ev == kExpNonFinite;
        double x[8];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const double2 d2 = *reinterpret_cast<const double2 *>(&tile[rr][tslot(rr, c8 * 8 + 2 * h)]);
            x[2 * h] = d2.x;
            x[2 * h + 1] = d2.y;
        }
        if constexpr (W * S <= 96) {
            if (bad) {
#pragma unroll
                for (int i = 0; i < 8; ++i) x[i] = 0.0;
            }
            Chunk64<W, S> c;
            c.init(x, bad ? 0 : Ev);
            emit64<W, S, CPX>(c, s, reverse, conj, planes, r, lb, k_pad, plane_stride, pol, use);
        } else {
            Digits<W, S> dg[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) dg[i].init(bad ? 0.0 : x[i], bad ? 0 : Ev);
            emit<W, S, CPX>(dg, s, reverse, conj, planes, r, lb, k_pad, plane_stride);
        }
    }
}

template <int W, int S, int CPX>
__device__ __forceinline__ void strided_tile(const double *__restrict__ M, int64_t ld,
                                             int64_t rows, int64_t kdim, int64_t k_pad, int s,
                                             int reverse, int conj, int8_t *__restrict__ planes,
                                             int64_t plane_stride, int64_t per_item,
                                             int64_t item_stride, int64_t r0, int64_t l0,
                                             double (*tile)[128], const int32_t *exps,
                                             uint64_t pol = 0, bool use = false) {
    strided_tile_load<CPX>(M, ld, rows, kdim, per_item, item_stride, r0, l0, tile, pol, use);
    __syncthreads();
    strided_tile_digits<W, S, CPX>(rows, k_pad, s, reverse, conj, planes, plane_stride, r0, l0,
                                   tile, exps, pol, use);
}

template <int W, int S, int CPX>
__global__ void __launch_bounds__(256) k_split_strided(const double *__restrict__ M, int64_t ld,
                                                       int64_t rows, int64_t kdim, int64_t k_pad,
                                                       int s, int reverse, int conj,
                                                       const int32_t *__restrict__ keys,
                                                       int8_t *__restrict__ planes,
                                                       int64_t plane_stride,
                                                       int32_t *__restrict__ E,
                                                       int64_t per_item, int64_t item_stride) {
    __shared__ __align__(16) double tile[32][128];  // [r][swizzled l]
    __shared__ int32_t exps[32];
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int64_t l0 = static_cast<int64_t>(blockIdx.y) * 128;
    const int tid = threadIdx.x;
    if (tid < 32) {
        const int64_t r = r0 + tid;
        int32_t e = 0;
        if (r < rows) {
            e = key_to_exp(keys[r]);
            if (blockIdx.y == 0) {
                if (CPX == 2) {
                    E[2 * r] = e;
                    E[2 * r + 1] = e;
                } else {
                    E[r] = e;
                }
            }
        }
        exps[tid] = e;
    }
    strided_tile<W, S, CPX>(M, ld, rows, kdim, k_pad, s, reverse, conj, planes, plane_stride,
                            per_item, item_stride, r0, l0, tile, exps);
}

// ---------------------------------------------------------------------------------
// Small strided operands (k_pad <= 2048): ONE launch and one read instead of the exponent-key
// memset, the scan and the slice kernel (three dependent launches, which at 1024^2-2048^2
// cost more than the data movement).  A cluster of CL <= 8 CTAs owns 32 vectors; CTA c loads
// its T <= 2 tiles of 32 vectors x 128 elements (columns [c T 128, (c+1) T 128)) into shared
// memory, computes the partial exponent key of each vector from shared memory, the CL
// partials are combined through distributed shared memory, and each CTA converts its own tiles
// (strided_tile_digits: the same digit code as k_split_strided).
// ---------------------------------------------------------------------------------
// One cluster's 32 vectors (group g) of a strided operand; c = this CTA's rank of CL; T tiles
// of shared memory at `tiles`.  Called by every thread of every CTA of the cluster.
template <int W, int S>
__device__ __forceinline__ void strided_cluster_group(
    const double *__restrict__ M, int64_t ld, int64_t rows, int64_t kdim, int64_t k_pad, int s,
    int reverse, int8_t *__restrict__ planes, int64_t plane_stride, int32_t *__restrict__ E,
    int64_t per_item, int64_t item_stride, int T, int64_t g, int c, int CL,
    double (*tiles)[128], int32_t (*red)[32], int32_t *pkey, int32_t *exps) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int64_t r0 = g * 32;
    const int64_t lb0 = (int64_t)c * T * 128;
    const int tid = threadIdx.x;
    for (int t = 0; t < T; ++t)
        strided_tile_load<0>(M, ld, rows, kdim, per_item, item_stride, r0, lb0 + t * 128,
                             tiles + 32 * t);
    __syncthreads();
    {  // partial key of vector rr over this CTA's columns: thread (rr, g) takes 16 of each tile
        const int rr = tid & 31, gg = tid >> 5;
        uint32_t mx = 0;
        int32_t ek = kKeyEmpty;
        for (int t = 0; t < T; ++t) {
            const double *trow = tiles[32 * t + rr];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const double x = trow[tslot(rr, gg * 16 + j)];
                mx = max(mx, abs_hi(x));
                ek = max(ek, exp_key(x));
            }
        }
        red[gg][rr] = key_from_hi(mx, [&]() { return ek; });
    }
    __syncthreads();
    if (tid < 32) {
        int32_t k = red[0][tid];
#pragma unroll
        for (int i = 1; i < 8; ++i) k = max(k, red[i][tid]);
        pkey[tid] = k;
    }
    cl.sync();  // every CTA's partial keys written
    if (tid < 32) {
        int32_t k = kKeyEmpty;
        for (int q = 0; q < CL; ++q) k = max(k, *cl.map_shared_rank(&pkey[tid], q));
        const int64_t r = r0 + tid;
        const int32_t e = r < rows ? key_to_exp(k) : 0;
        if (c == 0 && r < rows) E[r] = e;
        exps[tid] = e;
    }
    cl.sync();  // peers' partial keys read (none is overwritten or exits early); exps published
    for (int t = 0; t < T; ++t)
        strided_tile_digits<W, S, 0>(rows, k_pad, s, reverse, 0, planes, plane_stride, r0,
                                     lb0 + t * 128, tiles + 32 * t, exps);
}

template <int W, int S>
__global__ void __launch_bounds__(256) k_split_strided_cl(
    const double *__restrict__ M, int64_t ld, int64_t rows, int64_t kdim, int64_t k_pad, int s,
    int reverse, int8_t *__restrict__ planes, int64_t plane_stride, int32_t *__restrict__ E,
    int64_t per_item, int64_t item_stride, int T) {
    extern __shared__ __align__(16) double dsm[];  // T tiles [32][128] (swizzled, tslot)
    __shared__ int32_t red[8][32];
    __shared__ int32_t pkey[32];
    __shared__ int32_t exps[32];
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int CL = (int)cl.num_blocks();
    strided_cluster_group<W, S>(M, ld, rows, kdim, k_pad, s, reverse, planes, plane_stride, E,
                                per_item, item_stride, T, blockIdx.x / CL, (int)cl.block_rank(),
                                CL, reinterpret_cast<double(*)[128]>(dsm), red, pkey, exps);
}

template <int W, int S>
cudaError_t launch_strided_cl(const double *M, int64_t ld, int64_t rows, int64_t kdim,
                              int64_t k_pad, int s, bool reverse, int8_t *planes,
                              int64_t plane_stride, int32_t *E, cudaStream_t st, int *launches,
                              BatchMap vm) {
    const int64_t nt = ceil_div(k_pad, 128);  // 128-element tiles per vector
    const int CL = (int)(nt < 8 ? nt : 8);
    const int T = (int)ceil_div(nt, CL);
    const size_t smem = (size_t)T * 32 * 128 * sizeof(double);
    auto kern = k_split_strided_cl<W, S>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(ceil_div(rows, 32) * CL));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ++*launches;
    return cudaLaunchKernelEx(&cfg, kern, M, ld, rows, kdim, k_pad, s, (int)reverse, planes,
                              plane_stride, E, vm.per_item, vm.stride, T);
}

// ---------------------------------------------------------------------------------
// One read of the operand from HBM (large operands): exponent scan and digits in ONE
// persistent launch.  The vectors are grouped in panels of ~16 MB of input; the work items
// are, in this order, the scan tiles of panel 0, then for q = 1 .. NP-1 the scan tiles of
// panel q followed by the slice tiles of panel q-1, then the slice tiles of panel NP-1.
// A scan tile max-reduces the exponent keys of its elements into keys[r] (atomicMax) and
// counts itself in done[p]; a slice tile of panel p first waits until done[p] holds all of
// p's scan tiles.  Between the scan and the slice of an element the GPU reads ~1-2 panels,
// so the second read of the element hits L2 and HBM sees 8 B read + s B written per
// element (the two-launch path reads every element twice from HBM at these sizes).
// Items are claimed in order from an atomic counter, so every claimed item is held by a
// resident CTA and the scan tiles a slice tile waits for were claimed before it: the waits
// cannot deadlock whatever else runs on the GPU (e.g. the other operand's slicing on a
// second stream).  scratch: int32 keys[rows] | done[NP] | claim, all set to 0x80808080
// by the launcher (= kKeyEmpty for the keys; counters count up from that base).
// Tiles: strided vectors 32 x 512 (scan) and 32 x 128 (slice, as k_split_strided);
// contiguous vectors 1 x 4096 for both.
// ---------------------------------------------------------------------------------
constexpr uint32_t kCtrBase = 0x80808080u;
#ifndef OZ_FUSED_MINB
#define OZ_FUSED_MINB 4  // resident blocks per SM the register allocation targets
#endif

struct FusedGeo {
    int64_t PR;        // vectors per panel (a multiple of 32 for strided vectors)
    int64_t NP;        // panels
    int64_t nls, nlb;  // scan / slice l-blocks per vector
    int64_t TS, TL;    // scan / slice tiles per panel
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(uint32_t *p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// item -> (slice?, panel, tile)
__device__ __forceinline__ void fused_item(int64_t i, const FusedGeo &g, bool &slice,
                                           int64_t &p, int64_t &t) {
    if (i < g.TS) { slice = false; p = 0; t = i; return; }
    const int64_t j = i - g.TS, B = g.TS + g.TL;
    if (j < B * (g.NP - 1)) {
        const int64_t q = j / B, r = j - q * B;
        if (r < g.TS) { slice = false; p = q + 1; t = r; }
        else { slice = true; p = q; t = r - g.TS; }
        return;
    }
    slice = true;
    p = g.NP - 1;
    t = j - B * (g.NP - 1);
}

template <int W, int S, int CPX, bool CONTIG>
__global__ void __launch_bounds__(256, (W * S <= 96) ? OZ_FUSED_MINB : 1) k_split_fused(const double *__restrict__ M, int64_t ld,
                                                     int64_t rows, int64_t kdim, int64_t k_pad,
                                                     int s, int reverse, int conj,
                                                     int8_t *__restrict__ planes,
                                                     int64_t plane_stride,
                                                     int32_t *__restrict__ E,
                                                     int32_t *__restrict__ scratch, FusedGeo g,
                                                     int64_t per_item, int64_t item_stride,
                                                     int hints) {
    __shared__ __align__(16) double tile[CONTIG ? 1 : 32][128];
    __shared__ int32_t red[8][32];
    __shared__ int32_t exps[32];
    __shared__ uint32_t next_item[2];
    int32_t *keys = scratch;
    uint32_t *done = reinterpret_cast<uint32_t *>(scratch + rows);
    uint32_t *claim = done + g.NP;
    const int64_t total = (g.TS + g.TL) * g.NP;
    const int tid = threadIdx.x;
    // scan reads are kept in L2 for the slice tiles' second (last) read; planes streamed out
    const bool use = hints != 0;
    const uint64_t keep = use ? l2_policy(HINT_KEEP) : 0, strm = use ? l2_policy(HINT_STREAM) : 0;
    if (tid == 0) next_item[0] = atomicAdd(claim, 1u) - kCtrBase;
    __syncthreads();
    int64_t item = next_item[0];
    for (int iter = 0; item < total; ++iter) {
        uint32_t nx = 0;
        if (tid == 0) nx = atomicAdd(claim, 1u);  // next claim in flight while this tile runs
        bool slice;
        int64_t p, t;
        fused_item(item, g, slice, p, t);
        if (slice) {
            if (tid == 0) {
                while (ld_acquire_u32(done + p) - kCtrBase < (uint32_t)g.TS) __nanosleep(64);
            }
            __syncthreads();
        }
        if constexpr (CONTIG) {
            // tile: 1 vector x 4096 doubles, chunks c0 = 512 lb + tid and c0 + 256 (8 each)
            const int64_t vi = t / (slice ? g.nlb : g.nls);
            const int64_t lb = t - vi * (slice ? g.nlb : g.nls);
            const int64_t r = p * g.PR + vi;
            const int64_t c0 = lb * 512 + tid, c1 = c0 + 256;
            const bool act0 = r < rows && c0 * 8 < k_pad, act1 = r < rows && c1 * 8 < k_pad;
            const double *v = M + vec_off(r < rows ? r : 0, ld, per_item, item_stride);
            const bool al16 = ((reinterpret_cast<uintptr_t>(v) & 15) == 0);
            if (!slice) {
                double x0[8], x1[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) x0[i] = x1[i] = 0.0;
                if (act0) load8(v, c0 * 8, kdim, al16, x0, keep, use);
                if (act1) load8(v, c1 * 8, kdim, al16, x1, keep, use);
                uint32_t mx = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) mx = max(mx, max(abs_hi(x0[i]), abs_hi(x1[i])));
                int32_t key = key_from_hi(mx, [&]() {
                    int32_t k2 = kKeyEmpty;
#pragma unroll
                    for (int i = 0; i < 8; ++i) k2 = max(k2, max(exp_key(x0[i]), exp_key(x1[i])));
                    return k2;
                });
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffff, key, o));
                if ((tid & 31) == 0) red[0][tid >> 5] = key;
                __syncthreads();
                if (tid == 0) {
#pragma unroll
                    for (int i = 1; i < 8; ++i) key = max(key, red[0][i]);
                    if (r < rows && key != kKeyEmpty) atomicMax(keys + r, key);
                    red_release_add(done + p, 1u);
                }
            } else if (r < rows) {
                const int32_t Ev = key_to_exp(__ldcg(keys + r));
                if (tid == 0 && lb == 0) {
                    if (CPX == 2) {
                        E[2 * r] = Ev;
                        E[2 * r + 1] = Ev;
                    } else {
                        E[r] = Ev;
                    }
                }
                if (act0)
                    contig_chunk<W, S, CPX>(v, c0 * 8, kdim, al16, Ev, s, reverse, conj, planes, r,
                                            k_pad, plane_stride, strm, strm, use);
                if (act1)
                    contig_chunk<W, S, CPX>(v, c1 * 8, kdim, al16, Ev, s, reverse, conj, planes, r,
                                            k_pad, plane_stride, strm, strm, use);
            }
        } else if (!slice) {
            // scan tile: 32 vectors x 512 doubles; thread (rr, lane group lg) reads elements
            // l = l0 + lg + 8 it of vector r0 + rr (a warp reads 32 consecutive vectors)
            const int64_t rg = t / g.nls;
            const int64_t r0 = p * g.PR + rg * 32;
            const int64_t l0 = (t - rg * g.nls) * 512;
            const int rr = tid & 31, lg = tid >> 5;
            const int64_t r = r0 + rr;
            uint32_t mx = 0;
            int32_t key = kKeyEmpty;
            if (r < rows) {
                const int64_t ro = vec_off(r, 1, per_item, item_stride);
                if (CPX) {  // kdim counts doubles; complex element lc at Mc[ro + lc ld]
                    const double2 *q = reinterpret_cast<const double2 *>(M) + ro + (l0 / 2 + lg) * ld;
                    const int64_t kc = kdim / 2 - (l0 / 2 + lg);  // complex elements left
                    const int64_t step = 8 * ld;
                    const bool full = kc > 8 * 31;
#pragma unroll 1
                    for (int b = 0; b < 4; ++b) {
                        double2 x[8];
#pragma unroll
                        for (int it = 0; it < 8; ++it) {
                            x[it] = (full || 8 * (8 * b + it) < kc) ? ldg2_hint(q, keep, use)
                                                                    : make_double2(0.0, 0.0);
                            q += step;
                        }
#pragma unroll
                        for (int it = 0; it < 8; ++it) mx = max(mx, max(abs_hi(x[it].x), abs_hi(x[it].y)));
                        if (mx < 0x00100000u) {
#pragma unroll
                            for (int it = 0; it < 8; ++it)
                                key = max(key, max(exp_key(x[it].x), exp_key(x[it].y)));
                        }
                    }
                } else {
                    const double *q = M + ro + (l0 + lg) * ld;
                    const int64_t kl = kdim - (l0 + lg);  // elements left from this thread's first
                    const int64_t step = 8 * ld;
                    const bool full = kl > 8 * 63;
#pragma unroll 1
                    for (int b = 0; b < 4; ++b) {
                        double x[16];
#pragma unroll
                        for (int it = 0; it < 16; ++it) {
                            x[it] = (full || 8 * (16 * b + it) < kl) ? ldg1_hint(q, keep, use) : 0.0;
                            q += step;
                        }
#pragma unroll
                        for (int it = 0; it < 16; ++it) mx = max(mx, abs_hi(x[it]));
                        if (mx < 0x00100000u) {  // only subnormals / zeros so far: exact keys
#pragma unroll
                            for (int it = 0; it < 16; ++it) key = max(key, exp_key(x[it]));
                        }
                    }
                }
                // a normal / non-finite maximum decides the key; else `key` holds the exact
                // maximum over the (all subnormal or zero) elements
                key = key_from_hi(mx, [&]() { return key; });
            }
            red[lg][rr] = key;
            __syncthreads();
            if (tid < 32) {
#pragma unroll
                for (int i = 1; i < 8; ++i) key = max(key, red[i][tid]);
                if (r < rows && key != kKeyEmpty) atomicMax(keys + r, key);
            }
            __syncthreads();
            if (tid == 0) red_release_add(done + p, 1u);
        } else {
            const int64_t rg = t / g.nlb;
            const int64_t r0 = p * g.PR + rg * 32;
            const int64_t l0 = (t - rg * g.nlb) * 128;
            if (tid < 32) {
                const int64_t r = r0 + tid;
                int32_t e = 0;
                if (r < rows) {
                    e = key_to_exp(__ldcg(keys + r));
                    if (l0 == 0) {
                        if (CPX == 2) {
                            E[2 * r] = e;
                            E[2 * r + 1] = e;
                        } else {
                            E[r] = e;
                        }
                    }
                }
                exps[tid] = e;
            }
            strided_tile<W, S, CPX>(M, ld, rows, kdim, k_pad, s, reverse, conj, planes,
                                    plane_stride, per_item, item_stride, r0, l0, tile, exps, strm,
                                    use);
        }
        if (tid == 0) next_item[(iter + 1) & 1] = nx - kCtrBase;
        __syncthreads();
        item = next_item[(iter + 1) & 1];
    }
}

// ---------------------------------------------------------------------------------
// Small calls: op(A) AND op(B) sliced in ONE launch, with no memset and no second stream (the
// default path costs the exponent-key memset, the scan and the slice of a strided operand, the
// other operand on a second stream, an event fork / join and the wave-counter memset -- at
// 1024^3 more latency than data movement).  Block ranges: op(A)'s blocks, then op(B)'s, each
// a whole number of clusters of CL CTAs; a strided operand's cluster owns 32 vectors
// (strided_cluster_group), a contiguous operand's block owns 1 or 8 vectors (contig_group).
// Block 0 zeroes the GEMM's wave counter, and the kernel lets the GEMM (launched with
// programmatic stream serialisation) start its set-up as soon as every block has started.
// ---------------------------------------------------------------------------------
__host__ __device__ __forceinline__ int64_t small_blocks(const SmallOp &o, int CL) {
    if (o.rows <= 0) return 0;
    const int64_t b = o.contig ? (o.k_pad >= 2048 ? o.rows : (o.rows + 7) / 8)
                               : ((o.rows + 31) / 32) * CL;
    return (b + CL - 1) / CL * CL;
}

template <int W, int S>
__global__ void __launch_bounds__(256) k_split_small(const __grid_constant__ SmallOp a,
                                                     const __grid_constant__ SmallOp b, int s,
                                                     int T, unsigned int *zero_ctr) {
    extern __shared__ __align__(16) double dsm[];  // T tiles [32][128] (strided operands)
    __shared__ int32_t red[8][32];
    __shared__ int32_t pkey[32];
    __shared__ int32_t exps[32];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (zero_ctr && blockIdx.x == 0 && threadIdx.x == 0) *zero_ctr = 0u;
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int CL = (int)cl.num_blocks();
    const int64_t na = small_blocks(a, CL);
    const bool ia = (int64_t)blockIdx.x < na;
    const SmallOp &o = *(ia ? &a : &b);  // stays in the parameter space (__grid_constant__)
    const int64_t bi = ia ? blockIdx.x : blockIdx.x - na;
    if (o.contig) {  // cluster-uniform: an operand spans whole clusters
        if (o.k_pad >= 2048) {
            if (bi < o.rows)
                contig_group<256, W, S, 0>(o.M, o.ld, o.rows, o.kdim, o.k_pad, s, o.reverse, 0,
                                           o.planes, o.plane_stride, o.E, o.per_item,
                                           o.item_stride, bi, &red[0][0], 0, 0, false);
        } else if (bi * 8 < o.rows) {
            contig_group<32, W, S, 0>(o.M, o.ld, o.rows, o.kdim, o.k_pad, s, o.reverse, 0,
                                      o.planes, o.plane_stride, o.E, o.per_item, o.item_stride,
                                      bi, &red[0][0], 0, 0, false);
        }
        return;
    }
    strided_cluster_group<W, S>(o.M, o.ld, o.rows, o.kdim, o.k_pad, s, o.reverse, o.planes,
                                o.plane_stride, o.E, o.per_item, o.item_stride, T, bi / CL,
                                (int)cl.block_rank(), CL, reinterpret_cast<double(*)[128]>(dsm),
                                red, pkey, exps);
}

template <int W, int S>
cudaError_t launch_small_t(const SmallOp &a, const SmallOp &b, int s, unsigned int *zero_ctr,
                           int num_sms, cudaStream_t st) {
    (void)num_sms;
    const int64_t nt = ceil_div(a.k_pad, 128);  // 128-element tiles per vector (same k)
    const bool strided = !a.contig || !b.contig;
    // one 32 x 128 tile per CTA: clusters of up to 16 CTAs (16 = the non-portable maximum, for
    // 1024 < k_pad <= 2048), so every block of the launch reserves 32 KB of shared memory
    static const int max_cl =
        getenv("OZIMMU_SPLIT_SMALL_CL") ? atoi(getenv("OZIMMU_SPLIT_SMALL_CL")) : 16;
    const int CL = strided ? (int)(nt < max_cl ? nt : max_cl) : 1;
    const int T = strided ? (int)ceil_div(nt, CL) : 0;
    const size_t smem = (size_t)T * 32 * 128 * sizeof(double);
    auto kern = k_split_small<W, S>;
    if (CL > 8) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(small_blocks(a, CL) + small_blocks(b, CL)));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a, b, s, T, zero_ctr);
}

template <int W>
cudaError_t launch_small_w(const SmallOp &a, const SmallOp &b, int s, unsigned int *zero_ctr,
                           int num_sms, cudaStream_t st) {
    if (s <= 9) return launch_small_t<W, 9>(a, b, s, zero_ctr, num_sms, st);
    if (s <= 13) return launch_small_t<W, 13>(a, b, s, zero_ctr, num_sms, st);
    if (s <= 16) return launch_small_t<W, 16>(a, b, s, zero_ctr, num_sms, st);
    return launch_small_t<W, 32>(a, b, s, zero_ctr, num_sms, st);
}

}  // namespace

// Exponent keys of strided vectors (element l of vector r at M[r + l ld]; cpx: (re, im)
// pairs at 2 (r + l ld), kel counts complex elements): keys[r] = max exp_key over the vector.
cudaError_t launch_expscan(const double *M, int64_t ld, int64_t rows, int64_t kel, int32_t *keys,
                           int num_sms, cudaStream_t st, int *launches, int cpx, BatchMap vm) {
    cudaError_t e = cudaMemsetAsync(keys, 0x80, sizeof(int32_t) * rows, st);
    if (e != cudaSuccess) return e;
    const int64_t rblocks = ceil_div(rows, 256);
    int64_t ysplit = ceil_div(4 * (int64_t)num_sms, rblocks);
    ysplit = ysplit < 1 ? 1 : ysplit;
    int64_t lchunk = round_up(ceil_div(kel, ysplit), 8);
    // >= 64 elements per thread when that still gives >= 4 blocks per SM (fewer atomics);
    // small operands take shorter chunks so that every SM has work
    if (lchunk < 64 && rblocks * ceil_div(kel, 64) >= 4 * (int64_t)num_sms) lchunk = 64;
    ysplit = ceil_div(kel, lchunk);
    if (ysplit < 1) ysplit = 1;
    if (cpx)
        k_expscan_strided<1><<<dim3((unsigned)rblocks, (unsigned)ysplit), 256, 0, st>>>(
            M, ld, rows, kel, lchunk, keys, vm.per_item, vm.stride);
    else
        k_expscan_strided<0><<<dim3((unsigned)rblocks, (unsigned)ysplit), 256, 0, st>>>(
            M, ld, rows, kel, lchunk, keys, vm.per_item, vm.stride);
    ++*launches;
    return cudaGetLastError();
}

namespace {

int split_hints() {
    static const int h = getenv("OZIMMU_SPLIT_HINTS") ? atoi(getenv("OZIMMU_SPLIT_HINTS")) : 1;
    return h;
}

template <int W, int S, int CPX, bool CONTIG>
cudaError_t launch_fused(const double *M, int64_t ld, int64_t rows, int64_t kdim, int64_t k_pad,
                         int s, bool reverse, int conj, int8_t *planes, int64_t plane_stride,
                         int32_t *E, int32_t *scratch, int num_sms, cudaStream_t st,
                         int *launches, BatchMap vm) {
    // panel size (KB of input), OZIMMU_SPLIT_PANEL_KB (tests use small panels)
    static const int64_t panel_bytes =
        (int64_t)(getenv("OZIMMU_SPLIT_PANEL_KB") ? atoi(getenv("OZIMMU_SPLIT_PANEL_KB")) : 16384)
        << 10;
    const int64_t vec_bytes = k_pad * 8;
    int64_t PRt = panel_bytes / vec_bytes;
    PRt = PRt < 1 ? 1 : PRt;
    FusedGeo g;
    if (CONTIG) {
        g.PR = PRt < rows ? PRt : rows;
        g.nls = g.nlb = ceil_div(k_pad, 4096);
        g.NP = ceil_div(rows, g.PR);
        g.TS = g.TL = g.PR * g.nlb;
    } else {
        int64_t PR = PRt / 32 * 32;
        PR = PR < 32 ? 32 : PR;
        const int64_t rr = round_up(rows, 32);
        g.PR = PR < rr ? PR : rr;
        g.nls = ceil_div(k_pad, 512);
        g.nlb = ceil_div(k_pad, 128);
        g.NP = ceil_div(rows, g.PR);
        g.TS = g.PR / 32 * g.nls;
        g.TL = g.PR / 32 * g.nlb;
    }
    cudaError_t e =
        cudaMemsetAsync(scratch, 0x80, sizeof(int32_t) * (size_t)(rows + g.NP + 1), st);
    if (e != cudaSuccess) return e;
    auto kern = k_split_fused<W, S, CPX, CONTIG>;
    static int bpsm = 0;  // resident blocks per SM (the grid is persistent)
    if (bpsm == 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpsm, kern, 256, 0) != cudaSuccess ||
            bpsm < 1) {
            cudaGetLastError();
            bpsm = 4;
        }
    }
    const int64_t total = (g.TS + g.TL) * g.NP;
    static const int bps_env =
        getenv("OZIMMU_SPLIT_FUSED_BPS") ? atoi(getenv("OZIMMU_SPLIT_FUSED_BPS")) : 0;
    int64_t grid = (int64_t)num_sms * (bps_env > 0 && bps_env < bpsm ? bps_env : bpsm);
    grid = grid < total ? grid : total;
    kern<<<(unsigned)grid, 256, 0, st>>>(M, ld, rows, kdim, k_pad, s, reverse ? 1 : 0, conj,
                                         planes, plane_stride, E, scratch, g, vm.per_item,
                                         vm.stride, split_hints());
    ++*launches;
    return cudaGetLastError();
}

template <int W, int S, int CPX>
cudaError_t launch_split_t(const double *M, int64_t ld, bool contiguous, int64_t rows,
                           int64_t kdim, int64_t k_pad, int s, bool reverse, int conj,
                           int8_t *planes, int64_t plane_stride, int32_t *E, int32_t *key_scratch,
                           int num_sms, cudaStream_t st, int *launches, BatchMap vm) {
    // kdim / k_pad count doubles of the (embedded) vector: 2 per complex element
    // one-read fused path (k_split_fused) only with OZIMMU_SPLIT_FUSED=1: measured slower than
    // the two-pass kernels below; it needs contiguous vectors of >= 2048 doubles
    static const int fused_env =
        getenv("OZIMMU_SPLIT_FUSED") ? atoi(getenv("OZIMMU_SPLIT_FUSED")) : 0;
    const bool fused = fused_env && key_scratch && (!contiguous || k_pad >= 2048);
    if (contiguous && fused)
        return launch_fused<W, S, CPX, true>(M, ld, rows, kdim, k_pad, s, reverse, conj, planes,
                                             plane_stride, E, key_scratch, num_sms, st, launches,
                                             vm);
    if (contiguous) {
        // persistent grid of `bps` blocks per SM (OZIMMU_SPLIT_BPS, default 16 = as many as
        // fit).  Capping the vectors in flight to keep pass 2 in L2 did not pay (16384^2, s = 9:
        // 2/4/8/16 blocks per SM -> 3.53/3.31/3.24/3.21 ms for both operands): the digit
        // extraction is issue-bound (ncu: 62% issue slots busy at 73% of DRAM bandwidth)
        static const int bps = getenv("OZIMMU_SPLIT_BPS") ? atoi(getenv("OZIMMU_SPLIT_BPS")) : 16;
        const int64_t cap = (int64_t)num_sms * (bps > 0 ? bps : 16);
        if (k_pad >= 2048) {
            const int64_t g = rows < cap ? rows : cap;
            k_split_contig<256, W, S, CPX><<<(unsigned)g, 256, 0, st>>>(
                M, ld, rows, kdim, k_pad, s, reverse, conj, planes, plane_stride, E, vm.per_item,
                vm.stride, split_hints());
        } else {
            const int64_t nb = ceil_div(rows, 8);
            const int64_t g = nb < 8 * cap ? nb : 8 * cap;
            k_split_contig<32, W, S, CPX><<<(unsigned)g, 256, 0, st>>>(
                M, ld, rows, kdim, k_pad, s, reverse, conj, planes, plane_stride, E, vm.per_item,
                vm.stride, split_hints());
        }
        ++*launches;
        return cudaGetLastError();
    }
    // strided: exponent scan then transposing slice
    if (fused) return launch_fused<W, S, CPX, false>(M, ld, rows, kdim, k_pad, s, reverse, conj,
                                                      planes, plane_stride, E, key_scratch,
                                                      num_sms, st, launches, vm);
    // small real operands (k_pad <= 1024, <= OZIMMU_SPLIT_CL_MB of input, default 64): one
    // clustered launch (k_split_strided_cl) instead of memset + scan + slice (1024^2: 18.5 ->
    // 10 us of kernel time, cold; at k_pad = 2048 two tiles per CTA made it slower: 29.7 ->
    // 32.8 us)
    if constexpr (CPX == 0) {
        static const int64_t cl_mb =
            getenv("OZIMMU_SPLIT_CL_MB") ? atoi(getenv("OZIMMU_SPLIT_CL_MB")) : 64;
        if (k_pad <= 1024 && rows * kdim * 8 <= (cl_mb << 20))
            return launch_strided_cl<W, S>(M, ld, rows, kdim, k_pad, s, reverse, planes,
                                           plane_stride, E, st, launches, vm);
    }
    cudaError_t e = launch_expscan(M, ld, rows, CPX ? kdim / 2 : kdim, key_scratch, num_sms, st,
                                   launches, CPX ? 1 : 0, vm);
    if (e != cudaSuccess) return e;
    k_split_strided<W, S, CPX><<<dim3((unsigned)ceil_div(rows, 32), (unsigned)ceil_div(k_pad, 128)),
                                 256, 0, st>>>(M, ld, rows, kdim, k_pad, s, reverse, conj,
                                               key_scratch, planes, plane_stride, E,
                                               vm.per_item, vm.stride);
    ++*launches;
    return cudaGetLastError();
}

template <int W, int CPX>
cudaError_t launch_split_w(const double *M, int64_t ld, bool contiguous, int64_t rows,
                           int64_t kdim, int64_t k_pad, int s, bool reverse, int conj,
                           int8_t *planes, int64_t plane_stride, int32_t *E, int32_t *key_scratch,
                           int num_sms, cudaStream_t st, int *launches, BatchMap vm) {
    if (s <= 9)
        return launch_split_t<W, 9, CPX>(M, ld, contiguous, rows, kdim, k_pad, s, reverse, conj,
                                         planes, plane_stride, E, key_scratch, num_sms, st,
                                         launches, vm);
    if (s <= 13)  // 96-bit fraction window (W s <= 91): the fast digit path
        return launch_split_t<W, 13, CPX>(M, ld, contiguous, rows, kdim, k_pad, s, reverse, conj,
                                          planes, plane_stride, E, key_scratch, num_sms, st,
                                          launches, vm);
    if (s <= 16)
        return launch_split_t<W, 16, CPX>(M, ld, contiguous, rows, kdim, k_pad, s, reverse, conj,
                                          planes, plane_stride, E, key_scratch, num_sms, st,
                                          launches, vm);
    return launch_split_t<W, 32, CPX>(M, ld, contiguous, rows, kdim, k_pad, s, reverse, conj,
                                      planes, plane_stride, E, key_scratch, num_sms, st,
                                      launches, vm);
}

template <int CPX>
cudaError_t launch_split_c(const double *M, int64_t ld, bool contiguous, int64_t rows,
                           int64_t kdim, int64_t k_pad, int s, int w, bool reverse, int conj,
                           int8_t *planes, int64_t plane_stride, int32_t *E, int32_t *key_scratch,
                           int num_sms, cudaStream_t st, int *launches, BatchMap vm) {
    switch (w) {
    case 7: return launch_split_w<7, CPX>(M, ld, contiguous, rows, kdim, k_pad, s, reverse, conj,
                                          planes, plane_stride, E, key_scratch, num_sms, st,
                                          launches, vm);
    case 6: return launch_split_w<6, CPX>(M, ld, contiguous, rows, kdim, k_pad, s, reverse, conj,
                                          planes, plane_stride, E, key_scratch, num_sms, st,
                                          launches, vm);
    case 5: return launch_split_w<5, CPX>(M, ld, contiguous, rows, kdim, k_pad, s, reverse, conj,
                                          planes, plane_stride, E, key_scratch, num_sms, st,
                                          launches, vm);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace

cudaError_t launch_split(const double *M, int64_t ld, bool contiguous, int64_t rows, int64_t kdim,
                         int64_t k_pad, int s, int w, bool reverse, int8_t *planes,
                         int64_t plane_stride, int32_t *E, int32_t *key_scratch, int num_sms,
                         cudaStream_t st, int *launches, int cpx, int conj, BatchMap vm) {
    if (rows <= 0) return cudaSuccess;
    if (s < 1 || s > 32) return cudaErrorInvalidValue;
    switch (cpx) {
    case 0: return launch_split_c<0>(M, ld, contiguous, rows, kdim, k_pad, s, w, reverse, 0,
                                     planes, plane_stride, E, key_scratch, num_sms, st, launches, vm);
    case 1: return launch_split_c<1>(M, ld, contiguous, rows, kdim, k_pad, s, w, reverse, conj,
                                     planes, plane_stride, E, key_scratch, num_sms, st, launches, vm);
    case 2: return launch_split_c<2>(M, ld, contiguous, rows, kdim, k_pad, s, w, reverse, conj,
                                     planes, plane_stride, E, key_scratch, num_sms, st, launches, vm);
    default: return cudaErrorInvalidValue;
    }
}

// Both operands of a small call in one launch (see k_split_small): real operands whose input
// bytes sum to at most OZIMMU_SPLIT_SMALL_MB (default 80; 0 disables) and k_pad <= 1024 (one
// 32 x 128 tile per CTA of a strided operand's cluster).  Measured: 1024^3
// call 80.4 -> 77.1 us; with k_pad = 1536-2048 (two tiles, 64 KB of shared memory for every
// block of the launch) slower than the per-operand kernels (2048^3 313 -> 320 us), and so with
// one tile per CTA in clusters of up to 16 (2048^3 310 -> 325 us; OZIMMU_SPLIT_SMALL_K raises
// the k_pad limit for experiments).
bool split_small_ok(int64_t m, int64_t n, int64_t k_pad) {
    static const int64_t lim =
        (int64_t)(getenv("OZIMMU_SPLIT_SMALL_MB") ? atoi(getenv("OZIMMU_SPLIT_SMALL_MB")) : 80)
        << 20;
    static const int64_t kmax =
        getenv("OZIMMU_SPLIT_SMALL_K") ? atoi(getenv("OZIMMU_SPLIT_SMALL_K")) : 1024;
    return m > 0 && n > 0 && k_pad <= kmax && (m + n) * k_pad * 8 <= lim;
}

cudaError_t launch_split_small(const SmallOp &a, const SmallOp &b, int s, int w,
                               unsigned int *zero_ctr, int num_sms, cudaStream_t st,
                               int *launches) {
    if (s < 1 || s > 32) return cudaErrorInvalidValue;
    cudaError_t e;
    switch (w) {
    case 7: e = launch_small_w<7>(a, b, s, zero_ctr, num_sms, st); break;
    case 6: e = launch_small_w<6>(a, b, s, zero_ctr, num_sms, st); break;
    case 5: e = launch_small_w<5>(a, b, s, zero_ctr, num_sms, st); break;
    default: return cudaErrorInvalidValue;
    }
    ++*launches;
    return e;
}

}  // namespace ozimmu
