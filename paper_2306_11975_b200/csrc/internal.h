// internal.h -- host-side plan and kernel launchers shared by api.cu, split.cu, igemm.cu.
// Not part of the public ABI (see include/ozimmu.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ozimmu {

constexpr int32_t kExpNonFinite = 0x7fffffff;   // == OZIMMU_EXP_NONFINITE
constexpr int32_t kKeyEmpty = (int32_t)0x80808080;  // memset(0x80) pattern: "no nonzero seen"

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
inline int64_t ceil_div(int64_t x, int64_t a) { return (x + a - 1) / a; }

// launch_split's key_scratch: int32 keys[rows] + per-panel counters (<= rows) + a work counter
inline size_t split_scratch_bytes(int64_t rows) {
    return sizeof(int32_t) * (size_t)(2 * (rows > 0 ? rows : 1) + 2);
}

// A1 (Eq. alpha P:224-227 with l_acc = 31, BPS P:457-460 with l_in = 7):
// w = min(7, floor((31 - ceil(log2 k)) / 2)) -- the integer form of floor((31 - log2 k)/2).
inline int slice_width(int64_t k) {
    int c = 0;
    while (((int64_t)1 << c) < k) ++c;  // c = ceil(log2 k)
    int a = (31 - c) / 2;
    return a < 7 ? a : 7;
}

// ---- slicing (A2 + A3) -------------------------------------------------------------
// Vectors r = 0..rows-1 of length kdim; element l of vector r is
//   contiguous ? M[l + r*ld] : M[r + l*ld].
// Output planes: slice p (1..s) of vector r at planes + pidx*plane_stride + r*k_pad + l,
// pidx = reverse ? s - p : p - 1;  elements l in [kdim, k_pad) are written as 0.
// E[r]: frexp exponent of the vector's max |x| (0 for an all-zero vector,
// kExpNonFinite if any element is NaN/Inf -- its digits are then all 0).
// key_scratch: device scratch of split_scratch_bytes(rows) (exponent keys + the work
// counters of the one-read fused kernel); may be null only for contiguous vectors with
// k_pad < 2048 (then the fused kernel is not used).
// Complex operands (ZGEMM, reading A16): cpx = 1 -> vectors are complex rows of op(A)
// (kdim / k_pad count doubles: 2 per element, Im negated if conj); cpx = 2 -> vectors are
// complex columns of op(B), each emitting two plane rows 2r = (Re, -Im, ..) and
// 2r+1 = (Im, Re, ..).  For strided complex vectors `ld` is in complex elements; for
// contiguous ones it is in doubles.
// Batched operands stacked into one GEMM (strided-batched calls with a shared operand):
// vector r of the stacked operand is vector (r % per_item) of item r / per_item, whose
// data start at item_stride * (r / per_item) (same units as the vector's ld).
// per_item = 0: no batching.
struct BatchMap {
    int64_t per_item = 0;
    int64_t stride = 0;
};

cudaError_t launch_split(const double *M, int64_t ld, bool contiguous, int64_t rows, int64_t kdim,
                         int64_t k_pad, int s, int w, bool reverse, int8_t *planes,
                         int64_t plane_stride, int32_t *E, int32_t *key_scratch, int num_sms,
                         cudaStream_t st, int *launches, int cpx = 0, int conj = 0,
                         BatchMap vm = BatchMap());

// Small calls: both operands sliced in ONE launch (split.cu k_split_small; contiguous or
// strided vectors, real operands), which also zeroes the GEMM's wave counter (zero_ctr).
// split_small_ok: the call qualifies (both operands' input bytes <= OZIMMU_SPLIT_SMALL_MB,
// default 80 MB, and k_pad <= 1024).
struct SmallOp {
    const double *M;
    int64_t ld, rows, kdim, k_pad;
    int contig, reverse;
    int8_t *planes;
    int64_t plane_stride;
    int32_t *E;
    int64_t per_item, item_stride;
};
bool split_small_ok(int64_t m, int64_t n, int64_t k_pad);
cudaError_t launch_split_small(const SmallOp &a, const SmallOp &b, int s, int w,
                               unsigned int *zero_ctr, int num_sms, cudaStream_t st,
                               int *launches);

cudaError_t launch_expscan(const double *M, int64_t ld, int64_t rows, int64_t kel, int32_t *keys,
                           int num_sms, cudaStream_t st, int *launches, int cpx,
                           BatchMap vm = BatchMap());

// ---- INT8-AUTO mantissa-loss scan (f2) -------------------------------------------------
cudaError_t launch_mantissa_loss(const double *M, int64_t ld, bool contiguous, int64_t rows,
                                 int64_t kdim, int w, int s_max, unsigned long long *out,
                                 int32_t *key_scratch, int num_sms, cudaStream_t st,
                                 int *launches, int cpx = 0);

// ---- accuracy-targeted INT8-AUTO statistics (f2, reading A18) ----------------------------
// rho_out: device uint64 [s_max + 1] holding non-negative doubles, max-accumulated (zero it
// first); scratch: trunc_residual_scratch(rows, s_max) bytes of device memory.
cudaError_t launch_trunc_residual(const double *M, int64_t ld, bool contiguous, int64_t rows,
                                  int64_t kdim, int w, int s_max, unsigned long long *rho_out,
                                  void *scratch, int num_sms, cudaStream_t st, int *launches,
                                  int cpx = 0);
size_t trunc_residual_scratch(int64_t rows, int s_max);

// ---- fused GEMM (A4 + A5) ----------------------------------------------------------------
enum EpiMode : int { EPI_DGEMM = 0, EPI_LEVELS_I64 = 1, EPI_PAIR_I32 = 2, EPI_ZGEMM = 3 };

struct GemmArgs {
    const int8_t *a_planes;  // [s][m][k_pad], natural slice order
    const int8_t *b_planes;  // [s][n][k_pad], REVERSED slice order (index s - q)
    int64_t b_plane_rows;    // rows per B plane in memory (0 = n): column chunk of a larger buffer
    int64_t a_plane_rows;    // rows per A plane in memory (0 = m): row block of a larger buffer
    BatchMap c_rows, c_cols; // stacked batches: row r / column j of C -> item and its offset
                             // (stride in elements of C: doubles, or complex for EPI_ZGEMM)
    const int32_t *EA, *EB;  // exponents (EPI_DGEMM only)
    int64_t m, n, k_pad;
    int s, w;
    double alpha, beta;
    double alpha_im, beta_im;  // EPI_ZGEMM: complex alpha / beta
    double *C;               // EPI_DGEMM: column-major, ldc; EPI_ZGEMM: interleaved complex,
                             // ldc in complex elements, GEMM columns 2j / 2j+1 = Re / Im of C(:,j)
    int64_t ldc;
    void *out;               // EPI_LEVELS_I64: int64 [s][n][m];  EPI_PAIR_I32: int32 [n][m]
    int64_t *chunk_scratch;  // per-CTA partial level sums when k_chunks > 1
    unsigned int *wave_counter;  // 4-byte device scratch for the soft wave barrier (or null)
    bool counter_zeroed;         // wave_counter already zeroed on the stream (by k_split_small)
    long long *stats;            // optional per-CTA stall counters (development) or null
};

struct GemmPlan {
    int tile_n;       // N_c
    int k_block;      // K bytes per stage (= swizzle width)
    int stages;       // = a_stages (reported)
    int a_stages, b_stages;
    int64_t num_k_blocks;
    int64_t chunk_blocks;  // k-blocks per INT32-safe chunk
    int k_chunks;
    int G, T;          // INT32 sub-groups: T regions of <= G pairs per level
    int grid;
    size_t smem_bytes;
    int tmem_cols;
    int sk;            // stream-K schedule (small problems; see k_oz_gemm)
    int nacc;          // accumulator buffers in TMEM (2: short K, see KParams::nacc)
    int64_t tiles;     // stream-K arrival-counter slots (>= units x cluster size)
};

// Choose tile/pipeline parameters for (s, w, k_pad); returns false if unsupported.
bool plan_gemm(int s, int w, int64_t m, int64_t n, int64_t k_pad, int num_sms, GemmPlan *p);
size_t chunk_scratch_bytes(const GemmPlan &p, int s);
size_t chunk_scratch_bound(const GemmPlan &p, int s, int max_sms);
size_t sk_counters_bytes(int64_t tiles);
cudaError_t launch_gemm(const GemmArgs &a, const GemmPlan &p, EpiMode mode, cudaStream_t st,
                        int *launches);

}  // namespace ozimmu
