/*
 * ozimmu.h -- C ABI of the B200-native Ozaki-scheme DGEMM on INT8 tensor cores.
 *
 * Method: Ootomo, Ozaki, Yokota, "DGEMM on Integer Matrix Multiplication Unit",
 * arXiv 2306.11975.  Citations "P:<line>" refer to that paper's text
 * (PAPER.md), with section / algorithm / equation.
 *
 *   C = alpha * op(A) * op(B) + beta * C          (BLAS DGEMM semantics)
 *
 * computed as
 *   A1  w = min(7, floor((31 - log2 k)/2))                     Eq. alpha, BPS P:457-460
 *   A2  E_A[i] = frexp exponent of max_l |op(A)(i,l)|,  E_B[j] likewise per column of op(B)
 *                                                              Alg. 4 line 2, P:394 (reading A3)
 *   A3  digits d_p = sgn(x) * (floor(|x| 2^(wp - E)) mod 2^w), p = 1..s,  INT8
 *                                                              Alg. 4 lines 3-5, P:396-401 (A4, A5)
 *   A4  P_pq = A^(p) * B^(q)  (INT8 x INT8 -> INT32, exact) for p + q <= s + 1
 *                                                              Alg. 3 line 6
 *   A5  L_g = sum_{p+q=g} P_pq (exact);  acc = +0;  for g = s+1 down to 2: acc += L_g 2^(-wg);
 *       X = ldexp(acc, E_A[i] + E_B[j]);  C = alpha X (+ beta C)  Alg. 3 line 7, P:382 (A6-A8)
 * on sm_100a: A2/A3 by a slicing kernel, A4+A5 by one persistent tcgen05 kernel
 * (TMA -> SMEM, tcgen05.mma.kind::i8 into TMEM, fused FP64 epilogue).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Column-major matrices (cuBLAS convention).  Element (i, j) of a matrix X
 *    with leading dimension ldX is X[i + j*ldX].  For row-major (e.g. torch)
 *    tensors call with swapped operands: C^T = B^T A^T; the result is bitwise
 *    the same because the exponent assignment is symmetric.
 *  - A, B, C and the workspace are DEVICE pointers owned by the caller.
 *    alpha and beta are HOST pointers.  Nothing is freed by the library except
 *    the internal workspace it allocated itself.
 *  - Every computing call is asynchronous on the handle's stream (default: the
 *    legacy default stream); it never synchronises the device.  Argument errors
 *    are detected synchronously and returned before anything is launched;
 *    launch failures are returned as OZIMMU_ERR_CUDA (asynchronous execution
 *    errors surface at the caller's next synchronisation).
 *  - Quick returns (BLAS): m == 0 or n == 0 -> no-op; alpha == 0 or k == 0 ->
 *    C = beta*C without reading A or B; beta == 0 -> C is not read (NaN in C is
 *    ignored).
 *  - num_slices = s in [1, OZIMMU_MAX_SLICES], or 0 = INT8-AUTO: s is chosen
 *    per call from the inputs (ozimmu_set_auto); an AUTO call synchronises its stream once
 *    to read the mantissa-loss statistics (the paper's "check all the elements" pass).
 *  - k is limited to OZIMMU_MAX_K (w >= 5); larger k returns OZIMMU_ERR_UNSUPPORTED.
 *  - Non-finite inputs (reading A9): if row i of op(A) or column j of op(B)
 *    contains NaN/Inf, C(i,j) = NaN (for alpha != 0).  No error is returned.
 *  - Results are deterministic and independent of the launch configuration,
 *    the stream, the device and the row/column partitioning.
 */
#ifndef OZIMMU_H
#define OZIMMU_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define OZIMMU_API __attribute__((visibility("default")))
#else
#define OZIMMU_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define OZIMMU_MAX_SLICES 32
#define OZIMMU_MAX_K (1LL << 21)

typedef struct ozimmu_ctx *ozimmu_handle_t;

typedef enum { OZIMMU_OP_N = 0, OZIMMU_OP_T = 1, OZIMMU_OP_C = 2 } ozimmu_op_t;

typedef enum {
    OZIMMU_SUCCESS = 0,
    OZIMMU_ERR_INVALID_VALUE = 1, /* bad argument (negative size, ld too small, NULL, bad s) */
    OZIMMU_ERR_UNSUPPORTED = 2,   /* valid BLAS call outside what is implemented (s = 0, k too large) */
    OZIMMU_ERR_WORKSPACE = 3,     /* caller workspace too small / allocation failed */
    OZIMMU_ERR_CUDA = 4,          /* a CUDA runtime/driver call or launch failed */
    OZIMMU_ERR_NOT_INITIALIZED = 5, /* NULL handle */
    OZIMMU_ERR_NCCL = 6           /* NCCL could not be loaded, or an NCCL call / the caller's
                                     broadcast function failed (multi-GPU entry points) */
} ozimmu_status_t;

/* Per-call report of the last computing call on a handle (SPEC GemmReport, S:378-381;
 * the paper's time-breakdown phases). */
typedef struct {
    int num_slices;        /* s */
    int slice_width;       /* w (bits per slice, BPS) */
    int64_t gemm_pairs;    /* s(s+1)/2 INT8 GEMMs */
    int64_t int8_macs;     /* s(s+1)/2 * m * n * k */
    int64_t slice_bytes;   /* INT8 planes + exponents written by the slicing kernels */
    int tile_n;            /* output columns per CTA tile (TMEM-bounded) */
    int k_block;           /* K bytes per pipeline stage */
    int stages;            /* SMEM pipeline depth */
    int k_chunks;          /* INT32-overflow-safe K chunks per tile (A4 budget) */
    int launches;          /* kernels launched by the last call */
    int acc_regions;       /* TMEM accumulator regions per level (INT32 sub-groups of pairs) */
    int auto_mode;         /* 0: s given by the caller; OZIMMU_AUTO_LOSS / OZIMMU_AUTO_ACCURACY:
                              s chosen by INT8-AUTO with that rule */
    int auto_capped;       /* 1 if INT8-AUTO reached s_max without meeting its criterion (the
                              result is then less accurate than the rule asked for) */
} ozimmu_report_t;

/* ---- handle ------------------------------------------------------------- */

/* Create a handle bound to CUDA device `device`.  Errors: INVALID_VALUE (h NULL),
 * CUDA (no such device / device is not sm_100). */
OZIMMU_API ozimmu_status_t ozimmu_create(ozimmu_handle_t *h, int device);
/* Free the internal workspace (if any) and the handle.  NULL is a no-op. */
OZIMMU_API ozimmu_status_t ozimmu_destroy(ozimmu_handle_t h);
/* Set the stream (a cudaStream_t passed as void*); NULL = legacy default stream. */
OZIMMU_API ozimmu_status_t ozimmu_set_stream(ozimmu_handle_t h, void *stream);
/* Cap the SMs the fused GEMM kernel occupies (its persistent grid; 0 = all SMs of the device).
 * The GEMM holds one CTA of ~227 KB shared memory per SM, so a collective kernel enqueued
 * beside it (the multi-GPU driver's NCCL broadcast of the next B chunk) can only
 * run concurrently on SMs left free.  Results are bitwise independent of the cap.
 * Errors: NOT_INITIALIZED, INVALID_VALUE (max_sms < 0). */
OZIMMU_API ozimmu_status_t ozimmu_set_max_sms(ozimmu_handle_t h, int max_sms);
/* Bytes of device workspace ozimmu_dgemm needs for this shape (0 on invalid input).
 * = s*(m + n)*round_up(k,16) INT8 planes + 4(m+n) exponents + K-chunk scratch + alignment
 * (the paper's working-memory cost). */
OZIMMU_API size_t ozimmu_workspace_bytes(ozimmu_op_t transA, ozimmu_op_t transB, int64_t m, int64_t n,
                              int64_t k, int num_slices);
/* Give the handle a caller-owned device workspace (256-byte aligned).  Calls whose
 * need exceeds `bytes` return OZIMMU_ERR_WORKSPACE.  dptr = NULL reverts to the
 * internal, lazily grown cudaMalloc workspace. */
OZIMMU_API ozimmu_status_t ozimmu_set_workspace(ozimmu_handle_t h, void *dptr, size_t bytes);
/* Copy the report of the last computing call. */
OZIMMU_API ozimmu_status_t ozimmu_get_report(ozimmu_handle_t h, ozimmu_report_t *out);
/* Per-phase device time of one computing call, from CUDA events the library records on
 * the handle's stream around each of its kernels (the paper's time breakdown). */
typedef struct {
    float slice_b_ms; /* call start -> op(B) sliced (A2+A3 on op(B); ~0 for presliced calls) */
    float slice_a_ms; /* call start -> op(A) sliced.  ozimmu_dgemm slices op(B) on a second
                         stream concurrently with op(A), so the slicing phase takes
                         max(slice_a_ms, slice_b_ms); ozimmu_zgemm slices B then A */
    float gemm_ms;    /* A4+A5: the fused tcgen05 GEMM + epilogue kernel */
} ozimmu_timing_t;
/* Start recording phase events for the next `max_calls` computing calls (0 disables and
 * frees the events).  Recording adds event records only -- no synchronisation. */
OZIMMU_API ozimmu_status_t ozimmu_timing_enable(ozimmu_handle_t h, int max_calls);
/* Wait for the recorded events, copy up to max_out per-call timings to out, return the
 * number of recorded calls (< 0 on error), and restart recording from an empty ring. */
OZIMMU_API int ozimmu_timing_read(ozimmu_handle_t h, ozimmu_timing_t *out, int max_out);
/* Library version (major*10000 + minor*100 + patch). */
OZIMMU_API int ozimmu_version(void);
/* Human-readable status name (static string). */
OZIMMU_API const char *ozimmu_status_string(ozimmu_status_t s);

/* ---- the method ------------------------------------------------------------ */

/* C = alpha op(A) op(B) + beta C with s = num_slices INT8 slices (Alg. 3).
 * op(A) is m x k, op(B) is k x n, C is m x n.  lda >= max(1, rows of stored A),
 * ldb likewise, ldc >= max(1, m).  OZIMMU_OP_C equals OZIMMU_OP_T for real data. */
OZIMMU_API ozimmu_status_t ozimmu_dgemm(ozimmu_handle_t h, ozimmu_op_t transA, ozimmu_op_t transB,
                             int64_t m, int64_t n, int64_t k, const double *alpha,
                             const double *A, int64_t lda, const double *B, int64_t ldb,
                             const double *beta, double *C, int64_t ldc, int num_slices);

/* As ozimmu_dgemm with A, B and C in HOST memory (the call a host program makes; BJ
 * metric "including the matrix splitting" end to end).  Pinned (cudaHostAlloc /
 * cudaHostRegister) buffers overlap the PCIe copies with the computation; pageable buffers
 * work but serialise.  op(A) is processed in row blocks and op(B) in column chunks: the H2D
 * copies, the slicing of each chunk, the GEMM of each block and the D2H copy of each C
 * block run on three streams (the handle's stream + two internal copy streams), so tensor
 * work starts after the first chunk arrives.  C is bitwise identical to ozimmu_dgemm on the
 * same data.  num_slices = 0 (INT8-AUTO): op(A) row blocks and op(B) column chunks go H2D
 * while the AUTO statistics of each landed block are computed; s is chosen once both operands
 * are in, then C row blocks return while the next block's GEMM runs.  Device memory: an
 * internal buffer (grown on demand, freed by ozimmu_destroy) of about s(n + 2 m/8) k_pad + 8 k (2 n/8 + 2 m/8) + 16 (m/8) n bytes.  The call BLOCKS
 * until C is in host memory.  Errors: as ozimmu_dgemm; WORKSPACE if the buffer cannot be
 * allocated. */
OZIMMU_API ozimmu_status_t ozimmu_dgemm_host(ozimmu_handle_t h, ozimmu_op_t transA,
                                  ozimmu_op_t transB, int64_t m, int64_t n, int64_t k,
                                  const double *alpha, const double *A, int64_t lda,
                                  const double *B, int64_t ldb, const double *beta, double *C,
                                  int64_t ldc, int num_slices);

/* Complex GEMM (NEXT row f1; "separating the real and imaginary parts ... while
 * splitting").  Complex numbers are interleaved (re, im) doubles (cuDoubleComplex layout);
 * lda / ldb / ldc count complex elements; alpha and beta point to 2 doubles (re, im);
 * OZIMMU_OP_C = conjugate transpose.  Reading A16: the real embedding
 *   Ahat(i,2l) = Re op(A)(i,l), Ahat(i,2l+1) = Im op(A)(i,l),
 *   Bhat(:,2j) = (Re, -Im) and Bhat(:,2j+1) = (Im, Re) of op(B)(:,j) interleaved along K,
 * is computed by the method (s slices, K' = 2k, one shared exponent per complex row of op(A)
 * and complex column of op(B)); X = Xhat(:,2j) + i Xhat(:,2j+1);
 * C = alpha X (+ beta C) with z = a x as re = fma(ar, xr, -(ai xi)), im = fma(ar, xi, ai xr).
 * Effective rate: 8mnk flops. */
OZIMMU_API ozimmu_status_t ozimmu_zgemm(ozimmu_handle_t h, ozimmu_op_t transA, ozimmu_op_t transB,
                             int64_t m, int64_t n, int64_t k, const double *alpha,
                             const double *A, int64_t lda, const double *B, int64_t ldb,
                             const double *beta, double *C, int64_t ldc, int num_slices);
/* Workspace bytes for ozimmu_zgemm (0 on invalid input). */
OZIMMU_API size_t ozimmu_zgemm_workspace_bytes(ozimmu_op_t transA, ozimmu_op_t transB, int64_t m,
                                    int64_t n, int64_t k, int num_slices);

/* INT8-AUTO (NEXT row f2; "we select the number of splits so that the average
 * mantissa loss in the splitting process is equal to or smaller than a threshold T"): the
 * splits are chosen per call by one of two rules; both scan every element of both operands
 * on the device and read a few bytes back (the call synchronises its stream once).
 *
 * OZIMMU_AUTO_LOSS -- the paper's rule (reading A17): for a nonzero finite x of a row of
 * op(A) / column of op(B) with exponent E, the significant bits of |x|/2^E occupy positions
 * lead = E - ilogb(x) .. t_last = lead + vlen - 1 (vlen: bits from the MSB to the last 1 of
 * the significand); loss_s(x) = min(vlen, max(0, t_last - s*w)); s = the smallest
 * s in [1, s_max] whose mean loss over the nonzero finite elements is <= T for both operands.
 * ozimmu_set_auto(h, T, s_max) selects it (T >= 0; T = 0 is the paper's lossless setting).
 *
 * OZIMMU_AUTO_ACCURACY (default) -- the k-aware rule the Discussion asks for (P:713-734:
 * "the accumulation length should be one of the key factors"; reading A18): with rho_v(t)
 * the relative l1 truncation residual of a vector after t digits (fixed-point upper estimate)
 * and rho_A(t) / rho_B(t) its maximum over the rows of op(A) / columns of op(B), s = the
 * smallest s in [1, s_max] with eta(s) = sum_{t=0..s} rho_A(t) rho_B(s-t) <= tau u sqrt(k)
 * (u = 2^-53, k the accumulation length, 2k for ZGEMM's embedding): the predicted Ozaki error
 * in units of |A||B| no larger than tau times FP64 DGEMM's probabilistic error level.
 * ozimmu_set_auto_accuracy(h, tau, s_max) selects it (tau > 0; default tau = 1).
 *
 * s_max in [1, OZIMMU_MAX_SLICES], default 18; a call that reaches s_max without
 * meeting its criterion sets ozimmu_report_t.auto_capped.  ozimmu_auto_splits returns the s a
 * num_slices = 0 call would use (synchronises the stream). */
#define OZIMMU_AUTO_LOSS 1
#define OZIMMU_AUTO_ACCURACY 2
OZIMMU_API ozimmu_status_t ozimmu_set_auto(ozimmu_handle_t h, double threshold, int s_max);
OZIMMU_API ozimmu_status_t ozimmu_set_auto_accuracy(ozimmu_handle_t h, double tau, int s_max);
OZIMMU_API ozimmu_status_t ozimmu_auto_splits(ozimmu_handle_t h, ozimmu_op_t transA,
                                   ozimmu_op_t transB, int64_t m, int64_t n, int64_t k,
                                   const double *A, int64_t lda, const double *B, int64_t ldb,
                                   int *num_slices_out);

/* Strided-batched forms (NEXT row f3: the quantum-circuit gate application of P:645-650 as a
 * batch of matmul-(2^d, 2^o, 2^d) products): C_b = alpha op(A_b) op(B_b) + beta C_b for
 * b = 0..batch-1, X_b = X + b*strideX (strides in elements: doubles for D, complex for Z).
 * Each item is bitwise what ozimmu_dgemm / ozimmu_zgemm would return for it.  For D with a
 * shared op(B) (strideB = 0, num_slices > 0) B is sliced once and its B-slice buffer reused. */
OZIMMU_API ozimmu_status_t ozimmu_dgemm_strided_batched(ozimmu_handle_t h, ozimmu_op_t transA,
                                             ozimmu_op_t transB, int64_t m, int64_t n, int64_t k,
                                             const double *alpha, const double *A, int64_t lda,
                                             int64_t strideA, const double *B, int64_t ldb,
                                             int64_t strideB, const double *beta, double *C,
                                             int64_t ldc, int64_t strideC, int64_t batch,
                                             int num_slices);
OZIMMU_API ozimmu_status_t ozimmu_zgemm_strided_batched(ozimmu_handle_t h, ozimmu_op_t transA,
                                             ozimmu_op_t transB, int64_t m, int64_t n, int64_t k,
                                             const double *alpha, const double *A, int64_t lda,
                                             int64_t strideA, const double *B, int64_t ldb,
                                             int64_t strideB, const double *beta, double *C,
                                             int64_t ldc, int64_t strideC, int64_t batch,
                                             int num_slices);

/* ---- split-phase entry points (multi-GPU: slice B once, broadcast, reuse) -----
 * A "B-slice buffer" is one contiguous device buffer holding the INT8 planes of
 * the columns of op(B) plus their int32 exponents, in the exact layout the GEMM
 * kernel reads (so it can be moved between GPUs as plain bytes, e.g. one NCCL
 * broadcast over NVLink -- SURVEY s8e).  Its size depends only on (n, k, s). */
OZIMMU_API size_t ozimmu_b_slices_bytes(int64_t n, int64_t k, int num_slices);
/* Slice op(B) (k x n) into b_slices (device, ozimmu_b_slices_bytes bytes,
 * 256-byte aligned).  Alg. 4 applied to the columns of op(B). */
OZIMMU_API ozimmu_status_t ozimmu_slice_b(ozimmu_handle_t h, ozimmu_op_t transB, int64_t k, int64_t n,
                               const double *B, int64_t ldb, int num_slices, void *b_slices);
/* As ozimmu_dgemm, with op(B) given as a B-slice buffer produced by ozimmu_slice_b
 * for the same (k, n, num_slices).  Workspace need: ozimmu_workspace_bytes(.., n=0, ..). */
OZIMMU_API ozimmu_status_t ozimmu_dgemm_presliced_b(ozimmu_handle_t h, ozimmu_op_t transA, int64_t m,
                                         int64_t n, int64_t k, const double *alpha,
                                         const double *A, int64_t lda, const void *b_slices,
                                         const double *beta, double *C, int64_t ldc,
                                         int num_slices);

/* ---- multi-GPU: C row blocks, B sliced once and broadcast ---------------
 * BASELINE north_star: "C is partitioned into row blocks (2-D blocks for large n).  Each GPU
 * slices its own A rows, B's slices are computed once and NCCL-broadcast over NVLink, and there
 * are no other collectives."  One process (and one handle) per GPU.  Rank r passes its rows of
 * op(A) (A_local, m_local rows, stored like A with leading dimension lda) and of C (C_local,
 * ldc); op(B) (k x n) is read on `root` only (B may be NULL elsewhere).  The root slices op(B)
 * in column chunks into a B-slice buffer (Alg. 4 on the columns of op(B)) and every chunk is
 * broadcast to all ranks (s + 1 contiguous pieces: the chunk's rows of each INT8 plane and its
 * int32 exponents) on the handle's collective stream; each rank's GEMM on a chunk waits only
 * for that chunk, so later broadcasts overlap earlier GEMMs.  While broadcasts are in flight
 * the fused GEMM leaves reserve_sms SMs free for the collective kernels (ozimmu_set_dist).
 * C_local is bitwise what ozimmu_dgemm returns for those rows (no reduction exists; every
 * element has the single-GPU operation sequence).  The 2-D partition is the same call on a
 * communicator of {root} + one grid column, with that column block of op(B) as B (n = its
 * width) and m_local = 0 on the root for the blocks it does not own.
 * Every rank of the communicator must make the call, in the same order, with the same transB,
 * n, k, ldb, alpha (= 0 or not), num_slices and ozimmu_set_dist settings.  num_slices = 0
 * (INT8-AUTO) returns UNSUPPORTED: choosing s would need A's statistics from every rank.
 * Asynchronous on the handle's stream like ozimmu_dgemm (the caller synchronises).
 * Errors: as ozimmu_dgemm; OZIMMU_ERR_NCCL if libnccl cannot be loaded or a broadcast fails. */
#define OZIMMU_NCCL_UNIQUE_ID_BYTES 128
/* ncclGetUniqueId through the library's NCCL (root only; share the 128 bytes with the other
 * ranks, e.g. through torch.distributed). */
OZIMMU_API ozimmu_status_t ozimmu_nccl_get_unique_id(void *id_out);
/* ncclCommInitRank(Config) on `device` (an ncclComm_t returned as void*).  max_ctas > 0 caps
 * the CTAs of the communicator's kernels (ncclConfig_t.maxCTAs; pair it with reserve_sms). */
OZIMMU_API ozimmu_status_t ozimmu_nccl_comm_init(void **comm_out, int nranks, const void *id,
                                      int rank, int device, int max_ctas);
OZIMMU_API ozimmu_status_t ozimmu_nccl_comm_destroy(void *comm);
/* Multi-GPU settings of a handle: chunk_cols = columns per broadcast chunk (0: about n/8),
 * reserve_sms = SMs the GEMM leaves to the collective while broadcasts are in flight (default
 * 8), bcast_fp64 = 1 broadcasts FP64 op(B) (8 bytes per element instead of s) and slices each
 * chunk on every rank (needs transB = N and ldb = k, else the INT8 planes are broadcast). */
OZIMMU_API ozimmu_status_t ozimmu_set_dist(ozimmu_handle_t h, int chunk_cols, int reserve_sms,
                                int bcast_fp64);
/* comm: an ncclComm_t (e.g. from ozimmu_nccl_comm_init); rank and size are taken from it. */
OZIMMU_API ozimmu_status_t ozimmu_dgemm_nccl(ozimmu_handle_t h, void *comm, int root,
                                  ozimmu_op_t transA, ozimmu_op_t transB, int64_t m_local,
                                  int64_t n, int64_t k, const double *alpha,
                                  const double *A_local, int64_t lda, const double *B,
                                  int64_t ldb, const double *beta, double *C_local, int64_t ldc,
                                  int num_slices);
/* The same driver over a caller-supplied broadcast: fn(ctx, buf, bytes, root, stream) must
 * deliver `bytes` device bytes at buf from rank `root` to every rank, ordered after the work
 * already enqueued on `stream` (a cudaStream_t as void*) and before work enqueued on it later
 * (a synchronous implementation may synchronise the stream first); it returns 0 on success.
 * Used by the tests to run the multi-rank logic over gloo. */
typedef int (*ozimmu_bcast_fn)(void *ctx, void *buf, size_t bytes, int root, void *stream);
OZIMMU_API ozimmu_status_t ozimmu_dgemm_bcast(ozimmu_handle_t h, ozimmu_bcast_fn fn, void *ctx,
                                   int rank, int nranks, int root, ozimmu_op_t transA,
                                   ozimmu_op_t transB, int64_t m_local, int64_t n, int64_t k,
                                   const double *alpha, const double *A_local, int64_t lda,
                                   const double *B, int64_t ldb, const double *beta,
                                   double *C_local, int64_t ldc, int num_slices);

/* ---- debug / parity exports (same kernels as the product path) -------------- */

/* Slices and exponents of the rows of op(M) (is_rows = 1: M is the A operand,
 * op(M) is rows x kdim) or of the columns of op(M) (is_rows = 0: M is the B
 * operand, op(M) is kdim x rows).  planes_out: device int8 [s][rows][kdim]
 * (digit p of vector r, element l at ((p-1)*rows + r)*kdim + l);
 * exps_out: device int32 [rows]; a vector holding NaN/Inf gets exponent
 * OZIMMU_EXP_NONFINITE and zero digits. */
#define OZIMMU_EXP_NONFINITE 0x7fffffff
OZIMMU_API ozimmu_status_t ozimmu_debug_split(ozimmu_handle_t h, ozimmu_op_t op, int is_rows, int64_t rows,
                                   int64_t kdim, const double *M, int64_t ld, int num_slices,
                                   int8_t *planes_out, int32_t *exps_out);
/* Exact level sums L_g, g = 2..s+1, computed by the tcgen05 GEMM kernel:
 * Lg_out: device int64 [s][n][m] (level g at (g-2)*m*n + i + j*m). */
OZIMMU_API ozimmu_status_t ozimmu_debug_level_sums(ozimmu_handle_t h, ozimmu_op_t transA,
                                        ozimmu_op_t transB, int64_t m, int64_t n, int64_t k,
                                        const double *A, int64_t lda, const double *B,
                                        int64_t ldb, int num_slices, int64_t *Lg_out);
/* One INT8 x INT8 -> INT32 product P = Ai * Bj^T on the tcgen05 kernel.
 * Ai: device int8 [m][k] (row i contiguous), Bj: device int8 [n][k] (column j of
 * the right operand contiguous), P_out: device int32 [n][m] (P(i,j) at i + j*m).
 * Requires k * max|Ai| * max|Bj| <= 2^31 - 1 (caller's responsibility). */
OZIMMU_API ozimmu_status_t ozimmu_debug_pair(ozimmu_handle_t h, const int8_t *Ai, const int8_t *Bj,
                                  int64_t m, int64_t n, int64_t k, int32_t *P_out);
/* Statistics of the accuracy-targeted INT8-AUTO rule (reading A18, Discussion P:713-734) for
 * the vectors of one operand, as computed on the device before a num_slices = 0 call: rho[t],
 * t = 0..s_max = max over the vectors (rows of op(M) for is_rows = 1, columns of op(M) for
 * is_rows = 0; vector layout as ozimmu_debug_split) of the relative l1 truncation residual
 * after t digits of w bits, ((double)N_t / (double)D) 2^(-wt) from the exact fixed-point sums
 * N_t = sum ceil(frac(|x| 2^(wt-E)) 2^32), D = sum floor(|x| 2^(32-E)); vectors holding NaN/Inf
 * or only zeros are skipped (rho = 0 for all t if every vector is).  M: device; rho_out: HOST
 * double [s_max + 1]; w in [5, 7], s_max in [1, 32].  Synchronises the handle's stream. */
OZIMMU_API ozimmu_status_t ozimmu_debug_auto_rho(ozimmu_handle_t h, ozimmu_op_t op, int is_rows,
                                      int64_t rows, int64_t kdim, const double *M, int64_t ld,
                                      int w, int s_max, double *rho_out);

#ifdef __cplusplus
}
#endif
#endif /* OZIMMU_H */
