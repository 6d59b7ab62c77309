// api.cu -- host runtime behind include/ozimmu.h: handle, argument validation, plan,
// workspace, and the launch sequence  slice(A) -> slice(B) -> fused tcgen05 GEMM+epilogue.
#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <vector>
#include <cstring>
#include <cstdio>
#include <cuda_runtime.h>

#include "ozimmu.h"
#include "internal.h"
#include "handle.h"

using namespace ozimmu;
using namespace ozimmu::rt;

namespace ozimmu {
namespace rt {

// B-slice buffer: planes [s][n][k_pad] (reversed slice order) | int32 exponents [n]
size_t b_buf_planes_bytes(int64_t n, int64_t k_pad, int s) {
    return align_up((size_t)s * (size_t)n * (size_t)k_pad);
}
size_t b_buf_bytes(int64_t n, int64_t k_pad, int s) {
    return b_buf_planes_bytes(n, k_pad, s) + align_up(sizeof(int32_t) * (size_t)n);
}

Layout layout(int64_t m, int64_t n, int64_t k_pad, int s, size_t scratch) {
    Layout L;
    size_t off = 0;
    L.a_planes = off;
    off += align_up((size_t)s * m * k_pad);
    L.a_exp = off;
    off += align_up(sizeof(int32_t) * (size_t)m);
    L.b_buf = off;
    off += b_buf_bytes(n, k_pad, s);
    L.keys = off;
    off += align_up(split_scratch_bytes(m > n ? m : n));
    L.keys_b = off;  // B's slicing scratch (B is sliced concurrently with A)
    off += align_up(split_scratch_bytes(n));
    L.sync = off;
    off += kAlign;
    L.scratch = off;
    off += align_up(scratch);
    L.total = off;
    return L;
}

bool valid_op(ozimmu_op_t op) { return op == OZIMMU_OP_N || op == OZIMMU_OP_T || op == OZIMMU_OP_C; }

ozimmu_status_t get_ws(ozimmu_handle_t h, size_t need, void **ws) {
    if (h->user_ws) {
        if (need > h->user_ws_bytes) return OZIMMU_ERR_WORKSPACE;
        *ws = h->user_ws;
        return OZIMMU_SUCCESS;
    }
    if (need > h->own_ws_bytes) {
        if (h->own_ws) {
            cudaStreamSynchronize(h->stream);  // the old buffer may be in use by queued work
            cudaFree(h->own_ws);
            h->own_ws = nullptr;
            h->own_ws_bytes = 0;
        }
        size_t sz = need + need / 8;
        if (cudaMalloc(&h->own_ws, sz) != cudaSuccess) {
            cudaGetLastError();
            return OZIMMU_ERR_WORKSPACE;
        }
        h->own_ws_bytes = sz;
    }
    *ws = h->own_ws;
    return OZIMMU_SUCCESS;
}

__global__ void k_scale_c(double *C, int64_t ldc, int64_t m, int64_t n, double beta) {
    const int64_t total = m * n;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t % m, j = t / m;
        double *c = C + i + j * ldc;
        *c = beta == 0.0 ? 0.0 : __dmul_rn(beta, *c);
    }
}



// C = beta C for complex C (interleaved), same product as the ZGEMM epilogue (reading A16).
__global__ void k_scale_z(double2 *C, int64_t ldc, int64_t m, int64_t n, double br, double bi) {
    const int64_t total = m * n;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t % m, j = t / m;
        double2 *c = C + i + j * ldc;
        if (br == 0.0 && bi == 0.0) {
            *c = make_double2(0.0, 0.0);
        } else {
            const double2 v = *c;
            *c = make_double2(__fma_rn(br, v.x, -__dmul_rn(bi, v.y)), __fma_rn(br, v.y, __dmul_rn(bi, v.x)));
        }
    }
}

ozimmu_status_t cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return OZIMMU_SUCCESS;
    cudaGetLastError();
    return OZIMMU_ERR_CUDA;
}

// Common validation for the A side and the sizes.
ozimmu_status_t check_common(ozimmu_handle_t h, ozimmu_op_t transA, int64_t m, int64_t n,
                             int64_t k, const double *alpha, const double *A, int64_t lda,
                             const double *beta, double *C, int64_t ldc, int s) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (!valid_op(transA)) return OZIMMU_ERR_INVALID_VALUE;
    if (m < 0 || n < 0 || k < 0) return OZIMMU_ERR_INVALID_VALUE;
    if (!alpha || !beta) return OZIMMU_ERR_INVALID_VALUE;
    const int64_t arows = transA == OZIMMU_OP_N ? m : k;
    if (lda < (arows > 1 ? arows : 1)) return OZIMMU_ERR_INVALID_VALUE;
    if (ldc < (m > 1 ? m : 1)) return OZIMMU_ERR_INVALID_VALUE;
    if (m > 0 && n > 0 && !C) return OZIMMU_ERR_INVALID_VALUE;
    if (m > 0 && k > 0 && *alpha != 0.0 && !A) return OZIMMU_ERR_INVALID_VALUE;
    if (s < 0 || s > OZIMMU_MAX_SLICES) return OZIMMU_ERR_INVALID_VALUE;  // 0 = INT8-AUTO
    if (k > OZIMMU_MAX_K) return OZIMMU_ERR_UNSUPPORTED;
    return OZIMMU_SUCCESS;
}

void fill_report(ozimmu_handle_t h, int s, int w, int64_t m, int64_t n, int64_t k,
                 const GemmPlan *gp, int launches, int64_t slice_bytes) {
    ozimmu_report_t &r = h->report;
    r.num_slices = s;
    r.slice_width = w;
    r.gemm_pairs = (int64_t)s * (s + 1) / 2;
    r.int8_macs = r.gemm_pairs * m * n * k;
    r.slice_bytes = slice_bytes;
    r.tile_n = gp ? gp->tile_n : 0;
    r.k_block = gp ? gp->k_block : 0;
    r.stages = gp ? gp->stages : 0;
    r.k_chunks = gp ? gp->k_chunks : 0;
    r.launches = launches;
    r.acc_regions = gp ? gp->T : 0;
    r.auto_mode = 0;
    r.auto_capped = 0;
}

// After a num_slices = 0 call: which rule chose s and whether it hit s_max.
void note_auto(ozimmu_handle_t h) {
    h->report.auto_mode = h->auto_mode;
    h->report.auto_capped = h->auto_last_capped ? 1 : 0;
}

// C = beta C (alpha == 0 or k == 0 quick return; A and B are not read).
ozimmu_status_t scale_only(ozimmu_handle_t h, int64_t m, int64_t n, double beta, double *C,
                           int64_t ldc) {
    int launches = 0;
    if (beta != 1.0) {
        int64_t blocks = ceil_div(m * n, 256);
        if (blocks > 8 * (int64_t)h->num_sms) blocks = 8 * (int64_t)h->num_sms;
        k_scale_c<<<(unsigned)blocks, 256, 0, h->stream>>>(C, ldc, m, n, beta);
        ++launches;
        if (cudaGetLastError() != cudaSuccess) return OZIMMU_ERR_CUDA;
    }
    fill_report(h, 0, 0, m, n, 0, nullptr, launches, 0);
    return OZIMMU_SUCCESS;
}

// Slice op(A): rows of op(A) are contiguous along k iff transA != N.
cudaError_t slice_a(ozimmu_handle_t h, ozimmu_op_t transA, int64_t m, int64_t k, int64_t k_pad,
                    const double *A, int64_t lda, int s, int w, int8_t *planes, int32_t *E,
                    int32_t *keys, int *launches, BatchMap vm) {
    const bool contig = transA != OZIMMU_OP_N;
    return launch_split(A, lda, contig, m, k, k_pad, s, w, /*reverse=*/false, planes,
                        (int64_t)m * k_pad, E, keys, h->num_sms, h->stream, launches, 0, 0, vm);
}

// Slice op(B) into a B-slice buffer: columns of op(B) are contiguous along k iff transB == N.
cudaError_t slice_b(ozimmu_handle_t h, ozimmu_op_t transB, int64_t k, int64_t n, int64_t k_pad,
                    const double *B, int64_t ldb, int s, int w, uint8_t *bbuf, int32_t *keys,
                    int *launches, BatchMap vm, cudaStream_t st) {
    const bool contig = transB == OZIMMU_OP_N;
    int8_t *planes = reinterpret_cast<int8_t *>(bbuf);
    int32_t *E = reinterpret_cast<int32_t *>(bbuf + b_buf_planes_bytes(n, k_pad, s));
    return launch_split(B, ldb, contig, n, k, k_pad, s, w, /*reverse=*/true, planes,
                        (int64_t)n * k_pad, E, keys, h->num_sms, st ? st : h->stream, launches, 0,
                        0, vm);
}

// Fork / join helpers: work on h->aux runs concurrently with h->stream between them.
cudaError_t aux_fork(ozimmu_handle_t h) {
    if (!h->aux) {
        cudaError_t e = cudaStreamCreateWithFlags(&h->aux, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaEventRecord(h->ev_fork, h->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->aux, h->ev_fork, 0);
    return e;
}
cudaError_t aux_join(ozimmu_handle_t h) {
    cudaError_t e = cudaEventRecord(h->ev_join, h->aux);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->stream, h->ev_join, 0);
    return e;
}

// kAutoNS (handle.h): per-operand statistics slots (s_max <= 32)

// f2 INT8-AUTO decision (host side, from the device statistics of both operands; stat holds
// [2][kAutoNS] uint64).  LOSS (reading A17): the smallest s <= s_max whose mean
// mantissa loss is <= T for both operands.  ACCURACY (reading A18, Discussion P:713-734):
// the smallest s <= s_max with eta(s) = sum_{t=0..s} rho_A(t) rho_B(s-t) <= tau u sqrt(k_acc),
// u = 2^-53, summed in the order t = 0..s (the oracle's rule, oz_ref_auto_splits_acc).
// Candidates s = 1..s_lim (the statistics hold t <= s_lim); s_lim if none (*capped = true).
int auto_decide(ozimmu_handle_t h, const unsigned long long *stat, int64_t k_acc, int s_lim,
                bool *capped) {
    const int s_max = s_lim;
    *capped = false;
    if (h->auto_mode == OZIMMU_AUTO_LOSS) {
        for (int s = 1; s <= s_max; ++s) {
            const double ma = stat[32] ? (double)stat[s - 1] / (double)stat[32] : 0.0;
            const double mb = stat[kAutoNS + 32] ? (double)stat[kAutoNS + s - 1] /
                                                       (double)stat[kAutoNS + 32] : 0.0;
            if (ma <= h->auto_T && mb <= h->auto_T) return s;
        }
    } else {
        double ra[kAutoNS], rb[kAutoNS];
        memcpy(ra, stat, sizeof(ra));
        memcpy(rb, stat + kAutoNS, sizeof(rb));
        const double target = h->auto_tau * ldexp(sqrt((double)k_acc), -53);
        for (int s = 1; s <= s_max; ++s) {
            double eta = 0.0;
            for (int t = 0; t <= s; ++t) {
                const double p = ra[t] * rb[s - t];
                eta = eta + p;
            }
            if (eta <= target) return s;
        }
    }
    *capped = true;
    return s_max;
}

// Device statistics of op(A)'s rows / op(B)'s columns for the handle's AUTO rule into
// stat_dev [2][kAutoNS] (zeroed here), on stream st.  scratch: auto_scratch_bytes(..).
size_t auto_scratch_bytes(ozimmu_handle_t h, int64_t rows) {
    const size_t keys = align_up(sizeof(int32_t) * (size_t)(rows > 0 ? rows : 1));
    if (h->auto_mode == OZIMMU_AUTO_LOSS) return keys;
    const size_t r = align_up(trunc_residual_scratch(rows > 0 ? rows : 1, h->auto_smax));
    return r > keys ? r : keys;
}
cudaError_t auto_stats(ozimmu_handle_t h, const double *M, int64_t ld, bool contiguous,
                       int64_t rows, int64_t kdim, int w, int s_lim, unsigned long long *stat_op,
                       void *scratch, cudaStream_t st, int *launches, int cpx) {
    if (h->auto_mode == OZIMMU_AUTO_LOSS)
        return launch_mantissa_loss(M, ld, contiguous, rows, kdim, w, s_lim, stat_op,
                                    static_cast<int32_t *>(scratch), h->num_sms, st, launches, cpx);
    return launch_trunc_residual(M, ld, contiguous, rows, kdim, w, s_lim, stat_op, scratch,
                                 h->num_sms, st, launches, cpx);
}

// First-pass candidate limit: the accuracy rule's statistics cost grows with the number of t
// they cover, and s <= 12 decides almost every input; a capped first pass is redone with
// s_max (the statistics for t <= 12 are the same numbers, so the decision is unchanged).
int auto_first_limit(ozimmu_handle_t h) {
    return h->auto_mode == OZIMMU_AUTO_ACCURACY && h->auto_smax > 12 ? 12 : h->auto_smax;
}

// f2 INT8-AUTO: the statistics of both operands on the device, one D2H read (the call
// synchronises the stream), then auto_decide.
ozimmu_status_t auto_select(ozimmu_handle_t h, ozimmu_op_t transA, ozimmu_op_t transB, int64_t m,
                            int64_t n, int64_t k, const double *A, int64_t lda, const double *B,
                            int64_t ldb, int *s_out, int *launches, bool cpx) {
    const int64_t k_acc = cpx ? 2 * k : k;  // accumulation length of the (embedded) GEMM
    const int w = slice_width(k_acc);
    if (!h->auto_dev &&
        cudaMalloc(&h->auto_dev, 2 * kAutoNS * sizeof(unsigned long long)) != cudaSuccess) {
        cudaGetLastError();
        return OZIMMU_ERR_WORKSPACE;
    }
    void *ws = nullptr;
    ozimmu_status_t st = get_ws(h, auto_scratch_bytes(h, m > n ? m : n), &ws);
    if (st) return st;
    const bool ac = transA != OZIMMU_OP_N, bc = transB == OZIMMU_OP_N;
    bool capped = false;
    for (int lim = auto_first_limit(h);; lim = h->auto_smax) {
        cudaError_t e =
            cudaMemsetAsync(h->auto_dev, 0, 2 * kAutoNS * sizeof(unsigned long long), h->stream);
        // complex: contiguous vectors are 2k doubles (ld in doubles), strided ones k pairs
        if (e == cudaSuccess)
            e = auto_stats(h, A, cpx && ac ? 2 * lda : lda, ac, m, cpx && ac ? 2 * k : k, w, lim,
                           h->auto_dev, ws, h->stream, launches, cpx);
        if (e == cudaSuccess)
            e = auto_stats(h, B, cpx && bc ? 2 * ldb : ldb, bc, n, cpx && bc ? 2 * k : k, w, lim,
                           h->auto_dev + kAutoNS, ws, h->stream, launches, cpx);
        unsigned long long host[2 * kAutoNS];
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(host, h->auto_dev, sizeof(host), cudaMemcpyDeviceToHost, h->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess) return cuda_status(e);
        *s_out = auto_decide(h, host, k_acc, lim, &capped);
        if (!capped || lim == h->auto_smax) break;
    }
    h->auto_last_s = *s_out;
    h->auto_last_capped = capped;
    return OZIMMU_SUCCESS;
}

// The fused tcgen05 GEMM + FP64 epilogue (A4 + A5) on sliced operands.  b_plane_rows: rows
// per B plane in memory (0 = n; a column chunk of a wider B-slice buffer otherwise).
cudaError_t fused_gemm(ozimmu_handle_t h, const GemmPlan &gp, int64_t m, int64_t n, int64_t k_pad,
                       int s, int w, const int8_t *a_planes, const int32_t *EA,
                       const int8_t *b_planes, const int32_t *EB, int64_t b_plane_rows,
                       double alpha, double beta, double *C, int64_t ldc, int64_t *scratch,
                       unsigned int *sync, int *launches, BatchMap crow, BatchMap ccol,
                       int64_t a_plane_rows, bool counter_zeroed) {
    GemmArgs ga{};
    ga.counter_zeroed = counter_zeroed;
    ga.a_plane_rows = a_plane_rows;
    ga.c_rows = crow;
    ga.c_cols = ccol;
    ga.a_planes = a_planes;
    ga.b_planes = b_planes;
    ga.b_plane_rows = b_plane_rows;
    ga.EA = EA;
    ga.EB = EB;
    ga.m = m;
    ga.n = n;
    ga.k_pad = k_pad;
    ga.s = s;
    ga.w = w;
    ga.alpha = alpha;
    ga.beta = beta;
    ga.C = C;
    ga.ldc = ldc;
    ga.chunk_scratch = scratch;
    // soft per-wave grid barrier (L2 reuse); OZIMMU_NO_WAVE_SYNC=1 disables (experiments)
    static const bool no_sync = getenv("OZIMMU_NO_WAVE_SYNC") != nullptr;
    ga.wave_counter = no_sync ? nullptr : sync;
    // development instrumentation: OZIMMU_STATS=1 -> per-CTA stall counters, dumped below
    static const bool want_stats = getenv("OZIMMU_STATS") != nullptr;
    static long long *stats_buf = nullptr;
    if (want_stats && !stats_buf) cudaMalloc(&stats_buf, 14 * 1024 * sizeof(long long));
    ga.stats = want_stats ? stats_buf : nullptr;
    cudaError_t e = launch_gemm(ga, gp, EPI_DGEMM, h->stream, launches);
    if (e != cudaSuccess || !ga.stats) return e;
    // development only: synchronous dump of the stall counters
    constexpr int NS = 14;
    static long long host[NS * 1024];
    cudaStreamSynchronize(h->stream);
    cudaMemcpy(host, ga.stats, sizeof(long long) * NS * gp.grid, cudaMemcpyDeviceToHost);
    double acc[NS] = {0};
    for (int c = 0; c < gp.grid; ++c)
        for (int i = 0; i < NS; ++i) acc[i] += (double)host[c * NS + i];
    const char *names[NS] = {"total", "mma_wait_b", "mma_wait_a", "mma_wait_tmem", "prod_wave",
                             "prod_wait_a", "prod_wait_b", "epi_busy", "epi_tmem", "epi_store",
                             "mma_wait_a_first_kb", "mma_wait_b_kb0", "mma_ns", "unused"};
    fprintf(stderr, "[ozimmu stats] grid=%d avg cycles:", gp.grid);
    for (int i = 0; i < NS; ++i) fprintf(stderr, " %s=%.0f", names[i], acc[i] / gp.grid);
    fprintf(stderr, "\n");
    return cudaSuccess;
}

// amap / bmap: stacked batches of op(A) rows / op(B) columns; crow / ccol: the matching
// row / column maps of C (strided-batched calls with a shared operand).
ozimmu_status_t gemm_core(ozimmu_handle_t h, ozimmu_op_t transA, int64_t m, int64_t n, int64_t k,
                          double alpha, const double *A, int64_t lda, const uint8_t *bbuf_ext,
                          ozimmu_op_t transB, const double *B, int64_t ldb, double beta,
                          double *C, int64_t ldc, int s, BatchMap amap, BatchMap bmap,
                          BatchMap crow, BatchMap ccol) {
    const int w = slice_width(k);
    const int64_t k_pad = round_up(k, 16);
    GemmPlan gp;
    if (!plan_gemm(s, w, m, n, k_pad, gemm_sms(h), &gp)) return OZIMMU_ERR_UNSUPPORTED;
    const Layout L = layout(m, bbuf_ext ? 0 : n, k_pad, s, chunk_scratch_bytes(gp, s));
    void *ws = nullptr;
    ozimmu_status_t st = get_ws(h, L.total, &ws);
    if (st) return st;
    uint8_t *base = static_cast<uint8_t *>(ws);
    int8_t *a_planes = reinterpret_cast<int8_t *>(base + L.a_planes);
    int32_t *EA = reinterpret_cast<int32_t *>(base + L.a_exp);
    int32_t *keys = reinterpret_cast<int32_t *>(base + L.keys);
    const uint8_t *bbuf = bbuf_ext;
    int launches = 0;
    int64_t slice_bytes = (int64_t)s * m * k_pad + 4 * m;
    mark(h, PH_START);
    // Small calls: both operands in one launch on the handle's stream (k_split_small), which
    // also zeroes the GEMM's wave counter.
    bool counter_zeroed = false;
    if (!bbuf_ext && split_small_ok(m, n, k_pad)) {
        uint8_t *b = base + L.b_buf;
        SmallOp oa{A, lda, m, k, k_pad, transA != OZIMMU_OP_N, 0, a_planes, m * k_pad, EA,
                   amap.per_item, amap.stride};
        SmallOp ob{B, ldb, n, k, k_pad, transB == OZIMMU_OP_N, 1,
                   reinterpret_cast<int8_t *>(b), n * k_pad,
                   reinterpret_cast<int32_t *>(b + b_buf_planes_bytes(n, k_pad, s)),
                   bmap.per_item, bmap.stride};
        mark(h, PH_B);
        cudaError_t e = launch_split_small(oa, ob, s, w, reinterpret_cast<unsigned int *>(base + L.sync),
                                           h->num_sms, h->stream, &launches);
        if (e != cudaSuccess) return cuda_status(e);
        mark(h, PH_A);
        bbuf = b;
        slice_bytes += (int64_t)s * n * k_pad + 4 * n;
        counter_zeroed = true;
    }
    // op(B) is sliced on the handle's second stream while op(A) is sliced on its stream
    // (separate exponent-scan scratch); the GEMM waits for both.
    const bool fork = !bbuf_ext && !counter_zeroed;
    if (fork) {
        uint8_t *b = base + L.b_buf;
        cudaError_t e = aux_fork(h);
        if (e != cudaSuccess) return cuda_status(e);
        e = slice_b(h, transB, k, n, k_pad, B, ldb, s, w, b,
                    reinterpret_cast<int32_t *>(base + L.keys_b), &launches, bmap, h->aux);
        mark(h, PH_B, h->aux);
        if (e != cudaSuccess) {
            aux_join(h);  // never leave forked work unjoined (stream capture, later ordering)
            return cuda_status(e);
        }
        bbuf = b;
        slice_bytes += (int64_t)s * n * k_pad + 4 * n;
    } else if (!counter_zeroed) {
        mark(h, PH_B);
    }
    cudaError_t e = cudaSuccess;
    if (!counter_zeroed) {
        e = slice_a(h, transA, m, k, k_pad, A, lda, s, w, a_planes, EA, keys, &launches, amap);
        mark(h, PH_A);
    }
    if (fork) {
        const cudaError_t ej = aux_join(h);
        if (e == cudaSuccess) e = ej;
    }
    if (e != cudaSuccess) return cuda_status(e);
    mark(h, PH_GEMM0);
    e = fused_gemm(h, gp, m, n, k_pad, s, w, a_planes, EA, reinterpret_cast<const int8_t *>(bbuf),
                   reinterpret_cast<const int32_t *>(bbuf + b_buf_planes_bytes(n, k_pad, s)), 0,
                   alpha, beta, C, ldc, reinterpret_cast<int64_t *>(base + L.scratch),
                   reinterpret_cast<unsigned int *>(base + L.sync), &launches, crow, ccol, 0,
                   counter_zeroed);
    if (e != cudaSuccess) return cuda_status(e);
    mark(h, PH_GEMM1);
    mark_done(h);
    fill_report(h, s, w, m, n, k, &gp, launches, slice_bytes);
    return OZIMMU_SUCCESS;
}

}  // namespace rt
}  // namespace ozimmu

extern "C" {

int ozimmu_version(void) { return 100; }

const char *ozimmu_status_string(ozimmu_status_t s) {
    switch (s) {
    case OZIMMU_SUCCESS: return "OZIMMU_SUCCESS";
    case OZIMMU_ERR_INVALID_VALUE: return "OZIMMU_ERR_INVALID_VALUE";
    case OZIMMU_ERR_UNSUPPORTED: return "OZIMMU_ERR_UNSUPPORTED";
    case OZIMMU_ERR_WORKSPACE: return "OZIMMU_ERR_WORKSPACE";
    case OZIMMU_ERR_CUDA: return "OZIMMU_ERR_CUDA";
    case OZIMMU_ERR_NOT_INITIALIZED: return "OZIMMU_ERR_NOT_INITIALIZED";
    case OZIMMU_ERR_NCCL: return "OZIMMU_ERR_NCCL";
    }
    return "OZIMMU_UNKNOWN_STATUS";
}

ozimmu_status_t ozimmu_create(ozimmu_handle_t *h, int device) {
    if (!h) return OZIMMU_ERR_INVALID_VALUE;
    *h = nullptr;
    int major = 0, minor = 0, sms = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
        cudaGetLastError();
        return OZIMMU_ERR_CUDA;
    }
    if (major != 10 || minor != 0) return OZIMMU_ERR_CUDA;  // sm_100a binary only
    ozimmu_ctx *c = new ozimmu_ctx();
    c->device = device;
    c->num_sms = sms;
    *h = c;
    return OZIMMU_SUCCESS;
}

ozimmu_status_t ozimmu_timing_enable(ozimmu_handle_t h, int max_calls) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (max_calls < 0 || max_calls > 1 << 16) return OZIMMU_ERR_INVALID_VALUE;
    if (h->events) {
        cudaStreamSynchronize(h->stream);
        for (int i = 0; i < kPhases * h->timing_cap; ++i) cudaEventDestroy(h->events[i]);
        free(h->events);
        h->events = nullptr;
    }
    h->timing_cap = 0;
    h->timing_count = 0;
    if (max_calls == 0) return OZIMMU_SUCCESS;
    if (cudaSetDevice(h->device) != cudaSuccess) return OZIMMU_ERR_CUDA;
    h->events = static_cast<cudaEvent_t *>(calloc(kPhases * (size_t)max_calls, sizeof(cudaEvent_t)));
    if (!h->events) return OZIMMU_ERR_INVALID_VALUE;
    for (int i = 0; i < kPhases * max_calls; ++i)
        if (cudaEventCreate(&h->events[i]) != cudaSuccess) {
            for (int j = 0; j < i; ++j) cudaEventDestroy(h->events[j]);
            free(h->events);
            h->events = nullptr;
            cudaGetLastError();
            return OZIMMU_ERR_CUDA;
        }
    h->timing_cap = max_calls;
    return OZIMMU_SUCCESS;
}

int ozimmu_timing_read(ozimmu_handle_t h, ozimmu_timing_t *out, int max_out) {
    if (!h || (!out && max_out > 0)) return -1;
    const int n = h->timing_count;
    for (int c = 0; c < n && c < max_out; ++c) {
        cudaEvent_t *ev = h->events + kPhases * c;
        float t[3] = {0, 0, 0};
        const int from[3] = {PH_START, PH_START, PH_GEMM0}, to[3] = {PH_B, PH_A, PH_GEMM1};
        for (int p = 0; p < 3; ++p) {
            if (cudaEventSynchronize(ev[to[p]]) != cudaSuccess ||
                cudaEventElapsedTime(&t[p], ev[from[p]], ev[to[p]]) != cudaSuccess) {
                cudaGetLastError();
                return -1;
            }
        }
        out[c].slice_b_ms = t[0];
        out[c].slice_a_ms = t[1];
        out[c].gemm_ms = t[2];
    }
    h->timing_count = 0;
    return n;
}

ozimmu_status_t ozimmu_set_auto(ozimmu_handle_t h, double threshold, int s_max) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (!(threshold >= 0.0) || s_max < 1 || s_max > OZIMMU_MAX_SLICES) return OZIMMU_ERR_INVALID_VALUE;
    h->auto_mode = OZIMMU_AUTO_LOSS;
    h->auto_T = threshold;
    h->auto_smax = s_max;
    return OZIMMU_SUCCESS;
}

ozimmu_status_t ozimmu_set_auto_accuracy(ozimmu_handle_t h, double tau, int s_max) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (!(tau > 0.0) || !(tau < 1e300) || s_max < 1 || s_max > OZIMMU_MAX_SLICES)
        return OZIMMU_ERR_INVALID_VALUE;
    h->auto_mode = OZIMMU_AUTO_ACCURACY;
    h->auto_tau = tau;
    h->auto_smax = s_max;
    return OZIMMU_SUCCESS;
}

ozimmu_status_t ozimmu_auto_splits(ozimmu_handle_t h, ozimmu_op_t transA, ozimmu_op_t transB,
                                   int64_t m, int64_t n, int64_t k, const double *A, int64_t lda,
                                   const double *B, int64_t ldb, int *num_slices_out) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (!num_slices_out || !valid_op(transA) || !valid_op(transB) || m < 0 || n < 0 || k < 1)
        return OZIMMU_ERR_INVALID_VALUE;
    if (lda < (transA == OZIMMU_OP_N ? (m > 1 ? m : 1) : k) ||
        ldb < (transB == OZIMMU_OP_N ? k : (n > 1 ? n : 1)))
        return OZIMMU_ERR_INVALID_VALUE;
    if (k > OZIMMU_MAX_K) return OZIMMU_ERR_UNSUPPORTED;
    if ((m > 0 && !A) || (n > 0 && !B)) return OZIMMU_ERR_INVALID_VALUE;
    if (cudaSetDevice(h->device) != cudaSuccess) return OZIMMU_ERR_CUDA;
    int launches = 0;
    return auto_select(h, transA, transB, m, n, k, A, lda, B, ldb, num_slices_out, &launches);
}

ozimmu_status_t ozimmu_destroy(ozimmu_handle_t h) {
    if (!h) return OZIMMU_SUCCESS;
    if (h->auto_dev) cudaFree(h->auto_dev);
    if (h->auto_bbuf) cudaFree(h->auto_bbuf);
    if (h->aux) {
        cudaStreamSynchronize(h->aux);
        cudaStreamDestroy(h->aux);
        cudaEventDestroy(h->ev_fork);
        cudaEventDestroy(h->ev_join);
    }
    if (h->events) {
        cudaStreamSynchronize(h->stream);
        for (int i = 0; i < kPhases * h->timing_cap; ++i) cudaEventDestroy(h->events[i]);
        free(h->events);
    }
    if (h->own_ws) {
        cudaStreamSynchronize(h->stream);
        cudaFree(h->own_ws);
    }
    if (h->host_buf) {
        cudaDeviceSynchronize();
        cudaFree(h->host_buf);
    }
    if (h->h2d) cudaStreamDestroy(h->h2d);
    if (h->d2h) cudaStreamDestroy(h->d2h);
    if (h->comm) {
        cudaStreamSynchronize(h->comm);
        cudaStreamDestroy(h->comm);
    }
    if (h->dist_buf) {
        cudaDeviceSynchronize();
        cudaFree(h->dist_buf);
    }
    delete h;
    return OZIMMU_SUCCESS;
}

ozimmu_status_t ozimmu_set_stream(ozimmu_handle_t h, void *stream) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    h->stream = static_cast<cudaStream_t>(stream);
    return OZIMMU_SUCCESS;
}

ozimmu_status_t ozimmu_set_max_sms(ozimmu_handle_t h, int max_sms) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (max_sms < 0) return OZIMMU_ERR_INVALID_VALUE;
    h->gemm_sms = max_sms;
    return OZIMMU_SUCCESS;
}

size_t ozimmu_workspace_bytes(ozimmu_op_t transA, ozimmu_op_t transB, int64_t m, int64_t n,
                              int64_t k, int num_slices) {
    if (!valid_op(transA) || !valid_op(transB) || m < 0 || n < 0 || k < 1 || num_slices < 1 ||
        num_slices > OZIMMU_MAX_SLICES || k > OZIMMU_MAX_K)
        return 0;
    const int w = slice_width(k);
    const int64_t k_pad = round_up(k, 16);
    GemmPlan gp;
    if (!plan_gemm(num_slices, w, m > 0 ? m : 1, n > 0 ? n : 1, k_pad, 148, &gp)) return 0;
    // bound over every SM cap (the tile width can change with the cap) and devices <= 148 SMs
    return layout(m, n, k_pad, num_slices, chunk_scratch_bound(gp, num_slices, 148)).total;
}

ozimmu_status_t ozimmu_set_workspace(ozimmu_handle_t h, void *dptr, size_t bytes) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (dptr && (reinterpret_cast<uintptr_t>(dptr) % kAlign) != 0) return OZIMMU_ERR_INVALID_VALUE;
    h->user_ws = dptr;
    h->user_ws_bytes = dptr ? bytes : 0;
    return OZIMMU_SUCCESS;
}

ozimmu_status_t ozimmu_get_report(ozimmu_handle_t h, ozimmu_report_t *out) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (!out) return OZIMMU_ERR_INVALID_VALUE;
    *out = h->report;
    return OZIMMU_SUCCESS;
}

ozimmu_status_t ozimmu_dgemm(ozimmu_handle_t h, ozimmu_op_t transA, ozimmu_op_t transB, int64_t m,
                             int64_t n, int64_t k, const double *alpha, const double *A,
                             int64_t lda, const double *B, int64_t ldb, const double *beta,
                             double *C, int64_t ldc, int num_slices) {
    ozimmu_status_t st = check_common(h, transA, m, n, k, alpha, A, lda, beta, C, ldc, num_slices);
    if (st) return st;
    if (!valid_op(transB)) return OZIMMU_ERR_INVALID_VALUE;
    const int64_t brows = transB == OZIMMU_OP_N ? k : n;
    if (ldb < (brows > 1 ? brows : 1)) return OZIMMU_ERR_INVALID_VALUE;
    if (n > 0 && k > 0 && m > 0 && *alpha != 0.0 && !B) return OZIMMU_ERR_INVALID_VALUE;
    if (m == 0 || n == 0) {
        fill_report(h, 0, 0, m, n, k, nullptr, 0, 0);
        return OZIMMU_SUCCESS;
    }
    if (cudaSetDevice(h->device) != cudaSuccess) return OZIMMU_ERR_CUDA;
    if (*alpha == 0.0 || k == 0) return scale_only(h, m, n, *beta, C, ldc);
    int auto_launches = 0;
    const bool was_auto = num_slices == 0;
    if (was_auto) {  // INT8-AUTO
        ozimmu_status_t st2 = auto_select(h, transA, transB, m, n, k, A, lda, B, ldb, &num_slices,
                                          &auto_launches);
        if (st2) return st2;
    }
    ozimmu_status_t r = gemm_core(h, transA, m, n, k, *alpha, A, lda, nullptr, transB, B, ldb,
                                  *beta, C, ldc, num_slices);
    h->report.launches += auto_launches;
    if (was_auto) note_auto(h);
    return r;
}

size_t ozimmu_b_slices_bytes(int64_t n, int64_t k, int num_slices) {
    if (n < 0 || k < 1 || num_slices < 1 || num_slices > OZIMMU_MAX_SLICES) return 0;
    return b_buf_bytes(n, round_up(k, 16), num_slices);
}

ozimmu_status_t ozimmu_slice_b(ozimmu_handle_t h, ozimmu_op_t transB, int64_t k, int64_t n,
                               const double *B, int64_t ldb, int num_slices, void *b_slices) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (!valid_op(transB) || k < 1 || n < 0) return OZIMMU_ERR_INVALID_VALUE;
    if (num_slices == 0) return OZIMMU_ERR_UNSUPPORTED;
    if (num_slices < 0 || num_slices > OZIMMU_MAX_SLICES) return OZIMMU_ERR_INVALID_VALUE;
    if (k > OZIMMU_MAX_K) return OZIMMU_ERR_UNSUPPORTED;
    const int64_t brows = transB == OZIMMU_OP_N ? k : n;
    if (ldb < (brows > 1 ? brows : 1)) return OZIMMU_ERR_INVALID_VALUE;
    if (n == 0) return OZIMMU_SUCCESS;
    if (!B || !b_slices) return OZIMMU_ERR_INVALID_VALUE;
    if (reinterpret_cast<uintptr_t>(b_slices) % kAlign) return OZIMMU_ERR_INVALID_VALUE;
    if (cudaSetDevice(h->device) != cudaSuccess) return OZIMMU_ERR_CUDA;
    const int64_t k_pad = round_up(k, 16);
    void *ws = nullptr;
    ozimmu_status_t st = get_ws(h, align_up(sizeof(int32_t) * (size_t)n), &ws);
    if (st) return st;
    int launches = 0;
    cudaError_t e = slice_b(h, transB, k, n, k_pad, B, ldb, num_slices, slice_width(k),
                            static_cast<uint8_t *>(b_slices), static_cast<int32_t *>(ws), &launches);
    if (e != cudaSuccess) return cuda_status(e);
    fill_report(h, num_slices, slice_width(k), 0, n, k, nullptr, launches,
                (int64_t)num_slices * n * k_pad + 4 * n);
    return OZIMMU_SUCCESS;
}

ozimmu_status_t ozimmu_dgemm_presliced_b(ozimmu_handle_t h, ozimmu_op_t transA, int64_t m,
                                         int64_t n, int64_t k, const double *alpha,
                                         const double *A, int64_t lda, const void *b_slices,
                                         const double *beta, double *C, int64_t ldc,
                                         int num_slices) {
    ozimmu_status_t st = check_common(h, transA, m, n, k, alpha, A, lda, beta, C, ldc, num_slices);
    if (st) return st;
    if (m == 0 || n == 0) {
        fill_report(h, 0, 0, m, n, k, nullptr, 0, 0);
        return OZIMMU_SUCCESS;
    }
    if (cudaSetDevice(h->device) != cudaSuccess) return OZIMMU_ERR_CUDA;
    if (*alpha == 0.0 || k == 0) return scale_only(h, m, n, *beta, C, ldc);
    if (!b_slices || reinterpret_cast<uintptr_t>(b_slices) % kAlign) return OZIMMU_ERR_INVALID_VALUE;
    return gemm_core(h, transA, m, n, k, *alpha, A, lda, static_cast<const uint8_t *>(b_slices),
                     OZIMMU_OP_N, nullptr, 0, *beta, C, ldc, num_slices);
}

ozimmu_status_t ozimmu_debug_auto_rho(ozimmu_handle_t h, ozimmu_op_t op, int is_rows,
                                      int64_t rows, int64_t kdim, const double *M, int64_t ld,
                                      int w, int s_max, double *rho_out) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (!valid_op(op) || rows < 0 || kdim < 1 || w < 5 || w > 7 || s_max < 1 ||
        s_max > kAutoNS - 1 || !rho_out)
        return OZIMMU_ERR_INVALID_VALUE;
    if (kdim > OZIMMU_MAX_K) return OZIMMU_ERR_UNSUPPORTED;
    for (int t = 0; t <= s_max; ++t) rho_out[t] = 0.0;
    if (rows == 0) return OZIMMU_SUCCESS;
    if (!M) return OZIMMU_ERR_INVALID_VALUE;
    const bool contig = is_rows ? (op != OZIMMU_OP_N) : (op == OZIMMU_OP_N);
    const int64_t min_ld = contig ? kdim : rows;
    if (ld < (min_ld > 1 ? min_ld : 1)) return OZIMMU_ERR_INVALID_VALUE;
    if (cudaSetDevice(h->device) != cudaSuccess) return OZIMMU_ERR_CUDA;
    if (!h->auto_dev &&
        cudaMalloc(&h->auto_dev, 2 * kAutoNS * sizeof(unsigned long long)) != cudaSuccess) {
        cudaGetLastError();
        return OZIMMU_ERR_WORKSPACE;
    }
    void *ws = nullptr;
    ozimmu_status_t st = get_ws(h, align_up(trunc_residual_scratch(rows, s_max)), &ws);
    if (st) return st;
    int launches = 0;
    cudaError_t e = cudaMemsetAsync(h->auto_dev, 0, kAutoNS * sizeof(unsigned long long), h->stream);
    if (e == cudaSuccess)
        e = launch_trunc_residual(M, ld, contig, rows, kdim, w, s_max, h->auto_dev, ws,
                                  h->num_sms, h->stream, &launches);
    unsigned long long bits[kAutoNS];
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(bits, h->auto_dev, sizeof(bits), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_status(e);
    for (int t = 0; t <= s_max; ++t) {
        double d;
        memcpy(&d, &bits[t], sizeof(d));
        rho_out[t] = d;
    }
    return OZIMMU_SUCCESS;
}

ozimmu_status_t ozimmu_debug_split(ozimmu_handle_t h, ozimmu_op_t op, int is_rows, int64_t rows,
                                   int64_t kdim, const double *M, int64_t ld, int num_slices,
                                   int8_t *planes_out, int32_t *exps_out) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (!valid_op(op) || rows < 0 || kdim < 1 || num_slices < 1 ||
        num_slices > OZIMMU_MAX_SLICES)
        return OZIMMU_ERR_INVALID_VALUE;
    if (kdim > OZIMMU_MAX_K) return OZIMMU_ERR_UNSUPPORTED;
    if (rows == 0) return OZIMMU_SUCCESS;
    if (!M || !planes_out || !exps_out) return OZIMMU_ERR_INVALID_VALUE;
    // vector r element l: A operand (is_rows): op(M)(r,l); B operand: op(M)(l,r)
    const bool contig = is_rows ? (op != OZIMMU_OP_N) : (op == OZIMMU_OP_N);
    const int64_t min_ld = contig ? kdim : rows;
    if (ld < (min_ld > 1 ? min_ld : 1)) return OZIMMU_ERR_INVALID_VALUE;
    if (cudaSetDevice(h->device) != cudaSuccess) return OZIMMU_ERR_CUDA;
    const int w = slice_width(kdim);
    const int64_t k_pad = round_up(kdim, 16);
    const size_t pbytes = align_up((size_t)num_slices * rows * k_pad);
    void *ws = nullptr;
    ozimmu_status_t st = get_ws(h, pbytes + align_up(split_scratch_bytes(rows)), &ws);
    if (st) return st;
    int8_t *planes = static_cast<int8_t *>(ws);
    int32_t *keys = reinterpret_cast<int32_t *>(static_cast<uint8_t *>(ws) + pbytes);
    int launches = 0;
    cudaError_t e = launch_split(M, ld, contig, rows, kdim, k_pad, num_slices, w, false, planes,
                                 rows * k_pad, exps_out, keys, h->num_sms, h->stream, &launches);
    if (e != cudaSuccess) return cuda_status(e);
    // repack [s][rows][k_pad] -> [s][rows][kdim]
    e = cudaMemcpy2DAsync(planes_out, (size_t)kdim, planes, (size_t)k_pad, (size_t)kdim,
                          (size_t)num_slices * rows, cudaMemcpyDeviceToDevice, h->stream);
    if (e != cudaSuccess) return cuda_status(e);
    fill_report(h, num_slices, w, rows, 0, kdim, nullptr, launches, (int64_t)pbytes);
    return OZIMMU_SUCCESS;
}

ozimmu_status_t ozimmu_debug_level_sums(ozimmu_handle_t h, ozimmu_op_t transA,
                                        ozimmu_op_t transB, int64_t m, int64_t n, int64_t k,
                                        const double *A, int64_t lda, const double *B,
                                        int64_t ldb, int num_slices, int64_t *Lg_out) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (!valid_op(transA) || !valid_op(transB) || m < 1 || n < 1 || k < 1 || !A || !B || !Lg_out)
        return OZIMMU_ERR_INVALID_VALUE;
    if (lda < (transA == OZIMMU_OP_N ? m : k) || ldb < (transB == OZIMMU_OP_N ? k : n))
        return OZIMMU_ERR_INVALID_VALUE;
    if (num_slices < 1 || num_slices > OZIMMU_MAX_SLICES) return OZIMMU_ERR_INVALID_VALUE;
    if (k > OZIMMU_MAX_K) return OZIMMU_ERR_UNSUPPORTED;
    ozimmu_status_t st;
    if (cudaSetDevice(h->device) != cudaSuccess) return OZIMMU_ERR_CUDA;
    const int s = num_slices;
    const int w = slice_width(k);
    const int64_t k_pad = round_up(k, 16);
    GemmPlan gp;
    if (!plan_gemm(s, w, m, n, k_pad, gemm_sms(h), &gp)) return OZIMMU_ERR_UNSUPPORTED;
    const Layout L = layout(m, n, k_pad, s, chunk_scratch_bytes(gp, s));
    void *ws = nullptr;
    if ((st = get_ws(h, L.total, &ws))) return st;
    uint8_t *base = static_cast<uint8_t *>(ws);
    int launches = 0;
    int32_t *keys = reinterpret_cast<int32_t *>(base + L.keys);
    cudaError_t e = slice_b(h, transB, k, n, k_pad, B, ldb, s, w, base + L.b_buf, keys, &launches);
    if (e == cudaSuccess)
        e = slice_a(h, transA, m, k, k_pad, A, lda, s, w, reinterpret_cast<int8_t *>(base + L.a_planes),
                    reinterpret_cast<int32_t *>(base + L.a_exp), keys, &launches);
    if (e != cudaSuccess) return cuda_status(e);
    GemmArgs ga{};
    ga.a_planes = reinterpret_cast<const int8_t *>(base + L.a_planes);
    ga.b_planes = reinterpret_cast<const int8_t *>(base + L.b_buf);
    ga.m = m;
    ga.n = n;
    ga.k_pad = k_pad;
    ga.s = s;
    ga.w = w;
    ga.out = Lg_out;
    ga.chunk_scratch = reinterpret_cast<int64_t *>(base + L.scratch);
    ga.wave_counter = reinterpret_cast<unsigned int *>(base + L.sync);
    e = launch_gemm(ga, gp, EPI_LEVELS_I64, h->stream, &launches);
    if (e != cudaSuccess) return cuda_status(e);
    fill_report(h, s, w, m, n, k, &gp, launches, 0);
    return OZIMMU_SUCCESS;
}

ozimmu_status_t ozimmu_debug_pair(ozimmu_handle_t h, const int8_t *Ai, const int8_t *Bj, int64_t m,
                                  int64_t n, int64_t k, int32_t *P_out) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (m < 1 || n < 1 || k < 1 || !Ai || !Bj || !P_out) return OZIMMU_ERR_INVALID_VALUE;
    if (k > 133144) return OZIMMU_ERR_UNSUPPORTED;
    if (cudaSetDevice(h->device) != cudaSuccess) return OZIMMU_ERR_CUDA;
    const int64_t k_pad = round_up(k, 16);
    GemmPlan gp;
    if (!plan_gemm(1, 7, m, n, k_pad, gemm_sms(h), &gp)) return OZIMMU_ERR_UNSUPPORTED;
    gp.chunk_blocks = gp.num_k_blocks;  // caller guarantees the INT32 budget
    gp.k_chunks = 1;
    gp.T = 1;
    gp.G = 1;
    const size_t abytes = align_up((size_t)m * k_pad), bbytes = align_up((size_t)n * k_pad);
    void *ws = nullptr;
    ozimmu_status_t st = get_ws(h, abytes + bbytes, &ws);
    if (st) return st;
    int8_t *a = static_cast<int8_t *>(ws);
    int8_t *b = a + abytes;
    cudaError_t e = cudaMemsetAsync(ws, 0, abytes + bbytes, h->stream);
    if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(a, k_pad, Ai, k, k, m, cudaMemcpyDeviceToDevice, h->stream);
    if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(b, k_pad, Bj, k, k, n, cudaMemcpyDeviceToDevice, h->stream);
    if (e != cudaSuccess) return cuda_status(e);
    GemmArgs ga{};
    ga.a_planes = a;
    ga.b_planes = b;
    ga.m = m;
    ga.n = n;
    ga.k_pad = k_pad;
    ga.s = 1;
    ga.w = 7;
    ga.out = P_out;
    int launches = 0;
    e = launch_gemm(ga, gp, EPI_PAIR_I32, h->stream, &launches);
    if (e != cudaSuccess) return cuda_status(e);
    fill_report(h, 1, 7, m, n, k, &gp, launches, 0);
    return OZIMMU_SUCCESS;
}


// ---- f1: complex GEMM (reading A16: real embedding with interleaved K) -------------------

static size_t zgemm_ws(int64_t m, int64_t n, int64_t k, int s, int num_sms, GemmPlan *gp_out,
                       Layout *L_out, bool bound = false) {
    const int64_t K2 = 2 * k;
    const int w = slice_width(K2);
    const int64_t k_pad = round_up(K2, 16);
    GemmPlan gp;
    if (!plan_gemm(s, w, m > 0 ? m : 1, 2 * (n > 0 ? n : 1), k_pad, num_sms, &gp)) return 0;
    Layout L = layout(m, 2 * n, k_pad, s,
                      bound ? chunk_scratch_bound(gp, s, 148) : chunk_scratch_bytes(gp, s));
    if (gp_out) *gp_out = gp;
    if (L_out) *L_out = L;
    return L.total;
}

// ZGEMM after validation / AUTO (reading A16).  amap / bmap: stacked batches of rows of
// op(A) / columns of op(B) (strides in complex elements); crow / ccol: C maps (complex).
static ozimmu_status_t zgemm_core(ozimmu_handle_t h, ozimmu_op_t transA, ozimmu_op_t transB,
                                  int64_t m, int64_t n, int64_t k, const double *alpha,
                                  const double *A, int64_t lda, const double *B, int64_t ldb,
                                  const double *beta, double *C, int64_t ldc, int s,
                                  BatchMap amap = BatchMap(), BatchMap bmap = BatchMap(),
                                  BatchMap crow = BatchMap(), BatchMap ccol = BatchMap()) {
    ozimmu_status_t st;
    const int64_t K2 = 2 * k;
    const int w = slice_width(K2);
    const int64_t k_pad = round_up(K2, 16);
    GemmPlan gp;
    Layout L;
    if (!zgemm_ws(m, n, k, s, gemm_sms(h), &gp, &L)) return OZIMMU_ERR_UNSUPPORTED;
    void *ws = nullptr;
    if ((st = get_ws(h, L.total, &ws))) return st;
    uint8_t *base = static_cast<uint8_t *>(ws);
    int8_t *a_planes = reinterpret_cast<int8_t *>(base + L.a_planes);
    int32_t *EA = reinterpret_cast<int32_t *>(base + L.a_exp);
    uint8_t *bbuf = base + L.b_buf;
    int8_t *b_planes = reinterpret_cast<int8_t *>(bbuf);
    int32_t *EB = reinterpret_cast<int32_t *>(bbuf + b_buf_planes_bytes(2 * n, k_pad, s));
    int32_t *keys = reinterpret_cast<int32_t *>(base + L.keys);
    int launches = 0;
    mark(h, PH_START);
    // columns of op(B): contiguous (re, im) pairs iff transB == N -> 2n plane rows
    const bool bcontig = transB == OZIMMU_OP_N;
    // batch strides in the units of the vector ld: doubles (contiguous) or complex (strided)
    BatchMap bm = bmap;
    if (bcontig) bm.stride *= 2;
    cudaError_t e = launch_split(B, bcontig ? 2 * ldb : ldb, bcontig, n, K2, k_pad, s, w,
                                 /*reverse=*/true, b_planes, 2 * n * k_pad, EB, keys, h->num_sms,
                                 h->stream, &launches, /*cpx=*/2, transB == OZIMMU_OP_C, bm);
    if (e != cudaSuccess) return cuda_status(e);
    mark(h, PH_B);
    const bool acontig = transA != OZIMMU_OP_N;
    BatchMap am = amap;
    if (acontig) am.stride *= 2;
    e = launch_split(A, acontig ? 2 * lda : lda, acontig, m, K2, k_pad, s, w, /*reverse=*/false,
                     a_planes, m * k_pad, EA, keys, h->num_sms, h->stream, &launches, /*cpx=*/1,
                     transA == OZIMMU_OP_C, am);
    if (e != cudaSuccess) return cuda_status(e);
    mark(h, PH_A);
    mark(h, PH_GEMM0);
    GemmArgs ga{};
    ga.a_planes = a_planes;
    ga.b_planes = b_planes;
    ga.EA = EA;
    ga.EB = EB;
    ga.m = m;
    ga.n = 2 * n;
    ga.k_pad = k_pad;
    ga.s = s;
    ga.w = w;
    ga.alpha = alpha[0];
    ga.alpha_im = alpha[1];
    ga.beta = beta[0];
    ga.beta_im = beta[1];
    ga.C = C;
    ga.ldc = ldc;
    ga.c_rows = crow;
    // GEMM columns 2j / 2j+1 are complex column j: the column map acts on j (store_row)
    ga.c_cols = ccol;
    ga.chunk_scratch = reinterpret_cast<int64_t *>(base + L.scratch);
    static const bool no_sync = getenv("OZIMMU_NO_WAVE_SYNC") != nullptr;
    ga.wave_counter = no_sync ? nullptr : reinterpret_cast<unsigned int *>(base + L.sync);
    e = launch_gemm(ga, gp, EPI_ZGEMM, h->stream, &launches);
    if (e != cudaSuccess) return cuda_status(e);
    mark(h, PH_GEMM1);
    mark_done(h);
    fill_report(h, s, w, m, n, K2, &gp, launches,
                (int64_t)s * (m + 2 * n) * k_pad + 4 * (m + 2 * n));
    h->report.int8_macs = (int64_t)s * (s + 1) / 2 * m * (2 * n) * K2;
    return OZIMMU_SUCCESS;
}

size_t ozimmu_zgemm_workspace_bytes(ozimmu_op_t transA, ozimmu_op_t transB, int64_t m, int64_t n,
                                    int64_t k, int num_slices) {
    if (!valid_op(transA) || !valid_op(transB) || m < 0 || n < 0 || k < 1 || num_slices < 1 ||
        num_slices > OZIMMU_MAX_SLICES || 2 * k > OZIMMU_MAX_K)
        return 0;
    return zgemm_ws(m, n, k, num_slices, 148, nullptr, nullptr, /*bound=*/true);
}

ozimmu_status_t ozimmu_zgemm(ozimmu_handle_t h, ozimmu_op_t transA, ozimmu_op_t transB, int64_t m,
                             int64_t n, int64_t k, const double *alpha, const double *A,
                             int64_t lda, const double *B, int64_t ldb, const double *beta,
                             double *C, int64_t ldc, int num_slices) {
    ozimmu_status_t st = check_common(h, transA, m, n, k, alpha, A, lda, beta, C, ldc, num_slices);
    if (st) return st;
    if (!valid_op(transB)) return OZIMMU_ERR_INVALID_VALUE;
    const int64_t brows = transB == OZIMMU_OP_N ? k : n;
    if (ldb < (brows > 1 ? brows : 1)) return OZIMMU_ERR_INVALID_VALUE;
    const bool alpha0 = alpha[0] == 0.0 && alpha[1] == 0.0;
    if (n > 0 && k > 0 && m > 0 && !alpha0 && !B) return OZIMMU_ERR_INVALID_VALUE;
    if (2 * k > OZIMMU_MAX_K) return OZIMMU_ERR_UNSUPPORTED;
    if (m == 0 || n == 0) {
        fill_report(h, 0, 0, m, n, k, nullptr, 0, 0);
        return OZIMMU_SUCCESS;
    }
    if (cudaSetDevice(h->device) != cudaSuccess) return OZIMMU_ERR_CUDA;
    if (alpha0 || k == 0) {
        int launches = 0;
        if (!(beta[0] == 1.0 && beta[1] == 0.0)) {
            int64_t blocks = ceil_div(m * n, 256);
            if (blocks > 8 * (int64_t)h->num_sms) blocks = 8 * (int64_t)h->num_sms;
            k_scale_z<<<(unsigned)blocks, 256, 0, h->stream>>>(reinterpret_cast<double2 *>(C), ldc,
                                                               m, n, beta[0], beta[1]);
            ++launches;
            if (cudaGetLastError() != cudaSuccess) return OZIMMU_ERR_CUDA;
        }
        fill_report(h, 0, 0, m, n, 0, nullptr, launches, 0);
        return OZIMMU_SUCCESS;
    }
    int auto_launches = 0;
    const bool was_auto = num_slices == 0;
    if (was_auto) {  // INT8-AUTO on the embedded (reading A16) operands
        st = auto_select(h, transA, transB, m, n, k, A, lda, B, ldb, &num_slices, &auto_launches,
                         /*cpx=*/true);
        if (st) return st;
    }
    st = zgemm_core(h, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, num_slices);
    h->report.launches += auto_launches;
    if (was_auto) note_auto(h);
    return st;
}


// ---- f3: strided-batched forms (cuBLAS-style), quantum-circuit gate application -----------

// A batch with a shared operand (strideB == 0 or strideA == 0) and a fixed s runs as ONE
// fused GEMM: the rows of the op(A_b) (shared B) or the columns of the op(B_b) (shared A) are
// stacked through a BatchMap in the slicing kernels, the shared operand is sliced once, and
// the epilogue maps stacked rows / columns back to C_b.  Every element sees the operation
// sequence of the per-item call, so each C_b is bitwise what ozimmu_dgemm returns for it.
// Other batches (independent A_b and B_b, or INT8-AUTO, where s is chosen per item) loop.
static bool fuse_batch(int64_t m, int64_t n, int64_t k, int64_t strideA, int64_t strideB,
                       int64_t batch, int num_slices, bool alpha0) {
    static const bool off = getenv("OZIMMU_NO_BATCH_FUSE") != nullptr;  // experiments
    return !off && batch > 1 && num_slices > 0 && (strideA == 0 || strideB == 0) && m > 0 &&
           n > 0 && k > 0 && !alpha0;
}

ozimmu_status_t ozimmu_dgemm_strided_batched(ozimmu_handle_t h, ozimmu_op_t transA,
                                             ozimmu_op_t transB, int64_t m, int64_t n, int64_t k,
                                             const double *alpha, const double *A, int64_t lda,
                                             int64_t strideA, const double *B, int64_t ldb,
                                             int64_t strideB, const double *beta, double *C,
                                             int64_t ldc, int64_t strideC, int64_t batch,
                                             int num_slices) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (batch < 0 || strideA < 0 || strideB < 0 || strideC < 0) return OZIMMU_ERR_INVALID_VALUE;
    if (batch == 0) return OZIMMU_SUCCESS;
    if (alpha && fuse_batch(m, n, k, strideA, strideB, batch, num_slices, *alpha == 0.0)) {
        ozimmu_status_t st = check_common(h, transA, m, n, k, alpha, A, lda, beta, C, ldc,
                                          num_slices);
        if (st) return st;
        const int64_t brows = transB == OZIMMU_OP_N ? k : n;
        if (!valid_op(transB) || !B || ldb < (brows > 1 ? brows : 1)) return OZIMMU_ERR_INVALID_VALUE;
        if (cudaSetDevice(h->device) != cudaSuccess) return OZIMMU_ERR_CUDA;
        if (strideB == 0)  // shared op(B): stack the rows of op(A_b) and of C_b
            return gemm_core(h, transA, batch * m, n, k, *alpha, A, lda, nullptr, transB, B, ldb,
                             *beta, C, ldc, num_slices, BatchMap{m, strideA}, BatchMap(),
                             BatchMap{m, strideC}, BatchMap());
        // shared op(A): stack the columns of op(B_b) and of C_b
        return gemm_core(h, transA, m, batch * n, k, *alpha, A, lda, nullptr, transB, B, ldb,
                         *beta, C, ldc, num_slices, BatchMap(), BatchMap{n, strideB}, BatchMap(),
                         BatchMap{n, strideC});
    }
    int launches = 0;
    for (int64_t b = 0; b < batch; ++b) {
        ozimmu_status_t st = ozimmu_dgemm(h, transA, transB, m, n, k, alpha, A + b * strideA, lda,
                                          B + b * strideB, ldb, beta, C + b * strideC, ldc,
                                          num_slices);
        if (st) return st;
        launches += h->report.launches;
    }
    h->report.launches = launches;
    return OZIMMU_SUCCESS;
}

ozimmu_status_t ozimmu_zgemm_strided_batched(ozimmu_handle_t h, ozimmu_op_t transA,
                                             ozimmu_op_t transB, int64_t m, int64_t n, int64_t k,
                                             const double *alpha, const double *A, int64_t lda,
                                             int64_t strideA, const double *B, int64_t ldb,
                                             int64_t strideB, const double *beta, double *C,
                                             int64_t ldc, int64_t strideC, int64_t batch,
                                             int num_slices) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (batch < 0 || strideA < 0 || strideB < 0 || strideC < 0) return OZIMMU_ERR_INVALID_VALUE;
    if (batch == 0) return OZIMMU_SUCCESS;
    if (alpha && fuse_batch(m, n, k, strideA, strideB, batch, num_slices,
                            alpha[0] == 0.0 && alpha[1] == 0.0)) {
        ozimmu_status_t st = check_common(h, transA, m, n, k, alpha, A, lda, beta, C, ldc,
                                          num_slices);
        if (st) return st;
        const int64_t brows = transB == OZIMMU_OP_N ? k : n;
        if (!valid_op(transB) || !B || ldb < (brows > 1 ? brows : 1)) return OZIMMU_ERR_INVALID_VALUE;
        if (2 * k > OZIMMU_MAX_K) return OZIMMU_ERR_UNSUPPORTED;
        if (cudaSetDevice(h->device) != cudaSuccess) return OZIMMU_ERR_CUDA;
        if (strideB == 0)
            return zgemm_core(h, transA, transB, batch * m, n, k, alpha, A, lda, B, ldb, beta, C,
                              ldc, num_slices, BatchMap{m, strideA}, BatchMap(),
                              BatchMap{m, strideC}, BatchMap());
        return zgemm_core(h, transA, transB, m, batch * n, k, alpha, A, lda, B, ldb, beta, C, ldc,
                          num_slices, BatchMap(), BatchMap{n, strideB}, BatchMap(),
                          BatchMap{n, strideC});
    }
    int launches = 0;
    for (int64_t b = 0; b < batch; ++b) {  // strides in complex elements
        ozimmu_status_t st = ozimmu_zgemm(h, transA, transB, m, n, k, alpha, A + 2 * b * strideA,
                                          lda, B + 2 * b * strideB, ldb, beta,
                                          C + 2 * b * strideC, ldc, num_slices);
        if (st) return st;
        launches += h->report.launches;
    }
    h->report.launches = launches;
    return OZIMMU_SUCCESS;
}

}  // extern "C"


