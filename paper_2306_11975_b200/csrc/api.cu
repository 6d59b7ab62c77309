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

using namespace ozimmu;

struct ozimmu_ctx {
    int device = 0;
    int num_sms = 148;
    int gemm_sms = 0;  // ozimmu_set_max_sms: cap on the fused GEMM's persistent grid (0 = all)
    cudaStream_t stream = nullptr;
    void *user_ws = nullptr;
    size_t user_ws_bytes = 0;
    void *own_ws = nullptr;
    size_t own_ws_bytes = 0;
    ozimmu_report_t report{};
    // phase timing ring (ozimmu_timing_enable / _read)
    cudaEvent_t *events = nullptr;
    int timing_cap = 0;
    int timing_count = 0;
    // INT8-AUTO (num_slices = 0): threshold T on the mean mantissa loss, s cap
    double auto_T = 0.0;
    int auto_smax = 20;
    int auto_last_s = 0;
    unsigned long long *auto_dev = nullptr;  // device [2][33] loss sums
    // host-buffer entry point (ozimmu_dgemm_host): copy streams + device staging buffer
    cudaStream_t h2d = nullptr, d2h = nullptr;
    void *host_buf = nullptr;
    size_t host_buf_bytes = 0;
    void *auto_bbuf = nullptr;  // B-slice buffer of the INT8-AUTO host path (grown, kept)
    size_t auto_bbuf_bytes = 0;
    // second stream for slicing op(B) concurrently with op(A) (fork / join by events)
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

namespace {

constexpr size_t kAlign = 256;

// SMs the fused GEMM may occupy (ozimmu_set_max_sms)
inline int gemm_sms(ozimmu_handle_t h) {
    return (h->gemm_sms > 0 && h->gemm_sms < h->num_sms) ? h->gemm_sms : h->num_sms;
}

inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Layout {  // workspace carve-up for one dgemm call
    size_t a_planes, a_exp, b_buf, keys, keys_b, sync, scratch, total;
};

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
    off += align_up(sizeof(int32_t) * (size_t)(m > n ? m : n));
    L.keys_b = off;  // B's exponent-scan scratch (B is sliced concurrently with A)
    off += align_up(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
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

// Record phase event `ph` (0..3) of the current call if timing is on.
inline void mark(ozimmu_handle_t h, int ph) {
    if (h->timing_cap && h->timing_count < h->timing_cap)
        cudaEventRecord(h->events[4 * h->timing_count + ph], h->stream);
}
inline void mark_done(ozimmu_handle_t h) {
    if (h->timing_cap && h->timing_count < h->timing_cap) ++h->timing_count;
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
                    int32_t *keys, int *launches, BatchMap vm = BatchMap()) {
    const bool contig = transA != OZIMMU_OP_N;
    return launch_split(A, lda, contig, m, k, k_pad, s, w, /*reverse=*/false, planes,
                        (int64_t)m * k_pad, E, keys, h->num_sms, h->stream, launches, 0, 0, vm);
}

// Slice op(B) into a B-slice buffer: columns of op(B) are contiguous along k iff transB == N.
cudaError_t slice_b(ozimmu_handle_t h, ozimmu_op_t transB, int64_t k, int64_t n, int64_t k_pad,
                    const double *B, int64_t ldb, int s, int w, uint8_t *bbuf, int32_t *keys,
                    int *launches, BatchMap vm = BatchMap(), cudaStream_t st = nullptr) {
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

// f2 INT8-AUTO (reading A17): exact per-s mantissa-loss sums of the rows of
// op(A) and the columns of op(B) on the device, one D2H read (the call synchronises the
// stream), then the smallest s <= s_max whose mean loss is <= T for both operands.
ozimmu_status_t auto_select(ozimmu_handle_t h, ozimmu_op_t transA, ozimmu_op_t transB, int64_t m,
                            int64_t n, int64_t k, const double *A, int64_t lda, const double *B,
                            int64_t ldb, int *s_out, int *launches, bool cpx = false) {
    constexpr int NS = 33;
    const int s_max = h->auto_smax;
    const int w = slice_width(cpx ? 2 * k : k);
    if (!h->auto_dev && cudaMalloc(&h->auto_dev, 2 * NS * sizeof(unsigned long long)) != cudaSuccess) {
        cudaGetLastError();
        return OZIMMU_ERR_WORKSPACE;
    }
    void *ws = nullptr;
    ozimmu_status_t st = get_ws(h, align_up(sizeof(int32_t) * (size_t)(m > n ? m : n)), &ws);
    if (st) return st;
    int32_t *keys = static_cast<int32_t *>(ws);
    cudaError_t e = cudaMemsetAsync(h->auto_dev, 0, 2 * NS * sizeof(unsigned long long), h->stream);
    const bool ac = transA != OZIMMU_OP_N, bc = transB == OZIMMU_OP_N;
    // complex: contiguous vectors are 2k doubles (ld in doubles), strided ones k pairs
    if (e == cudaSuccess)
        e = launch_mantissa_loss(A, cpx && ac ? 2 * lda : lda, ac, m, cpx && ac ? 2 * k : k, w,
                                 s_max, h->auto_dev, keys, h->num_sms, h->stream, launches, cpx);
    if (e == cudaSuccess)
        e = launch_mantissa_loss(B, cpx && bc ? 2 * ldb : ldb, bc, n, cpx && bc ? 2 * k : k, w,
                                 s_max, h->auto_dev + NS, keys, h->num_sms, h->stream, launches,
                                 cpx);
    unsigned long long host[2 * NS];
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(host, h->auto_dev, sizeof(host), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_status(e);
    int chosen = s_max;
    for (int s = 1; s <= s_max; ++s) {
        const double ma = host[32] ? (double)host[s - 1] / (double)host[32] : 0.0;
        const double mb = host[NS + 32] ? (double)host[NS + s - 1] / (double)host[NS + 32] : 0.0;
        if (ma <= h->auto_T && mb <= h->auto_T) {
            chosen = s;
            break;
        }
    }
    *s_out = chosen;
    h->auto_last_s = chosen;
    return OZIMMU_SUCCESS;
}

// The fused tcgen05 GEMM + FP64 epilogue (A4 + A5) on sliced operands.  b_plane_rows: rows
// per B plane in memory (0 = n; a column chunk of a wider B-slice buffer otherwise).
cudaError_t fused_gemm(ozimmu_handle_t h, const GemmPlan &gp, int64_t m, int64_t n, int64_t k_pad,
                       int s, int w, const int8_t *a_planes, const int32_t *EA,
                       const int8_t *b_planes, const int32_t *EB, int64_t b_plane_rows,
                       double alpha, double beta, double *C, int64_t ldc, int64_t *scratch,
                       unsigned int *sync, int *launches, BatchMap crow = BatchMap(),
                       BatchMap ccol = BatchMap(), int64_t a_plane_rows = 0) {
    GemmArgs ga{};
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
    if (want_stats && !stats_buf) cudaMalloc(&stats_buf, 12 * 1024 * sizeof(long long));
    ga.stats = want_stats ? stats_buf : nullptr;
    cudaError_t e = launch_gemm(ga, gp, EPI_DGEMM, h->stream, launches);
    if (e != cudaSuccess || !ga.stats) return e;
    // development only: synchronous dump of the stall counters
    constexpr int NS = 12;
    static long long host[NS * 1024];
    cudaStreamSynchronize(h->stream);
    cudaMemcpy(host, ga.stats, sizeof(long long) * NS * gp.grid, cudaMemcpyDeviceToHost);
    double acc[NS] = {0};
    for (int c = 0; c < gp.grid; ++c)
        for (int i = 0; i < NS; ++i) acc[i] += (double)host[c * NS + i];
    const char *names[NS] = {"total", "mma_wait_b", "mma_wait_a", "mma_wait_tmem", "prod_wave",
                             "prod_wait_a", "prod_wait_b", "epi_busy", "epi_tmem", "epi_store",
                             "mma_wait_a_first_kb", "mma_wait_b_kb0"};
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
                          double *C, int64_t ldc, int s, BatchMap amap = BatchMap(),
                          BatchMap bmap = BatchMap(), BatchMap crow = BatchMap(),
                          BatchMap ccol = BatchMap()) {
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
    mark(h, 0);
    // op(B) is sliced on the handle's second stream while op(A) is sliced on its stream
    // (separate exponent-scan scratch); the GEMM waits for both.  Phase marks: 0 -> 2 is
    // the whole (overlapped) slicing.
    const bool fork = !bbuf_ext;
    if (fork) {
        uint8_t *b = base + L.b_buf;
        cudaError_t e = aux_fork(h);
        if (e == cudaSuccess)
            e = slice_b(h, transB, k, n, k_pad, B, ldb, s, w, b,
                        reinterpret_cast<int32_t *>(base + L.keys_b), &launches, bmap, h->aux);
        if (e != cudaSuccess) return cuda_status(e);
        bbuf = b;
        slice_bytes += (int64_t)s * n * k_pad + 4 * n;
    }
    mark(h, 1);
    cudaError_t e = slice_a(h, transA, m, k, k_pad, A, lda, s, w, a_planes, EA, keys, &launches,
                            amap);
    if (e == cudaSuccess && fork) e = aux_join(h);
    if (e != cudaSuccess) return cuda_status(e);
    mark(h, 2);
    e = fused_gemm(h, gp, m, n, k_pad, s, w, a_planes, EA, reinterpret_cast<const int8_t *>(bbuf),
                   reinterpret_cast<const int32_t *>(bbuf + b_buf_planes_bytes(n, k_pad, s)), 0,
                   alpha, beta, C, ldc, reinterpret_cast<int64_t *>(base + L.scratch),
                   reinterpret_cast<unsigned int *>(base + L.sync), &launches, crow, ccol);
    if (e != cudaSuccess) return cuda_status(e);
    mark(h, 3);
    mark_done(h);
    fill_report(h, s, w, m, n, k, &gp, launches, slice_bytes);
    return OZIMMU_SUCCESS;
}

}  // namespace

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
        for (int i = 0; i < 4 * h->timing_cap; ++i) cudaEventDestroy(h->events[i]);
        free(h->events);
        h->events = nullptr;
    }
    h->timing_cap = 0;
    h->timing_count = 0;
    if (max_calls == 0) return OZIMMU_SUCCESS;
    if (cudaSetDevice(h->device) != cudaSuccess) return OZIMMU_ERR_CUDA;
    h->events = static_cast<cudaEvent_t *>(calloc(4 * (size_t)max_calls, sizeof(cudaEvent_t)));
    if (!h->events) return OZIMMU_ERR_INVALID_VALUE;
    for (int i = 0; i < 4 * max_calls; ++i)
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
        cudaEvent_t *ev = h->events + 4 * c;
        float t[3] = {0, 0, 0};
        for (int p = 0; p < 3; ++p) {
            if (cudaEventSynchronize(ev[p + 1]) != cudaSuccess ||
                cudaEventElapsedTime(&t[p], ev[p], ev[p + 1]) != cudaSuccess) {
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
    h->auto_T = threshold;
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
        for (int i = 0; i < 4 * h->timing_cap; ++i) cudaEventDestroy(h->events[i]);
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
    gp.grid = gp.grid < 148 ? 148 : gp.grid;  // upper bound over devices up to 148 SMs
    return layout(m, n, k_pad, num_slices, chunk_scratch_bytes(gp, num_slices)).total;
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
    if (*alpha == 0.0 || k == 0) return scale_only(h, m, n, *beta, C, ldc);
    if (cudaSetDevice(h->device) != cudaSuccess) return OZIMMU_ERR_CUDA;
    int auto_launches = 0;
    if (num_slices == 0) {  // INT8-AUTO
        ozimmu_status_t st2 = auto_select(h, transA, transB, m, n, k, A, lda, B, ldb, &num_slices,
                                          &auto_launches);
        if (st2) return st2;
    }
    ozimmu_status_t r = gemm_core(h, transA, m, n, k, *alpha, A, lda, nullptr, transB, B, ldb,
                                  *beta, C, ldc, num_slices);
    h->report.launches += auto_launches;
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
    if (*alpha == 0.0 || k == 0) return scale_only(h, m, n, *beta, C, ldc);
    if (!b_slices || reinterpret_cast<uintptr_t>(b_slices) % kAlign) return OZIMMU_ERR_INVALID_VALUE;
    if (cudaSetDevice(h->device) != cudaSuccess) return OZIMMU_ERR_CUDA;
    return gemm_core(h, transA, m, n, k, *alpha, A, lda, static_cast<const uint8_t *>(b_slices),
                     OZIMMU_OP_N, nullptr, 0, *beta, C, ldc, num_slices);
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
    ozimmu_status_t st = get_ws(h, pbytes + align_up(4 * (size_t)rows), &ws);
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
                       Layout *L_out) {
    const int64_t K2 = 2 * k;
    const int w = slice_width(K2);
    const int64_t k_pad = round_up(K2, 16);
    GemmPlan gp;
    if (!plan_gemm(s, w, m > 0 ? m : 1, 2 * (n > 0 ? n : 1), k_pad, num_sms, &gp)) return 0;
    Layout L = layout(m, 2 * n, k_pad, s, chunk_scratch_bytes(gp, s));
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
    mark(h, 0);
    // columns of op(B): contiguous (re, im) pairs iff transB == N -> 2n plane rows
    const bool bcontig = transB == OZIMMU_OP_N;
    // batch strides in the units of the vector ld: doubles (contiguous) or complex (strided)
    BatchMap bm = bmap;
    if (bcontig) bm.stride *= 2;
    cudaError_t e = launch_split(B, bcontig ? 2 * ldb : ldb, bcontig, n, K2, k_pad, s, w,
                                 /*reverse=*/true, b_planes, 2 * n * k_pad, EB, keys, h->num_sms,
                                 h->stream, &launches, /*cpx=*/2, transB == OZIMMU_OP_C, bm);
    if (e != cudaSuccess) return cuda_status(e);
    mark(h, 1);
    const bool acontig = transA != OZIMMU_OP_N;
    BatchMap am = amap;
    if (acontig) am.stride *= 2;
    e = launch_split(A, acontig ? 2 * lda : lda, acontig, m, K2, k_pad, s, w, /*reverse=*/false,
                     a_planes, m * k_pad, EA, keys, h->num_sms, h->stream, &launches, /*cpx=*/1,
                     transA == OZIMMU_OP_C, am);
    if (e != cudaSuccess) return cuda_status(e);
    mark(h, 2);
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
    mark(h, 3);
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
    return zgemm_ws(m, n, k, num_slices, 148, nullptr, nullptr);
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
    if (num_slices == 0) {  // INT8-AUTO on the embedded (reading A16) operands
        st = auto_select(h, transA, transB, m, n, k, A, lda, B, ldb, &num_slices, &auto_launches,
                         /*cpx=*/true);
        if (st) return st;
    }
    st = zgemm_core(h, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, num_slices);
    h->report.launches += auto_launches;
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


// ---- host-buffer entry point: H2D copies, slicing, GEMM and D2H overlapped ----------------
//
// op(A) is cut into row blocks A_0..A_{P-1} and op(B) into column chunks B_0..B_{J-1}.  Copy
// order on the H2D stream: A_0, B_0..B_{J-1}, A_1, .., A_{P-1}; compute stream: slice A_0, then
// per chunk j slice B_j into the full B-slice buffer and run GEMM(A_0, B_j) (so tensor work
// starts after the first chunk, not after all of B), then per block i >= 1 slice A_i and run
// GEMM(A_i, B) on the whole B-slice buffer; the D2H stream returns C block i as soon as its
// GEMM ends.  Every element of C sees the same operation sequence as ozimmu_dgemm (rows of
// op(A) and columns of op(B) are sliced independently; the epilogue is per element), so the
// result is bitwise identical to the device-pointer call.  Staging slots are double-buffered
// with events; the call blocks until C is back in host memory.
namespace {

// Host-buffer pipeline (ozimmu_dgemm_host): op(A) in P row blocks of mb rows, op(B) in J
// column chunks of nb columns.  Device buffers: the full A planes [s][m][k_pad] + E_A, the
// full B-slice buffer, double-buffered FP64 staging for one A block / one B chunk, C (m x n,
// ld m) and the GEMM scratch.
struct HostPlan {
    int64_t mb, nb, P, J;
    std::vector<int64_t> rb, cb;  // row-block / column-chunk boundaries (P+1 / J+1 entries)
    size_t o_apl, o_bbuf, o_ast[2], o_bst[2], o_c, o_keys, o_sync, o_scratch, total;
};

bool host_plan(ozimmu_handle_t h, int64_t m, int64_t n, int64_t k, int s, HostPlan *hp) {
    const int w = slice_width(k);
    const int64_t k_pad = round_up(k, 16);
    static const int64_t env_mb = getenv("OZIMMU_HOST_MB") ? atoll(getenv("OZIMMU_HOST_MB")) : 0;
    static const int64_t env_nb = getenv("OZIMMU_HOST_NB") ? atoll(getenv("OZIMMU_HOST_NB")) : 0;
    // 16 blocks per operand: the first GEMM waits for one A block and one B chunk (~1/16 of
    // the H2D bytes); measured at 16384^3: 16 blocks 145.6 ms, 8 blocks 149.9, 4 blocks 156.7
    int64_t mb = env_mb > 0 ? env_mb : round_up(ceil_div(m, 16), 128);
    int64_t nb = env_nb > 0 ? env_nb : round_up(ceil_div(n, 16), 96);
    if (mb < 512) mb = 512;
    if (nb < 512) nb = 512;
    if (mb > m) mb = m;
    if (nb > n) nb = n;
    hp->mb = mb;
    hp->nb = nb;
    // the first and the last block are half-size: the first GEMM waits for less H2D, the
    // last region's D2H (the drain after the last GEMM) moves less
    // Past ~45 % of an operand the tensor cores are behind the copies (the computable area
    // grows as a square), so later blocks are twice as large: fewer, larger C regions and
    // fewer partial last waves (OZIMMU_HOST_GROW=0 keeps equal blocks).
    static const bool grow = !(getenv("OZIMMU_HOST_GROW") && atoi(getenv("OZIMMU_HOST_GROW")) == 0);
    auto bounds = [](int64_t total, int64_t blk, int64_t align, std::vector<int64_t> &b) {
        b.assign(1, 0);
        int64_t half = round_up(blk / 2, align);
        if (half >= blk || total <= blk) {  // no halving: equal blocks
            for (int64_t x = blk; x < total; x += blk) b.push_back(x);
            b.push_back(total);
            return;
        }
        int64_t x = half;
        b.push_back(x);
        while (total - x > blk + half) {
            const int64_t step = (grow && x >= total * 45 / 100 && total - x > 2 * blk + half)
                                     ? 2 * blk : blk;
            x += step;
            b.push_back(x);
        }
        if (total - x > half) b.push_back(total - half);
        b.push_back(total);
    };
    bounds(m, mb, 128, hp->rb);
    bounds(n, nb, 96, hp->cb);
    hp->P = (int64_t)hp->rb.size() - 1;
    hp->J = (int64_t)hp->cb.size() - 1;
    for (size_t i = 1; i < hp->rb.size(); ++i) mb = std::max(mb, hp->rb[i] - hp->rb[i - 1]);
    for (size_t i = 1; i < hp->cb.size(); ++i) nb = std::max(nb, hp->cb[i] - hp->cb[i - 1]);
    hp->mb = mb;  // largest block: staging-buffer and scratch sizes
    hp->nb = nb;
    size_t scratch = 0;
    const int64_t shapes[3][2] = {{mb, nb}, {m, nb}, {mb, n}};
    for (auto &sh : shapes) {
        GemmPlan gp;
        if (!plan_gemm(s, w, sh[0], sh[1], k_pad, gemm_sms(h), &gp)) return false;
        const size_t c = chunk_scratch_bytes(gp, s);
        if (c > scratch) scratch = c;
    }
    size_t off = 0;
    hp->o_apl = off;
    off += align_up((size_t)s * m * k_pad) + align_up(sizeof(int32_t) * (size_t)m);
    hp->o_bbuf = off;
    off += b_buf_bytes(n, k_pad, s);
    for (int i = 0; i < 2; ++i) { hp->o_ast[i] = off; off += align_up((size_t)mb * k * sizeof(double)); }
    for (int i = 0; i < 2; ++i) { hp->o_bst[i] = off; off += align_up((size_t)k * nb * sizeof(double)); }
    hp->o_c = off;
    off += align_up((size_t)m * n * sizeof(double));
    hp->o_keys = off;
    off += align_up(sizeof(int32_t) * (size_t)(mb > nb ? mb : nb));
    hp->o_sync = off;
    off += kAlign;
    hp->o_scratch = off;
    off += align_up(scratch);
    hp->total = off;
    return true;
}

ozimmu_status_t host_buffers(ozimmu_handle_t h, size_t need) {
    if (!h->h2d && cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking) != cudaSuccess)
        return cuda_status(cudaErrorUnknown);
    if (!h->d2h && cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking) != cudaSuccess)
        return cuda_status(cudaErrorUnknown);
    if (need <= h->host_buf_bytes) return OZIMMU_SUCCESS;
    if (h->host_buf) {
        cudaDeviceSynchronize();
        cudaFree(h->host_buf);
        h->host_buf = nullptr;
        h->host_buf_bytes = 0;
    }
    if (cudaMalloc(&h->host_buf, need) != cudaSuccess) {
        cudaGetLastError();
        return OZIMMU_ERR_WORKSPACE;
    }
    h->host_buf_bytes = need;
    return OZIMMU_SUCCESS;
}

// 2-D column-major copy: `cols` columns of `rows` doubles, leading dimensions in doubles.
inline cudaError_t copy2d(double *dst, int64_t ldd, const double *src, int64_t lds, int64_t rows,
                          int64_t cols, cudaMemcpyKind kind, cudaStream_t st) {
    if (rows <= 0 || cols <= 0) return cudaSuccess;
    return cudaMemcpy2DAsync(dst, ldd * sizeof(double), src, lds * sizeof(double),
                             rows * sizeof(double), cols, kind, st);
}

// Non-pipelined host path (INT8-AUTO needs both operands on the device before s is known;
// degenerate alpha = 0 / k = 0 calls): copy in, ozimmu_dgemm, copy out.
ozimmu_status_t host_full(ozimmu_handle_t h, ozimmu_op_t transA, ozimmu_op_t transB, int64_t m,
                          int64_t n, int64_t k, const double *alpha, const double *A, int64_t lda,
                          const double *B, int64_t ldb, const double *beta, double *C,
                          int64_t ldc, int num_slices) {
    const bool use_ab = *alpha != 0.0 && k > 0;
    const int64_t ar = transA == OZIMMU_OP_N ? m : k, ac = transA == OZIMMU_OP_N ? k : m;
    const int64_t br = transB == OZIMMU_OP_N ? k : n, bc = transB == OZIMMU_OP_N ? n : k;
    const size_t sa = use_ab ? align_up(sizeof(double) * (size_t)ar * ac) : 0;
    const size_t sb = use_ab ? align_up(sizeof(double) * (size_t)br * bc) : 0;
    const size_t sc = align_up(sizeof(double) * (size_t)m * n);
    ozimmu_status_t st = host_buffers(h, sa + sb + sc);
    if (st) return st;
    uint8_t *base = static_cast<uint8_t *>(h->host_buf);
    double *dA = reinterpret_cast<double *>(base), *dB = reinterpret_cast<double *>(base + sa);
    double *dC = reinterpret_cast<double *>(base + sa + sb);
    cudaError_t e = cudaSuccess;
    if (use_ab) {
        e = copy2d(dA, ar, A, lda, ar, ac, cudaMemcpyHostToDevice, h->stream);
        if (e == cudaSuccess) e = copy2d(dB, br, B, ldb, br, bc, cudaMemcpyHostToDevice, h->stream);
    }
    if (e == cudaSuccess && *beta != 0.0)
        e = copy2d(dC, m, C, ldc, m, n, cudaMemcpyHostToDevice, h->stream);
    if (e != cudaSuccess) return cuda_status(e);
    st = ozimmu_dgemm(h, transA, transB, m, n, k, alpha, use_ab ? dA : nullptr, ar > 1 ? ar : 1,
                      use_ab ? dB : nullptr, br > 1 ? br : 1, beta, dC, m > 1 ? m : 1, num_slices);
    if (st) return st;
    e = copy2d(C, ldc, dC, m, m, n, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    return cuda_status(e);
}

// INT8-AUTO with host buffers, pipelined (f2): op(A) row blocks and op(B) column
// chunks go H2D on one stream while the mantissa-loss scan of each arrived block runs on the
// compute stream (row / column exponents are local to a block, and the per-s loss sums are
// additive); one D2H read picks s; B is sliced once, then C is computed in row blocks whose
// D2H overlaps the next block's GEMM.  Bitwise equal to ozimmu_dgemm with num_slices = 0.
ozimmu_status_t host_auto(ozimmu_handle_t h, ozimmu_op_t transA, ozimmu_op_t transB, int64_t m,
                          int64_t n, int64_t k, const double *alpha, const double *A, int64_t lda,
                          const double *B, int64_t ldb, const double *beta, double *C,
                          int64_t ldc) {
    constexpr int NS = 33;
    const int s_max = h->auto_smax;
    const int w = slice_width(k);
    const bool a_contig = transA != OZIMMU_OP_N, b_contig = transB == OZIMMU_OP_N;
    const int64_t ar = a_contig ? k : m, ac = a_contig ? m : k;  // stored shapes
    const int64_t br = b_contig ? k : n, bc = b_contig ? n : k;
    const size_t sa = align_up(sizeof(double) * (size_t)ar * ac);
    const size_t sb = align_up(sizeof(double) * (size_t)br * bc);
    const size_t sc = align_up(sizeof(double) * (size_t)m * n);
    const size_t sk = align_up(sizeof(int32_t) * (size_t)(m > n ? m : n));
    ozimmu_status_t st = host_buffers(h, sa + sb + sc + sk);
    if (st) return st;
    if (!h->auto_dev && cudaMalloc(&h->auto_dev, 2 * NS * sizeof(unsigned long long)) != cudaSuccess) {
        cudaGetLastError();
        return OZIMMU_ERR_WORKSPACE;
    }
    uint8_t *base = static_cast<uint8_t *>(h->host_buf);
    double *dA = reinterpret_cast<double *>(base), *dB = reinterpret_cast<double *>(base + sa);
    double *dC = reinterpret_cast<double *>(base + sa + sb);
    int32_t *keys = reinterpret_cast<int32_t *>(base + sa + sb + sc);
    const int64_t nblk = 8;
    const int64_t mb = round_up(ceil_div(m, nblk), 128), nbk = round_up(ceil_div(n, nblk), 96);
    const int64_t P = ceil_div(m, mb), J = ceil_div(n, nbk);
    std::vector<cudaEvent_t> ev((size_t)(P + J + P + 1));
    cudaError_t e = cudaSuccess;
    size_t made = 0;
    for (; made < ev.size() && e == cudaSuccess; ++made)
        e = cudaEventCreateWithFlags(&ev[made], cudaEventDisableTiming);
    cudaEvent_t *ev_in = ev.data(), *ev_cdone = ev.data() + P + J, ev_start = ev[ev.size() - 1];
    cudaStream_t cs = h->stream;
    int launches = 0;
    void *bbuf = nullptr;
    int s = s_max;
#define OZ_TRY(x) do { if (e == cudaSuccess) e = (x); } while (0)
    OZ_TRY(cudaEventRecord(ev_start, cs));
    OZ_TRY(cudaStreamWaitEvent(h->h2d, ev_start, 0));
    OZ_TRY(cudaStreamWaitEvent(h->d2h, ev_start, 0));
    OZ_TRY(cudaMemsetAsync(h->auto_dev, 0, 2 * NS * sizeof(unsigned long long), cs));
    // ---- H2D in blocks, scan each block as it lands ----
    for (int64_t i = 0; i < P; ++i) {
        const int64_t r0 = i * mb, mi = (i == P - 1) ? m - r0 : mb;
        const double *src = a_contig ? dA + r0 * k : dA + r0;
        if (a_contig)  // stored k x m: op(A) rows r0.. = columns r0..
            OZ_TRY(copy2d(dA + r0 * k, k, A + r0 * lda, lda, k, mi, cudaMemcpyHostToDevice, h->h2d));
        else
            OZ_TRY(copy2d(dA + r0, m, A + r0, lda, mi, k, cudaMemcpyHostToDevice, h->h2d));
        OZ_TRY(cudaEventRecord(ev_in[i], h->h2d));
        OZ_TRY(cudaStreamWaitEvent(cs, ev_in[i], 0));
        OZ_TRY(launch_mantissa_loss(src, a_contig ? k : m, a_contig, mi, k, w, s_max, h->auto_dev,
                                    keys, h->num_sms, cs, &launches));
    }
    for (int64_t j = 0; j < J; ++j) {
        const int64_t c0 = j * nbk, nc = (j == J - 1) ? n - c0 : nbk;
        const double *src = b_contig ? dB + c0 * k : dB + c0;
        if (b_contig)  // stored k x n: op(B) columns c0..
            OZ_TRY(copy2d(dB + c0 * k, k, B + c0 * ldb, ldb, k, nc, cudaMemcpyHostToDevice, h->h2d));
        else
            OZ_TRY(copy2d(dB + c0, n, B + c0, ldb, nc, k, cudaMemcpyHostToDevice, h->h2d));
        OZ_TRY(cudaEventRecord(ev_in[P + j], h->h2d));
        OZ_TRY(cudaStreamWaitEvent(cs, ev_in[P + j], 0));
        OZ_TRY(launch_mantissa_loss(src, b_contig ? k : n, b_contig, nc, k, w, s_max,
                                    h->auto_dev + NS, keys, h->num_sms, cs, &launches));
    }
    if (*beta != 0.0) OZ_TRY(copy2d(dC, m, C, ldc, m, n, cudaMemcpyHostToDevice, h->h2d));
    // ---- choose s (one D2H read) ----
    unsigned long long sums[2 * NS];
    OZ_TRY(cudaMemcpyAsync(sums, h->auto_dev, sizeof(sums), cudaMemcpyDeviceToHost, cs));
    OZ_TRY(cudaStreamSynchronize(cs));
    OZ_TRY(cudaStreamSynchronize(h->h2d));  // C (beta != 0) is on the device too
    if (e == cudaSuccess) {
        for (int q = 1; q <= s_max; ++q) {
            const double ma = sums[32] ? (double)sums[q - 1] / (double)sums[32] : 0.0;
            const double mbv = sums[NS + 32] ? (double)sums[NS + q - 1] / (double)sums[NS + 32] : 0.0;
            if (ma <= h->auto_T && mbv <= h->auto_T) {
                s = q;
                break;
            }
        }
        h->auto_last_s = s;
        const size_t need = ozimmu_b_slices_bytes(n, k, s);
        if (need > h->auto_bbuf_bytes) {
            if (h->auto_bbuf) cudaFree(h->auto_bbuf);
            h->auto_bbuf = nullptr;
            h->auto_bbuf_bytes = 0;
            if (cudaMalloc(&h->auto_bbuf, need) != cudaSuccess) {
                cudaGetLastError();
                e = cudaErrorMemoryAllocation;
            } else {
                h->auto_bbuf_bytes = need;
            }
        }
        bbuf = h->auto_bbuf;
    }
    // ---- slice B once, then C row blocks: GEMM i overlaps the D2H of block i-1 ----
    ozimmu_status_t st2 = OZIMMU_SUCCESS;
    int64_t total_launches = launches;
    if (e == cudaSuccess) {
        st2 = ozimmu_slice_b(h, transB, k, n, dB, b_contig ? k : n, s, bbuf);
        total_launches += h->report.launches;
    }
    int64_t done = 0;
    for (int64_t i = 0; i < P && e == cudaSuccess && st2 == OZIMMU_SUCCESS; ++i, ++done) {
        const int64_t r0 = i * mb, mi = (i == P - 1) ? m - r0 : mb;
        const double *Ai = a_contig ? dA + r0 * k : dA + r0;
        st2 = ozimmu_dgemm_presliced_b(h, transA, mi, n, k, alpha, Ai, a_contig ? k : m, bbuf,
                                       beta, dC + r0, m, s);
        total_launches += h->report.launches;
        if (st2) break;
        OZ_TRY(cudaEventRecord(ev_cdone[i], cs));
        OZ_TRY(cudaStreamWaitEvent(h->d2h, ev_cdone[i], 0));
        OZ_TRY(copy2d(C + r0, ldc, dC + r0, m, mi, n, cudaMemcpyDeviceToHost, h->d2h));
    }
    OZ_TRY(cudaStreamSynchronize(h->d2h));
    OZ_TRY(cudaStreamSynchronize(cs));
#undef OZ_TRY
    if (e != cudaSuccess || st2) {
        cudaStreamSynchronize(h->h2d);
        cudaStreamSynchronize(h->d2h);
        cudaStreamSynchronize(cs);
    }
    for (size_t i = 0; i < made; ++i) cudaEventDestroy(ev[i]);
    if (st2) return st2;
    if (e != cudaSuccess) return cuda_status(e);
    GemmPlan gp;
    plan_gemm(s, w, mb, n, round_up(k, 16), gemm_sms(h), &gp);
    fill_report(h, s, w, m, n, k, &gp, (int)total_launches,
                (int64_t)s * (m + n) * round_up(k, 16) + 4 * (m + n));
    return OZIMMU_SUCCESS;
}

}  // namespace

extern "C" ozimmu_status_t ozimmu_dgemm_host(ozimmu_handle_t h, ozimmu_op_t transA,
                                             ozimmu_op_t transB, int64_t m, int64_t n, int64_t k,
                                             const double *alpha, const double *A, int64_t lda,
                                             const double *B, int64_t ldb, const double *beta,
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
    if (num_slices == 0 && *alpha != 0.0 && k > 0 && k <= OZIMMU_MAX_K)
        return host_auto(h, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
    if (num_slices == 0 || *alpha == 0.0 || k == 0)
        return host_full(h, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc,
                         num_slices);
    const int s = num_slices;
    const int w = slice_width(k);
    const int64_t k_pad = round_up(k, 16);
    HostPlan hp;
    if (!host_plan(h, m, n, k, s, &hp)) return OZIMMU_ERR_UNSUPPORTED;
    st = host_buffers(h, hp.total);
    if (st) return st;
    uint8_t *base = static_cast<uint8_t *>(h->host_buf);
    int8_t *a_planes = reinterpret_cast<int8_t *>(base + hp.o_apl);
    int32_t *EA = reinterpret_cast<int32_t *>(base + hp.o_apl + align_up((size_t)s * m * k_pad));
    uint8_t *bbuf = base + hp.o_bbuf;
    int8_t *b_planes = reinterpret_cast<int8_t *>(bbuf);
    int32_t *EB = reinterpret_cast<int32_t *>(bbuf + b_buf_planes_bytes(n, k_pad, s));
    double *dC = reinterpret_cast<double *>(base + hp.o_c);
    int32_t *keys = reinterpret_cast<int32_t *>(base + hp.o_keys);
    int64_t *scratch = reinterpret_cast<int64_t *>(base + hp.o_scratch);
    unsigned int *sync = reinterpret_cast<unsigned int *>(base + hp.o_sync);
    const bool has_beta = *beta != 0.0;
    const bool a_rows_contig = transA != OZIMMU_OP_N;  // device copy of a row block
    const bool b_cols_contig = transB == OZIMMU_OP_N;

    // Transfers alternate between A row blocks and B column chunks (A_0, B_0, A_1, B_1, ...),
    // so the computable part of C grows as a square: after A_i arrives, C block row i
    // against the chunks already sliced is one GEMM; after B_j arrives, C chunk j against the
    // row blocks already sliced is one GEMM.  The tensor cores start after the first block
    // and chunk, and every C region goes back to the host as soon as its GEMM is done.
    const int64_t P = hp.P, J = hp.J;
    const int64_t n_ev = 1 + 2 * P + 2 * J + 3 * (P + J);
    cudaEvent_t *ev = static_cast<cudaEvent_t *>(calloc((size_t)n_ev, sizeof(cudaEvent_t)));
    if (!ev) return OZIMMU_ERR_WORKSPACE;
    cudaError_t e = cudaSuccess;
    int64_t made = 0;
    for (; made < n_ev && e == cudaSuccess; ++made)
        e = cudaEventCreateWithFlags(&ev[made], cudaEventDisableTiming);
    cudaEvent_t ev_start = ev[0];
    cudaEvent_t *ev_ain = ev + 1, *ev_afree = ev_ain + P, *ev_bin = ev_afree + P,
                *ev_bfree = ev_bin + J, *ev_cin = ev_bfree + J, *ev_cdone = ev_cin + (P + J),
                *ev_cout = ev_cdone + (P + J);
    int64_t nreg = 0;  // C regions issued
    int launches = 0;
    cudaStream_t cs = h->stream;
#define OZ_TRY(x) do { if (e == cudaSuccess) e = (x); } while (0)
    OZ_TRY(cudaEventRecord(ev_start, cs));
    OZ_TRY(cudaStreamWaitEvent(h->h2d, ev_start, 0));
    OZ_TRY(cudaStreamWaitEvent(h->d2h, ev_start, 0));

    auto rows_of = [&](int64_t i) { return hp.rb[i + 1] - hp.rb[i]; };
    auto cols_of = [&](int64_t j) { return hp.cb[j + 1] - hp.cb[j]; };
    // C region rows [r0, r0+mr) x cols [c0, c0+nc): (beta C in), GEMM, C out
    auto region = [&](int64_t r0, int64_t mr, int64_t c0, int64_t nc) {
        if (mr <= 0 || nc <= 0) return;
        const int64_t q = nreg++;
        double *dCr = dC + r0 + c0 * m;
        if (has_beta) {
            OZ_TRY(copy2d(dCr, m, C + r0 + c0 * ldc, ldc, mr, nc, cudaMemcpyHostToDevice, h->h2d));
            OZ_TRY(cudaEventRecord(ev_cin[q], h->h2d));
            OZ_TRY(cudaStreamWaitEvent(cs, ev_cin[q], 0));
        }
        GemmPlan gp;
        if (!plan_gemm(s, w, mr, nc, k_pad, gemm_sms(h), &gp)) {
            if (e == cudaSuccess) e = cudaErrorInvalidValue;
            return;
        }
        OZ_TRY(fused_gemm(h, gp, mr, nc, k_pad, s, w, a_planes + r0 * k_pad, EA + r0,
                          b_planes + c0 * k_pad, EB + c0, n, *alpha, *beta, dCr, m, scratch,
                          sync, &launches, BatchMap(), BatchMap(), m));
        OZ_TRY(cudaEventRecord(ev_cdone[q], cs));
        OZ_TRY(cudaStreamWaitEvent(h->d2h, ev_cdone[q], 0));
        OZ_TRY(copy2d(C + r0 + c0 * ldc, ldc, dCr, m, mr, nc, cudaMemcpyDeviceToHost, h->d2h));
        OZ_TRY(cudaEventRecord(ev_cout[q], h->d2h));
    };
    int64_t ia = 0, jb = 0;  // A blocks / B chunks sliced so far
    while (ia < P || jb < J) {
        const bool take_a = ia < P && (jb >= J || ia * J <= jb * P);
        if (take_a) {
            const int64_t i = ia, r0 = hp.rb[i], mi = rows_of(i);
            double *dst = reinterpret_cast<double *>(base + hp.o_ast[i & 1]);
            if (i >= 2) OZ_TRY(cudaStreamWaitEvent(h->h2d, ev_afree[i - 2], 0));
            if (a_rows_contig)  // stored k x m: columns r0 .. r0+mi
                OZ_TRY(copy2d(dst, k, A + r0 * lda, lda, k, mi, cudaMemcpyHostToDevice, h->h2d));
            else  // stored m x k: rows r0 .. r0+mi of every column
                OZ_TRY(copy2d(dst, mi, A + r0, lda, mi, k, cudaMemcpyHostToDevice, h->h2d));
            OZ_TRY(cudaEventRecord(ev_ain[i], h->h2d));
            OZ_TRY(cudaStreamWaitEvent(cs, ev_ain[i], 0));
            OZ_TRY(launch_split(dst, a_rows_contig ? k : mi, a_rows_contig, mi, k, k_pad, s, w,
                                /*reverse=*/false, a_planes + r0 * k_pad, m * k_pad, EA + r0,
                                keys, h->num_sms, cs, &launches));
            OZ_TRY(cudaEventRecord(ev_afree[i], cs));
            ++ia;
            region(r0, mi, 0, hp.cb[jb]);
        } else {
            const int64_t j = jb, c0 = hp.cb[j], nc = cols_of(j);
            double *dst = reinterpret_cast<double *>(base + hp.o_bst[j & 1]);
            if (j >= 2) OZ_TRY(cudaStreamWaitEvent(h->h2d, ev_bfree[j - 2], 0));
            if (b_cols_contig)  // stored k x n: columns c0 .. c0+nc
                OZ_TRY(copy2d(dst, k, B + c0 * ldb, ldb, k, nc, cudaMemcpyHostToDevice, h->h2d));
            else  // stored n x k: rows c0 .. c0+nc
                OZ_TRY(copy2d(dst, nc, B + c0, ldb, nc, k, cudaMemcpyHostToDevice, h->h2d));
            OZ_TRY(cudaEventRecord(ev_bin[j], h->h2d));
            OZ_TRY(cudaStreamWaitEvent(cs, ev_bin[j], 0));
            OZ_TRY(launch_split(dst, b_cols_contig ? k : nc, b_cols_contig, nc, k, k_pad, s, w,
                                /*reverse=*/true, b_planes + c0 * k_pad, n * k_pad, EB + c0, keys,
                                h->num_sms, cs, &launches));
            OZ_TRY(cudaEventRecord(ev_bfree[j], cs));
            ++jb;
            region(0, hp.rb[ia], c0, nc);
        }
    }
    for (int64_t q = 0; q < nreg; ++q) OZ_TRY(cudaStreamWaitEvent(cs, ev_cout[q], 0));
    OZ_TRY(cudaStreamSynchronize(cs));
#undef OZ_TRY
    if (e != cudaSuccess) {
        cudaStreamSynchronize(h->h2d);
        cudaStreamSynchronize(h->d2h);
        cudaStreamSynchronize(cs);
    }
    for (int64_t i = 0; i < made; ++i) cudaEventDestroy(ev[i]);
    free(ev);
    if (e != cudaSuccess) return cuda_status(e);
    GemmPlan gp;
    plan_gemm(s, w, hp.mb, n, k_pad, gemm_sms(h), &gp);
    fill_report(h, s, w, m, n, k, &gp, launches, (int64_t)s * (m + n) * k_pad + 4 * (m + n));
    return OZIMMU_SUCCESS;
}
