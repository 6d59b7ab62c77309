// handle.h -- private runtime header of libozimmu: the handle and the host-side helpers shared
// by api.cu (the method's entry points), host.cu (host-buffer pipeline) and dist.cu (multi-GPU).
// Not part of the public ABI (see include/ozimmu.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ozimmu.h"
#include "internal.h"

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
    // INT8-AUTO (num_slices = 0): the accuracy-targeted rule (reading A18, tau) by default, or
    // the paper's mean-mantissa-loss rule (reading A17, threshold T); s cap (18)
    int auto_mode = OZIMMU_AUTO_ACCURACY;
    double auto_T = 0.0;
    double auto_tau = 1.0;
    int auto_smax = 18;
    int auto_last_s = 0;
    bool auto_last_capped = false;
    unsigned long long *auto_dev = nullptr;  // device [2][33]: loss sums or rho (double bits)
    // host-buffer entry point (ozimmu_dgemm_host): copy streams + device staging buffer
    cudaStream_t h2d = nullptr, d2h = nullptr;
    void *host_buf = nullptr;
    size_t host_buf_bytes = 0;
    void *auto_bbuf = nullptr;  // B-slice buffer of the INT8-AUTO host path (grown, kept)
    size_t auto_bbuf_bytes = 0;
    // second stream for slicing op(B) concurrently with op(A) (fork / join by events)
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // multi-GPU (dist.cu): collective stream, settings (ozimmu_set_dist), the
    // FP64 receive buffer of the FP64-broadcast variant
    cudaStream_t comm = nullptr;
    int dist_chunk_cols = 0;   // 0: about n/8 columns per broadcast chunk
    int dist_reserve_sms = 8;  // SMs left to the collective while broadcasts are in flight
    int dist_bcast_fp64 = 0;   // 1: broadcast FP64 B and slice it on every rank
    void *dist_buf = nullptr;
    size_t dist_buf_bytes = 0;
};

namespace ozimmu {
namespace rt {

constexpr size_t kAlign = 256;

// SMs the fused GEMM may occupy (ozimmu_set_max_sms)
inline int gemm_sms(ozimmu_handle_t h) {
    return (h->gemm_sms > 0 && h->gemm_sms < h->num_sms) ? h->gemm_sms : h->num_sms;
}

inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Layout {  // workspace carve-up for one dgemm call
    size_t a_planes, a_exp, b_buf, keys, keys_b, sync, scratch, total;
};

// Phase events of one computing call (ozimmu_timing_read): start, B sliced (on the stream
// that sliced it), A sliced, GEMM start (after the join), GEMM end.
enum : int { PH_START = 0, PH_B = 1, PH_A = 2, PH_GEMM0 = 3, PH_GEMM1 = 4, kPhases = 5 };
// Record phase event `ph` of the current call on stream `st` (default: the handle's stream)
// if timing is on.
inline void mark(ozimmu_handle_t h, int ph, cudaStream_t st = nullptr) {
    if (h->timing_cap && h->timing_count < h->timing_cap)
        cudaEventRecord(h->events[kPhases * h->timing_count + ph], st ? st : h->stream);
}
inline void mark_done(ozimmu_handle_t h) {
    if (h->timing_cap && h->timing_count < h->timing_cap) ++h->timing_count;
}

// B-slice buffer: planes [s][n][k_pad] (reversed slice order) | int32 exponents [n]
size_t b_buf_planes_bytes(int64_t n, int64_t k_pad, int s);
size_t b_buf_bytes(int64_t n, int64_t k_pad, int s);
Layout layout(int64_t m, int64_t n, int64_t k_pad, int s, size_t scratch);
bool valid_op(ozimmu_op_t op);
// The workspace for one call: the caller's (ozimmu_set_workspace) or the handle's own,
// grown on demand (synchronising the stream before freeing the old one).
ozimmu_status_t get_ws(ozimmu_handle_t h, size_t need, void **ws);
ozimmu_status_t cuda_status(cudaError_t e);
// Validation shared by the real entry points (the A side, sizes, alpha/beta, C, s).
ozimmu_status_t check_common(ozimmu_handle_t h, ozimmu_op_t transA, int64_t m, int64_t n,
                             int64_t k, const double *alpha, const double *A, int64_t lda,
                             const double *beta, double *C, int64_t ldc, int s);
void fill_report(ozimmu_handle_t h, int s, int w, int64_t m, int64_t n, int64_t k,
                 const GemmPlan *gp, int launches, int64_t slice_bytes);
void note_auto(ozimmu_handle_t h);
// C = beta C (alpha == 0 or k == 0 quick return; A and B are not read).
ozimmu_status_t scale_only(ozimmu_handle_t h, int64_t m, int64_t n, double beta, double *C,
                           int64_t ldc);
// Slice op(A) (rows) into planes [s][m][k_pad] + E_A.
cudaError_t slice_a(ozimmu_handle_t h, ozimmu_op_t transA, int64_t m, int64_t k, int64_t k_pad,
                    const double *A, int64_t lda, int s, int w, int8_t *planes, int32_t *E,
                    int32_t *keys, int *launches, BatchMap vm = BatchMap());
// Slice op(B) (columns) into a B-slice buffer of n columns.
cudaError_t slice_b(ozimmu_handle_t h, ozimmu_op_t transB, int64_t k, int64_t n, int64_t k_pad,
                    const double *B, int64_t ldb, int s, int w, uint8_t *bbuf, int32_t *keys,
                    int *launches, BatchMap vm = BatchMap(), cudaStream_t st = nullptr);
// Fork / join of the handle's second stream (work on h->aux runs concurrently in between).
cudaError_t aux_fork(ozimmu_handle_t h);
cudaError_t aux_join(ozimmu_handle_t h);
// INT8-AUTO (f2): statistics slots, decision, scratch, statistics kernels, selection.
constexpr int kAutoNS = 33;
int auto_decide(ozimmu_handle_t h, const unsigned long long *stat, int64_t k_acc, int s_lim,
                bool *capped);
size_t auto_scratch_bytes(ozimmu_handle_t h, int64_t rows);
cudaError_t auto_stats(ozimmu_handle_t h, const double *M, int64_t ld, bool contiguous,
                       int64_t rows, int64_t kdim, int w, int s_lim, unsigned long long *stat_op,
                       void *scratch, cudaStream_t st, int *launches, int cpx);
int auto_first_limit(ozimmu_handle_t h);
ozimmu_status_t auto_select(ozimmu_handle_t h, ozimmu_op_t transA, ozimmu_op_t transB, int64_t m,
                            int64_t n, int64_t k, const double *A, int64_t lda, const double *B,
                            int64_t ldb, int *s_out, int *launches, bool cpx = false);
// The fused tcgen05 GEMM + FP64 epilogue (A4 + A5) on sliced operands, on h->stream.
// b_plane_rows / a_plane_rows: rows per plane in memory (0 = n / m: a column chunk / row
// block of a larger slice buffer otherwise).
cudaError_t fused_gemm(ozimmu_handle_t h, const GemmPlan &gp, int64_t m, int64_t n, int64_t k_pad,
                       int s, int w, const int8_t *a_planes, const int32_t *EA,
                       const int8_t *b_planes, const int32_t *EB, int64_t b_plane_rows,
                       double alpha, double beta, double *C, int64_t ldc, int64_t *scratch,
                       unsigned int *sync, int *launches, BatchMap crow = BatchMap(),
                       BatchMap ccol = BatchMap(), int64_t a_plane_rows = 0,
                       bool counter_zeroed = false);
// slice(B) || slice(A) -> fused GEMM for one real call (bbuf_ext: B already sliced).
ozimmu_status_t gemm_core(ozimmu_handle_t h, ozimmu_op_t transA, int64_t m, int64_t n, int64_t k,
                          double alpha, const double *A, int64_t lda, const uint8_t *bbuf_ext,
                          ozimmu_op_t transB, const double *B, int64_t ldb, double beta,
                          double *C, int64_t ldc, int s, BatchMap amap = BatchMap(),
                          BatchMap bmap = BatchMap(), BatchMap crow = BatchMap(),
                          BatchMap ccol = BatchMap());

}  // namespace rt
}  // namespace ozimmu
