// host.cu -- ozimmu_dgemm_host: the host-buffer entry point (H2D copies, slicing, GEMM and
// D2H overlapped on three streams; BJ metric "including the matrix splitting" end to end).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>

#include "ozimmu.h"
#include "internal.h"
#include "handle.h"

using namespace ozimmu;
using namespace ozimmu::rt;

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
        const size_t c = chunk_scratch_bound(gp, s, h->num_sms);  // any region shape
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
    off += align_up(split_scratch_bytes(mb > nb ? mb : nb));
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
    constexpr int NS = kAutoNS;
    const int s_max = h->auto_smax;
    const int w = slice_width(k);
    const bool a_contig = transA != OZIMMU_OP_N, b_contig = transB == OZIMMU_OP_N;
    const int64_t ar = a_contig ? k : m, ac = a_contig ? m : k;  // stored shapes
    const int64_t br = b_contig ? k : n, bc = b_contig ? n : k;
    const size_t sa = align_up(sizeof(double) * (size_t)ar * ac);
    const size_t sb = align_up(sizeof(double) * (size_t)br * bc);
    const size_t sc = align_up(sizeof(double) * (size_t)m * n);
    const size_t sk = auto_scratch_bytes(h, m > n ? m : n);
    ozimmu_status_t st = host_buffers(h, sa + sb + sc + sk);
    if (st) return st;
    if (!h->auto_dev && cudaMalloc(&h->auto_dev, 2 * NS * sizeof(unsigned long long)) != cudaSuccess) {
        cudaGetLastError();
        return OZIMMU_ERR_WORKSPACE;
    }
    uint8_t *base = static_cast<uint8_t *>(h->host_buf);
    double *dA = reinterpret_cast<double *>(base), *dB = reinterpret_cast<double *>(base + sa);
    double *dC = reinterpret_cast<double *>(base + sa + sb);
    void *keys = base + sa + sb + sc;  // AUTO statistics scratch
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
    const int lim1 = auto_first_limit(h);
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
        OZ_TRY(auto_stats(h, src, a_contig ? k : m, a_contig, mi, k, w, lim1, h->auto_dev, keys,
                          cs, &launches, 0));
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
        OZ_TRY(auto_stats(h, src, b_contig ? k : n, b_contig, nc, k, w, lim1, h->auto_dev + NS,
                          keys, cs, &launches, 0));
    }
    if (*beta != 0.0) OZ_TRY(copy2d(dC, m, C, ldc, m, n, cudaMemcpyHostToDevice, h->h2d));
    // ---- choose s (one D2H read) ----
    unsigned long long sums[2 * NS];
    OZ_TRY(cudaMemcpyAsync(sums, h->auto_dev, sizeof(sums), cudaMemcpyDeviceToHost, cs));
    OZ_TRY(cudaStreamSynchronize(cs));
    OZ_TRY(cudaStreamSynchronize(h->h2d));  // C (beta != 0) is on the device too
    bool capped = false;
    if (e == cudaSuccess) s = auto_decide(h, sums, k, lim1, &capped);
    if (e == cudaSuccess && capped && lim1 < s_max) {
        // second pass over the whole (landed) operands with every candidate s
        OZ_TRY(cudaMemsetAsync(h->auto_dev, 0, 2 * NS * sizeof(unsigned long long), cs));
        OZ_TRY(auto_stats(h, dA, a_contig ? k : m, a_contig, m, k, w, s_max, h->auto_dev, keys,
                          cs, &launches, 0));
        OZ_TRY(auto_stats(h, dB, b_contig ? k : n, b_contig, n, k, w, s_max, h->auto_dev + NS,
                          keys, cs, &launches, 0));
        OZ_TRY(cudaMemcpyAsync(sums, h->auto_dev, sizeof(sums), cudaMemcpyDeviceToHost, cs));
        OZ_TRY(cudaStreamSynchronize(cs));
        if (e == cudaSuccess) s = auto_decide(h, sums, k, s_max, &capped);
    }
    if (e == cudaSuccess) {
        h->auto_last_capped = capped;
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
    note_auto(h);
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
    // OZIMMU_HOST_TRACE=1 (development): timing events and a timeline on stderr after the call
    static const bool trace = getenv("OZIMMU_HOST_TRACE") != nullptr;
    const int64_t n_ev = 1 + 2 * P + 2 * J + 4 * (P + J);
    cudaEvent_t *ev = static_cast<cudaEvent_t *>(calloc((size_t)n_ev, sizeof(cudaEvent_t)));
    if (!ev) return OZIMMU_ERR_WORKSPACE;
    cudaError_t e = cudaSuccess;
    int64_t made = 0;
    for (; made < n_ev && e == cudaSuccess; ++made)
        e = cudaEventCreateWithFlags(&ev[made], trace ? cudaEventDefault : cudaEventDisableTiming);
    cudaEvent_t ev_start = ev[0];
    cudaEvent_t *ev_ain = ev + 1, *ev_afree = ev_ain + P, *ev_bin = ev_afree + P,
                *ev_bfree = ev_bin + J, *ev_cin = ev_bfree + J, *ev_cdone = ev_cin + (P + J),
                *ev_cout = ev_cdone + (P + J), *ev_gstart = ev_cout + (P + J);
    std::vector<int64_t> reg_shape;  // trace: rows, cols of each region
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
        if (trace) {
            OZ_TRY(cudaEventRecord(ev_gstart[q], cs));
            reg_shape.push_back(mr);
            reg_shape.push_back(nc);
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
    if (trace && e == cudaSuccess) {
        auto at = [&](cudaEvent_t x) {
            float ms = -1.f;
            cudaEventElapsedTime(&ms, ev_start, x);
            return ms;
        };
        for (int64_t i = 0; i < P; ++i)
            fprintf(stderr, "[host trace] A%lld rows %lld in %.3f\n", (long long)i,
                    (long long)rows_of(i), at(ev_ain[i]));
        for (int64_t j = 0; j < J; ++j)
            fprintf(stderr, "[host trace] B%lld cols %lld in %.3f\n", (long long)j,
                    (long long)cols_of(j), at(ev_bin[j]));
        for (int64_t q = 0; q < nreg; ++q)
            fprintf(stderr, "[host trace] R%lld %lldx%lld gemm %.3f..%.3f out %.3f\n", (long long)q,
                    (long long)reg_shape[2 * q], (long long)reg_shape[2 * q + 1], at(ev_gstart[q]),
                    at(ev_cdone[q]), at(ev_cout[q]));
    }
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
