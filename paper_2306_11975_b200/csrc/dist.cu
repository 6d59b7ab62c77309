// dist.cu -- multi-GPU Ozaki DGEMM inside the library (BASELINE north_star:
// "C is partitioned into row blocks ... Each GPU slices its own A rows, B's slices are
// computed once and NCCL-broadcast over NVLink, and there are no other collectives").
//
// One process per GPU.  Rank r owns rows of C and of op(A) (m_local of them) and slices them
// itself: row exponents are per row (Alg. 4 line 2), so no communication is needed.
// op(B) is read on the root only.  The root slices it column chunk by column chunk into the
// B-slice buffer (planes [s][n][k_pad] in reversed slice order + int32 exponents [n], the
// layout the GEMM's TMA reads), and each chunk goes to every rank as ONE group of s + 1
// broadcasts (the chunk's rows of each plane and its exponents are contiguous) on the handle's
// collective stream.  The GEMM of a chunk waits only for that chunk's broadcast, so the
// transfer of later chunks overlaps the tensor work on earlier ones.  GEMM launches cover
// 1, 1, 2, 4, ... chunks (fewer launches once the broadcasts are ahead), and while broadcasts
// are still in flight the persistent GEMM leaves `reserve_sms` SMs free: it holds one
// ~227 KB-shared-memory CTA per SM, so a collective kernel enqueued beside it could otherwise
// only start when it ends.  There is no reduction: every element of C is computed on one GPU
// by the canonical operation sequence, so C is bitwise identical to the single-GPU call for
// every world size and partition.
//
// The byte trade-off of s8e is selectable (ozimmu_set_dist): broadcast B's INT8 planes (s
// bytes per element, the default and the north_star's design) or FP64 B (8 bytes per element)
// and slice every chunk on every rank.
//
// Transports: NCCL (ozimmu_dgemm_nccl; libnccl is dlopen'ed, preferring the copy the process
// already loaded, so the library still loads without NCCL) or a caller-supplied broadcast
// function (ozimmu_dgemm_bcast; the tests' gloo transport).
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <dlfcn.h>
#include <vector>
#include <cuda_runtime.h>
#include <nccl.h>

#include "ozimmu.h"
#include "internal.h"
#include "handle.h"

using namespace ozimmu;
using namespace ozimmu::rt;

namespace {

// ---- NCCL, resolved at run time ---------------------------------------------------------
struct Nccl {
    bool tried = false, ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitRankConfig)(ncclComm_t *, int, ncclUniqueId, int, ncclConfig_t *) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommUserRank)(const ncclComm_t, int *) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int *) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
};

Nccl &nccl() {
    static Nccl N;
    if (N.tried) return N;
    N.tried = true;
    void *lib = nullptr;
    if (const char *p = getenv("OZIMMU_NCCL_LIB")) lib = dlopen(p, RTLD_NOW | RTLD_LOCAL);
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // e.g. torch's copy
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!lib) return N;
#define OZ_SYM(f) N.f = reinterpret_cast<decltype(N.f)>(dlsym(lib, "nccl" #f))
    OZ_SYM(GetUniqueId);
    OZ_SYM(CommInitRank);
    OZ_SYM(CommInitRankConfig);
    OZ_SYM(CommDestroy);
    OZ_SYM(CommUserRank);
    OZ_SYM(CommCount);
    OZ_SYM(Broadcast);
    OZ_SYM(GroupStart);
    OZ_SYM(GroupEnd);
#undef OZ_SYM
    N.ok = N.GetUniqueId && N.CommInitRank && N.CommDestroy && N.CommUserRank && N.CommCount &&
           N.Broadcast && N.GroupStart && N.GroupEnd;
    return N;
}

// ---- transports ---------------------------------------------------------------------------
struct Transport {
    virtual ~Transport() = default;
    virtual ozimmu_status_t begin() { return OZIMMU_SUCCESS; }
    // enqueue: `bytes` at `buf` from root to every rank, ordered on stream st
    virtual ozimmu_status_t bcast(void *buf, size_t bytes, int root, cudaStream_t st) = 0;
    virtual ozimmu_status_t end() { return OZIMMU_SUCCESS; }
};

struct NcclTransport : Transport {
    ncclComm_t comm;
    explicit NcclTransport(ncclComm_t c) : comm(c) {}
    ozimmu_status_t begin() override {
        return nccl().GroupStart() == ncclSuccess ? OZIMMU_SUCCESS : OZIMMU_ERR_NCCL;
    }
    ozimmu_status_t bcast(void *buf, size_t bytes, int root, cudaStream_t st) override {
        return nccl().Broadcast(buf, buf, bytes, ncclUint8, root, comm, st) == ncclSuccess
                   ? OZIMMU_SUCCESS : OZIMMU_ERR_NCCL;
    }
    ozimmu_status_t end() override {
        return nccl().GroupEnd() == ncclSuccess ? OZIMMU_SUCCESS : OZIMMU_ERR_NCCL;
    }
};

struct FnTransport : Transport {
    ozimmu_bcast_fn fn;
    void *ctx;
    FnTransport(ozimmu_bcast_fn f, void *c) : fn(f), ctx(c) {}
    ozimmu_status_t bcast(void *buf, size_t bytes, int root, cudaStream_t st) override {
        return fn(ctx, buf, bytes, root, st) == 0 ? OZIMMU_SUCCESS : OZIMMU_ERR_NCCL;
    }
};

// Column chunks [cb[j], cb[j+1]) of the broadcast and the GEMM launch groups over them: launch
// g covers chunks [gb[g], gb[g+1]) -- 1, 1, 2, 4, ... chunks.
struct DistPlan {
    std::vector<int64_t> cb;
    std::vector<int> gb;
};

DistPlan dist_plan(int64_t n, int64_t chunk_cols) {
    DistPlan d;
    for (int64_t c = 0; c < n; c += chunk_cols) d.cb.push_back(c);
    d.cb.push_back(n);
    const int J = (int)d.cb.size() - 1;
    d.gb.push_back(0);
    int size = 1;
    for (int j = 0; j < J;) {
        if (j >= 2) size *= 2;
        j = j + size < J ? j + size : J;
        d.gb.push_back(j);
    }
    return d;
}

// The shared driver of ozimmu_dgemm_nccl / ozimmu_dgemm_bcast (arguments validated).
ozimmu_status_t dist_core(ozimmu_handle_t h, Transport &tr, int rank, int root, ozimmu_op_t transA,
                          ozimmu_op_t transB, int64_t m_loc, int64_t n, int64_t k, double alpha,
                          const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                          double *C, int64_t ldc, int s) {
    const bool is_root = rank == root;
    const int w = slice_width(k);
    const int64_t k_pad = round_up(k, 16);
    int64_t cc = h->dist_chunk_cols > 0 ? h->dist_chunk_cols : round_up(ceil_div(n, 8), 96);
    if (cc > n) cc = n;
    const DistPlan dp = dist_plan(n, cc);
    const int J = (int)dp.cb.size() - 1;
    // FP64 broadcast of op(B) needs its columns contiguous on the root (transB = N, ldb = k);
    // every rank must take the same decision, so it depends on the shared arguments only
    const bool fp64 = h->dist_bcast_fp64 && transB == OZIMMU_OP_N && ldb == k;
    const int sms = h->num_sms;
    const int capped = sms - h->dist_reserve_sms > 0 ? sms - h->dist_reserve_sms : 1;
    // workspace: this rank's A planes + the full B-slice buffer (+ the GEMM scratch bound)
    GemmPlan gp_full;
    if (!plan_gemm(s, w, m_loc > 0 ? m_loc : 1, n, k_pad, sms, &gp_full)) return OZIMMU_ERR_UNSUPPORTED;
    const Layout L = layout(m_loc, n, k_pad, s, chunk_scratch_bound(gp_full, s, sms));
    void *ws = nullptr;
    ozimmu_status_t st = get_ws(h, L.total, &ws);
    if (st) return st;
    uint8_t *base = static_cast<uint8_t *>(ws);
    int8_t *a_planes = reinterpret_cast<int8_t *>(base + L.a_planes);
    int32_t *EA = reinterpret_cast<int32_t *>(base + L.a_exp);
    uint8_t *bbuf = base + L.b_buf;
    int8_t *b_planes = reinterpret_cast<int8_t *>(bbuf);
    int32_t *EB = reinterpret_cast<int32_t *>(bbuf + b_buf_planes_bytes(n, k_pad, s));
    // FP64 variant: non-root ranks receive op(B) into a handle-owned buffer (k x n, ld k)
    double *Bf = nullptr;
    if (fp64) {
        if (is_root) {
            Bf = const_cast<double *>(B);
        } else {
            const size_t need = sizeof(double) * (size_t)k * (size_t)n;
            if (need > h->dist_buf_bytes) {
                if (h->dist_buf) {
                    cudaDeviceSynchronize();
                    cudaFree(h->dist_buf);
                }
                h->dist_buf = nullptr;
                h->dist_buf_bytes = 0;
                if (cudaMalloc(&h->dist_buf, need) != cudaSuccess) {
                    cudaGetLastError();
                    return OZIMMU_ERR_WORKSPACE;
                }
                h->dist_buf_bytes = need;
            }
            Bf = static_cast<double *>(h->dist_buf);
        }
    }
    cudaError_t e = cudaSuccess;
    if (!h->comm) e = cudaStreamCreateWithFlags(&h->comm, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_status(e);
    std::vector<cudaEvent_t> ev((size_t)(2 * J + 1), nullptr);
    for (auto &x : ev)
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
    cudaEvent_t ev_start = ev[0], *ev_ready = ev.data() + 1, *ev_recv = ev.data() + 1 + J;
    int launches = 0;
    bool forked = false;
#define OZ_TRY(x) do { if (e == cudaSuccess) e = (x); } while (0)
    mark(h, PH_START);
    // the B-slice buffer may still be read by the previous call's GEMMs on h->stream
    OZ_TRY(cudaEventRecord(ev_start, h->stream));
    OZ_TRY(cudaStreamWaitEvent(h->comm, ev_start, 0));
    // ---- root: slice op(B) chunk by chunk on the second stream ----
    const bool bcontig = transB == OZIMMU_OP_N;
    if (is_root && !fp64 && e == cudaSuccess) {
        OZ_TRY(aux_fork(h));
        forked = e == cudaSuccess;
        int32_t *keys_b = reinterpret_cast<int32_t *>(base + L.keys_b);
        for (int j = 0; j < J && e == cudaSuccess; ++j) {
            const int64_t c0 = dp.cb[j], nc = dp.cb[j + 1] - c0;
            const double *Bj = bcontig ? B + c0 * ldb : B + c0;
            OZ_TRY(launch_split(Bj, ldb, bcontig, nc, k, k_pad, s, w, /*reverse=*/true,
                                b_planes + c0 * k_pad, n * k_pad, EB + c0, keys_b, sms, h->aux,
                                &launches));
            OZ_TRY(cudaEventRecord(ev_ready[j], h->aux));
        }
    }
    // ---- every rank: one group of broadcasts per chunk on the collective stream ----
    for (int j = 0; j < J && e == cudaSuccess; ++j) {
        const int64_t c0 = dp.cb[j], nc = dp.cb[j + 1] - c0;
        if (is_root && !fp64) OZ_TRY(cudaStreamWaitEvent(h->comm, ev_ready[j], 0));
        if (e != cudaSuccess) break;
        if ((st = tr.begin())) break;
        if (fp64) {
            st = tr.bcast(Bf + c0 * k, sizeof(double) * (size_t)(nc * k), root, h->comm);
        } else {
            for (int p = 0; p < s && !st; ++p)
                st = tr.bcast(b_planes + (int64_t)p * n * k_pad + c0 * k_pad, (size_t)(nc * k_pad),
                              root, h->comm);
            if (!st) st = tr.bcast(EB + c0, sizeof(int32_t) * (size_t)nc, root, h->comm);
        }
        const ozimmu_status_t st2 = tr.end();
        if (!st) st = st2;
        if (st) break;
        OZ_TRY(cudaEventRecord(ev_recv[j], h->comm));
    }
    // ---- this rank's rows of op(A), then the GEMMs as their chunks arrive ----
    if (e == cudaSuccess && !st && m_loc > 0) {
        OZ_TRY(slice_a(h, transA, m_loc, k, k_pad, A, lda, s, w, a_planes, EA,
                       reinterpret_cast<int32_t *>(base + L.keys), &launches));
        mark(h, PH_A);
        int32_t *keys_b = reinterpret_cast<int32_t *>(base + L.keys_b);
        const int G = (int)dp.gb.size() - 1;
        for (int g = 0; g < G && e == cudaSuccess; ++g) {
            const int j0 = dp.gb[g], j1 = dp.gb[g + 1];
            const int64_t c0 = dp.cb[j0], nc = dp.cb[j1] - c0;
            if (fp64) {  // slice the received FP64 chunks of this launch on this rank
                for (int j = j0; j < j1 && e == cudaSuccess; ++j) {
                    const int64_t d0 = dp.cb[j], dn = dp.cb[j + 1] - d0;
                    OZ_TRY(cudaStreamWaitEvent(h->stream, ev_recv[j], 0));
                    OZ_TRY(launch_split(Bf + d0 * k, k, true, dn, k, k_pad, s, w, true,
                                        b_planes + d0 * k_pad, n * k_pad, EB + d0, keys_b, sms,
                                        h->stream, &launches));
                }
            } else {
                OZ_TRY(cudaStreamWaitEvent(h->stream, ev_recv[j1 - 1], 0));
            }
            if (g == 0) mark(h, PH_GEMM0);
            // broadcasts still in flight after this launch: leave SMs to the collective
            GemmPlan gp;
            if (!plan_gemm(s, w, m_loc, nc, k_pad, j1 < J ? capped : sms, &gp)) {
                if (e == cudaSuccess) e = cudaErrorInvalidValue;
                break;
            }
            OZ_TRY(fused_gemm(h, gp, m_loc, nc, k_pad, s, w, a_planes, EA, b_planes + c0 * k_pad,
                              EB + c0, n, alpha, beta, C + c0 * ldc, ldc,
                              reinterpret_cast<int64_t *>(base + L.scratch),
                              reinterpret_cast<unsigned int *>(base + L.sync), &launches));
        }
    }
    // join: the caller's stream covers the broadcasts (and the root's slicing)
    if (J > 0 && ev_recv[J - 1] && e == cudaSuccess && !st)
        OZ_TRY(cudaStreamWaitEvent(h->stream, ev_recv[J - 1], 0));
    if (forked) {
        const cudaError_t ej = aux_join(h);
        if (e == cudaSuccess) e = ej;
    }
    mark(h, PH_B, h->comm);
    if (m_loc <= 0) {
        mark(h, PH_A);
        mark(h, PH_GEMM0);
    }
    mark(h, PH_GEMM1);
    mark_done(h);
#undef OZ_TRY
    for (auto &x : ev)
        if (x) cudaEventDestroy(x);
    if (st) return st;
    if (e != cudaSuccess) return cuda_status(e);
    fill_report(h, s, w, m_loc, n, k, &gp_full, launches,
                (int64_t)s * m_loc * k_pad + (is_root ? (int64_t)s * n * k_pad : 0));
    return OZIMMU_SUCCESS;
}

// Validation shared by both entry points; returns SUCCESS with *done = true for the BLAS quick
// returns handled here (identical on every rank: they depend on the shared arguments only).
ozimmu_status_t dist_check(ozimmu_handle_t h, int rank, int root, int nranks, ozimmu_op_t transA,
                           ozimmu_op_t transB, int64_t m_loc, int64_t n, int64_t k,
                           const double *alpha, const double *A, int64_t lda, const double *B,
                           int64_t ldb, const double *beta, double *C, int64_t ldc, int s,
                           bool *done) {
    *done = false;
    ozimmu_status_t st = check_common(h, transA, m_loc, n, k, alpha, A, lda, beta, C, ldc, s);
    if (st) return st;
    if (!valid_op(transB)) return OZIMMU_ERR_INVALID_VALUE;
    if (root < 0 || root >= nranks || rank < 0 || rank >= nranks) return OZIMMU_ERR_INVALID_VALUE;
    if (s == 0) return OZIMMU_ERR_UNSUPPORTED;  // AUTO would need an all-reduce of A's statistics
    if (rank == root && n > 0 && k > 0 && *alpha != 0.0) {
        const int64_t brows = transB == OZIMMU_OP_N ? k : n;
        if (!B || ldb < (brows > 1 ? brows : 1)) return OZIMMU_ERR_INVALID_VALUE;
    } else if (ldb < 1) {
        return OZIMMU_ERR_INVALID_VALUE;
    }
    if (cudaSetDevice(h->device) != cudaSuccess) return OZIMMU_ERR_CUDA;
    if (n == 0) {
        fill_report(h, 0, 0, m_loc, n, k, nullptr, 0, 0);
        *done = true;
        return OZIMMU_SUCCESS;
    }
    if (*alpha == 0.0 || k == 0) {  // C = beta C on every rank, nothing is broadcast
        *done = true;
        return m_loc > 0 ? scale_only(h, m_loc, n, *beta, C, ldc) : OZIMMU_SUCCESS;
    }
    return OZIMMU_SUCCESS;
}

}  // namespace

extern "C" {

ozimmu_status_t ozimmu_nccl_get_unique_id(void *id_out) {
    if (!id_out) return OZIMMU_ERR_INVALID_VALUE;
    Nccl &N = nccl();
    if (!N.ok) return OZIMMU_ERR_NCCL;
    ncclUniqueId id;
    if (N.GetUniqueId(&id) != ncclSuccess) return OZIMMU_ERR_NCCL;
    static_assert(sizeof(ncclUniqueId) == OZIMMU_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
    memcpy(id_out, &id, sizeof(id));
    return OZIMMU_SUCCESS;
}

ozimmu_status_t ozimmu_nccl_comm_init(void **comm_out, int nranks, const void *id, int rank,
                                      int device, int max_ctas) {
    if (!comm_out || !id || nranks < 1 || rank < 0 || rank >= nranks || max_ctas < 0)
        return OZIMMU_ERR_INVALID_VALUE;
    *comm_out = nullptr;
    Nccl &N = nccl();
    if (!N.ok) return OZIMMU_ERR_NCCL;
    if (cudaSetDevice(device) != cudaSuccess) {
        cudaGetLastError();
        return OZIMMU_ERR_CUDA;
    }
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    ncclResult_t r;
    if (max_ctas > 0 && N.CommInitRankConfig) {
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        cfg.maxCTAs = max_ctas;
        cfg.minCTAs = 1;
        r = N.CommInitRankConfig(&c, nranks, uid, rank, &cfg);
    } else {
        r = N.CommInitRank(&c, nranks, uid, rank);
    }
    if (r != ncclSuccess) return OZIMMU_ERR_NCCL;
    *comm_out = c;
    return OZIMMU_SUCCESS;
}

ozimmu_status_t ozimmu_nccl_comm_destroy(void *comm) {
    if (!comm) return OZIMMU_SUCCESS;
    Nccl &N = nccl();
    if (!N.ok) return OZIMMU_ERR_NCCL;
    return N.CommDestroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? OZIMMU_SUCCESS
                                                                       : OZIMMU_ERR_NCCL;
}

ozimmu_status_t ozimmu_set_dist(ozimmu_handle_t h, int chunk_cols, int reserve_sms, int bcast_fp64) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (chunk_cols < 0 || reserve_sms < 0 || (bcast_fp64 != 0 && bcast_fp64 != 1))
        return OZIMMU_ERR_INVALID_VALUE;
    h->dist_chunk_cols = chunk_cols;
    h->dist_reserve_sms = reserve_sms;
    h->dist_bcast_fp64 = bcast_fp64;
    return OZIMMU_SUCCESS;
}

ozimmu_status_t ozimmu_dgemm_nccl(ozimmu_handle_t h, void *comm, int root, ozimmu_op_t transA,
                                  ozimmu_op_t transB, int64_t m_local, int64_t n, int64_t k,
                                  const double *alpha, const double *A_local, int64_t lda,
                                  const double *B, int64_t ldb, const double *beta,
                                  double *C_local, int64_t ldc, int num_slices) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (!comm) return OZIMMU_ERR_INVALID_VALUE;
    Nccl &N = nccl();
    if (!N.ok) return OZIMMU_ERR_NCCL;
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    int rank = 0, nranks = 0;
    if (N.CommUserRank(c, &rank) != ncclSuccess || N.CommCount(c, &nranks) != ncclSuccess)
        return OZIMMU_ERR_NCCL;
    bool done = false;
    ozimmu_status_t st = dist_check(h, rank, root, nranks, transA, transB, m_local, n, k, alpha,
                                    A_local, lda, B, ldb, beta, C_local, ldc, num_slices, &done);
    if (st || done) return st;
    NcclTransport tr(c);
    return dist_core(h, tr, rank, root, transA, transB, m_local, n, k, *alpha, A_local, lda, B,
                     ldb, *beta, C_local, ldc, num_slices);
}

ozimmu_status_t ozimmu_dgemm_bcast(ozimmu_handle_t h, ozimmu_bcast_fn fn, void *ctx, int rank,
                                   int nranks, int root, ozimmu_op_t transA, ozimmu_op_t transB,
                                   int64_t m_local, int64_t n, int64_t k, const double *alpha,
                                   const double *A_local, int64_t lda, const double *B,
                                   int64_t ldb, const double *beta, double *C_local, int64_t ldc,
                                   int num_slices) {
    if (!h) return OZIMMU_ERR_NOT_INITIALIZED;
    if (!fn) return OZIMMU_ERR_INVALID_VALUE;
    bool done = false;
    ozimmu_status_t st = dist_check(h, rank, root, nranks, transA, transB, m_local, n, k, alpha,
                                    A_local, lda, B, ldb, beta, C_local, ldc, num_slices, &done);
    if (st || done) return st;
    FnTransport tr(fn, ctx);
    return dist_core(h, tr, rank, root, transA, transB, m_local, n, k, *alpha, A_local, lda, B,
                     ldb, *beta, C_local, ldc, num_slices);
}

}  // extern "C"
