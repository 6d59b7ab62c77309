// cublas_shim.cpp -- NEXT row f3: transparent replacement of cuBLAS double-precision GEMMs by
// the INT8 Ozaki scheme, as the paper did for its quantum-circuit simulation:
// "Intercepting cuBLAS double-precision GEMM function calls and executing INT8-AUTO instead.
// We use an environmental variable LD_PRELOAD to realize it."
//
//   LD_PRELOAD=.../libozimmu_cublas_shim.so  <application>
//
// Interposed symbols: cublasDgemm_v2, cublasZgemm_v2, cublasDgemmStridedBatched,
// cublasZgemmStridedBatched.  Calls are executed by libozimmu on the cuBLAS handle's stream
// with host-pointer alpha/beta; everything else (device pointer mode, OZIMMU_SHIM_DISABLE=1,
// an ozimmu error) is forwarded unchanged to the real cuBLAS function (RTLD_NEXT).
// Environment: OZIMMU_SHIM_SLICES (default 0 = INT8-AUTO), OZIMMU_SHIM_AUTO = acc (default:
// the accuracy-targeted rule, reading A18, tau = OZIMMU_SHIM_AUTO_TAU, default 1) or loss (the
// paper's rule, T = OZIMMU_SHIM_AUTO_T, default 0), OZIMMU_SHIM_SMAX (default 18),
// OZIMMU_SHIM_LOG=1 (one stderr line per intercepted call).  A call that falls through to
// cuBLAS is counted (ozimmu_shim_counters) and reported on stderr the first time, so a silent
// degradation to FP64 cuBLAS cannot go unnoticed.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "ozimmu.h"

namespace {

struct State {
    std::mutex mu;
    ozimmu_handle_t h[64] = {};
    int slices = 0;
    bool auto_loss = false;
    double auto_T = 0.0, auto_tau = 1.0;
    int s_max = 18;
    bool disabled = false;
    bool log = false;
    std::atomic<long long> intercepted{0}, fell_through{0};
    State() {
        const char *e;
        if ((e = getenv("OZIMMU_SHIM_SLICES"))) slices = atoi(e);
        if ((e = getenv("OZIMMU_SHIM_AUTO"))) auto_loss = strcmp(e, "loss") == 0;
        if ((e = getenv("OZIMMU_SHIM_AUTO_T"))) auto_T = atof(e);
        if ((e = getenv("OZIMMU_SHIM_AUTO_TAU"))) auto_tau = atof(e);
        if ((e = getenv("OZIMMU_SHIM_SMAX"))) s_max = atoi(e);
        disabled = getenv("OZIMMU_SHIM_DISABLE") != nullptr;
        log = getenv("OZIMMU_SHIM_LOG") != nullptr;
    }
};

State &state() {
    static State s;
    return s;
}

// The real cuBLAS entry point.  RTLD_NEXT covers libcublas linked into the global scope;
// applications that dlopen() cuBLAS with RTLD_LOCAL (Python extension modules) are reached
// through the already-loaded library's soname.
template <typename F>
F real(const char *name) {
    static_assert(sizeof(F) == sizeof(void *), "function pointer");
    void *p = dlsym(RTLD_NEXT, name);
    if (!p) {
        void *lib = dlopen("libcublas.so.12", RTLD_NOW | RTLD_NOLOAD);
        if (!lib) lib = dlopen("libcublas.so", RTLD_NOW | RTLD_NOLOAD);
        if (lib) p = dlsym(lib, name);
    }
    return reinterpret_cast<F>(p);
}

// A cuBLAS call routed to libozimmu: holds the shim's lock for the whole call, with the
// per-device handle bound to the cuBLAS handle's stream inside that critical section (so no
// other thread can re-bind it to another stream between set_stream and the computation).
struct Route {
    std::unique_lock<std::mutex> lock;
    ozimmu_handle_t h = nullptr;
    const char *why = nullptr;  // reason for falling through (h == nullptr)
};

void route(cublasHandle_t ch, Route &r) {
    State &S = state();
    if (S.disabled) {
        r.why = "OZIMMU_SHIM_DISABLE";
        return;
    }
    using GetMode = cublasStatus_t (*)(cublasHandle_t, cublasPointerMode_t *);
    using GetStream = cublasStatus_t (*)(cublasHandle_t, cudaStream_t *);
    static GetMode get_mode = real<GetMode>("cublasGetPointerMode_v2");
    static GetStream get_stream = real<GetStream>("cublasGetStream_v2");
    if (!get_mode || !get_stream) {
        r.why = "cuBLAS query entry points not found";
        return;
    }
    cublasPointerMode_t mode;
    if (get_mode(ch, &mode) != CUBLAS_STATUS_SUCCESS || mode != CUBLAS_POINTER_MODE_HOST) {
        r.why = "device pointer mode (alpha/beta on the device)";
        return;
    }
    cudaStream_t stream;
    if (get_stream(ch, &stream) != CUBLAS_STATUS_SUCCESS) {
        r.why = "cublasGetStream failed";
        return;
    }
    // the device of the current context, through the driver API the application already
    // loaded (the shim links no CUDA runtime of its own)
    using CtxGetDevice = int (*)(int *);
    static CtxGetDevice ctx_dev = [] {
        void *lib = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
        if (!lib) lib = dlopen("libcuda.so.1", RTLD_NOW);
        return lib ? reinterpret_cast<CtxGetDevice>(dlsym(lib, "cuCtxGetDevice")) : nullptr;
    }();
    int dev = 0;
    if (!ctx_dev || ctx_dev(&dev) != 0 || dev < 0 || dev >= 64) {
        r.why = "no current CUDA device";
        return;
    }
    r.lock = std::unique_lock<std::mutex>(S.mu);
    if (!S.h[dev]) {
        if (ozimmu_create(&S.h[dev], dev) != OZIMMU_SUCCESS) {
            S.h[dev] = nullptr;
            r.why = "ozimmu_create failed";
            return;
        }
        if (S.auto_loss)
            ozimmu_set_auto(S.h[dev], S.auto_T, S.s_max);
        else
            ozimmu_set_auto_accuracy(S.h[dev], S.auto_tau, S.s_max);
    }
    ozimmu_set_stream(S.h[dev], stream);
    r.h = S.h[dev];
}

// Count the outcome of a routed call; a fall-through is reported on stderr the first time.
bool done(const char *fn, Route &r, ozimmu_status_t st) {
    State &S = state();
    if (r.h && st == OZIMMU_SUCCESS) {
        S.intercepted.fetch_add(1);
        return true;
    }
    const long long nth = S.fell_through.fetch_add(1);
    if ((nth == 0 && !S.disabled) || S.log)
        fprintf(stderr, "[ozimmu shim] WARNING %s ran on cuBLAS FP64 instead: %s\n", fn,
                r.h ? ozimmu_status_string(st) : r.why);
    return false;
}

ozimmu_op_t op(cublasOperation_t t) {
    return t == CUBLAS_OP_N ? OZIMMU_OP_N : (t == CUBLAS_OP_T ? OZIMMU_OP_T : OZIMMU_OP_C);
}

char op_char(cublasOperation_t t) { return t == CUBLAS_OP_N ? 'N' : (t == CUBLAS_OP_T ? 'T' : 'C'); }

void log_call(const char *fn, cublasOperation_t ta, cublasOperation_t tb, int m, int n, int k,
              long batch, ozimmu_status_t st, ozimmu_handle_t h) {
    if (!state().log) return;
    ozimmu_report_t r{};
    ozimmu_get_report(h, &r);
    fprintf(stderr, "[ozimmu shim] %s ta=%c tb=%c m=%d n=%d k=%d batch=%ld -> %s (s=%d)\n", fn,
            op_char(ta), op_char(tb), m, n, k, batch, ozimmu_status_string(st), r.num_slices);
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) cublasStatus_t cublasDgemm_v2(
    cublasHandle_t handle, cublasOperation_t transa, cublasOperation_t transb, int m, int n, int k,
    const double *alpha, const double *A, int lda, const double *B, int ldb, const double *beta,
    double *C, int ldc) {
    using Fn = cublasStatus_t (*)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int,
                                  int, const double *, const double *, int, const double *, int,
                                  const double *, double *, int);
    static Fn next = real<Fn>("cublasDgemm_v2");
    Route r;
    route(handle, r);
    ozimmu_status_t st = OZIMMU_ERR_NOT_INITIALIZED;
    if (r.h) {
        st = ozimmu_dgemm(r.h, op(transa), op(transb), m, n, k, alpha, A, lda, B, ldb, beta, C,
                          ldc, state().slices);
        log_call("cublasDgemm_v2", transa, transb, m, n, k, 1, st, r.h);
    }
    if (done("cublasDgemm_v2", r, st)) return CUBLAS_STATUS_SUCCESS;
    r = Route();
    return next ? next(handle, transa, transb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc)
                : CUBLAS_STATUS_NOT_INITIALIZED;
}

__attribute__((visibility("default"))) cublasStatus_t cublasZgemm_v2(
    cublasHandle_t handle, cublasOperation_t transa, cublasOperation_t transb, int m, int n, int k,
    const cuDoubleComplex *alpha, const cuDoubleComplex *A, int lda, const cuDoubleComplex *B,
    int ldb, const cuDoubleComplex *beta, cuDoubleComplex *C, int ldc) {
    using Fn = cublasStatus_t (*)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int,
                                  int, const cuDoubleComplex *, const cuDoubleComplex *, int,
                                  const cuDoubleComplex *, int, const cuDoubleComplex *,
                                  cuDoubleComplex *, int);
    static Fn next = real<Fn>("cublasZgemm_v2");
    Route r;
    route(handle, r);
    ozimmu_status_t st = OZIMMU_ERR_NOT_INITIALIZED;
    if (r.h) {
        st = ozimmu_zgemm(
            r.h, op(transa), op(transb), m, n, k, reinterpret_cast<const double *>(alpha),
            reinterpret_cast<const double *>(A), lda, reinterpret_cast<const double *>(B), ldb,
            reinterpret_cast<const double *>(beta), reinterpret_cast<double *>(C), ldc,
            state().slices);
        log_call("cublasZgemm_v2", transa, transb, m, n, k, 1, st, r.h);
    }
    if (done("cublasZgemm_v2", r, st)) return CUBLAS_STATUS_SUCCESS;
    r = Route();
    return next ? next(handle, transa, transb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc)
                : CUBLAS_STATUS_NOT_INITIALIZED;
}

__attribute__((visibility("default"))) cublasStatus_t cublasDgemmStridedBatched(
    cublasHandle_t handle, cublasOperation_t transa, cublasOperation_t transb, int m, int n, int k,
    const double *alpha, const double *A, int lda, long long strideA, const double *B, int ldb,
    long long strideB, const double *beta, double *C, int ldc, long long strideC, int batch) {
    using Fn = cublasStatus_t (*)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int,
                                  int, const double *, const double *, int, long long,
                                  const double *, int, long long, const double *, double *, int,
                                  long long, int);
    static Fn next = real<Fn>("cublasDgemmStridedBatched");
    Route r;
    route(handle, r);
    ozimmu_status_t st = OZIMMU_ERR_NOT_INITIALIZED;
    if (r.h) {
        st = ozimmu_dgemm_strided_batched(
            r.h, op(transa), op(transb), m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C,
            ldc, strideC, batch, state().slices);
        log_call("cublasDgemmStridedBatched", transa, transb, m, n, k, batch, st, r.h);
    }
    if (done("cublasDgemmStridedBatched", r, st)) return CUBLAS_STATUS_SUCCESS;
    r = Route();
    return next ? next(handle, transa, transb, m, n, k, alpha, A, lda, strideA, B, ldb, strideB,
                       beta, C, ldc, strideC, batch)
                : CUBLAS_STATUS_NOT_INITIALIZED;
}

__attribute__((visibility("default"))) cublasStatus_t cublasZgemmStridedBatched(
    cublasHandle_t handle, cublasOperation_t transa, cublasOperation_t transb, int m, int n, int k,
    const cuDoubleComplex *alpha, const cuDoubleComplex *A, int lda, long long strideA,
    const cuDoubleComplex *B, int ldb, long long strideB, const cuDoubleComplex *beta,
    cuDoubleComplex *C, int ldc, long long strideC, int batch) {
    using Fn = cublasStatus_t (*)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int,
                                  int, const cuDoubleComplex *, const cuDoubleComplex *, int,
                                  long long, const cuDoubleComplex *, int, long long,
                                  const cuDoubleComplex *, cuDoubleComplex *, int, long long, int);
    static Fn next = real<Fn>("cublasZgemmStridedBatched");
    Route r;
    route(handle, r);
    ozimmu_status_t st = OZIMMU_ERR_NOT_INITIALIZED;
    if (r.h) {
        st = ozimmu_zgemm_strided_batched(
            r.h, op(transa), op(transb), m, n, k, reinterpret_cast<const double *>(alpha),
            reinterpret_cast<const double *>(A), lda, strideA, reinterpret_cast<const double *>(B),
            ldb, strideB, reinterpret_cast<const double *>(beta), reinterpret_cast<double *>(C),
            ldc, strideC, batch, state().slices);
        log_call("cublasZgemmStridedBatched", transa, transb, m, n, k, batch, st, r.h);
    }
    if (done("cublasZgemmStridedBatched", r, st)) return CUBLAS_STATUS_SUCCESS;
    r = Route();
    return next ? next(handle, transa, transb, m, n, k, alpha, A, lda, strideA, B, ldb, strideB,
                       beta, C, ldc, strideC, batch)
                : CUBLAS_STATUS_NOT_INITIALIZED;
}

// Calls executed by libozimmu / calls that fell through to cuBLAS, since the process started.
__attribute__((visibility("default"))) void ozimmu_shim_counters(long long *intercepted,
                                                                 long long *fell_through) {
    if (intercepted) *intercepted = state().intercepted.load();
    if (fell_through) *fell_through = state().fell_through.load();
}

}  // extern "C"
