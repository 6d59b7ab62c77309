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
// Environment: OZIMMU_SHIM_SLICES (default 0 = INT8-AUTO), OZIMMU_SHIM_AUTO_T (default 0),
// OZIMMU_SHIM_LOG=1 (one stderr line per intercepted call).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "ozimmu.h"

namespace {

struct State {
    std::mutex mu;
    ozimmu_handle_t h[64] = {};
    int slices = 0;
    double auto_T = 0.0;
    bool disabled = false;
    bool log = false;
    State() {
        const char *e;
        if ((e = getenv("OZIMMU_SHIM_SLICES"))) slices = atoi(e);
        if ((e = getenv("OZIMMU_SHIM_AUTO_T"))) auto_T = atof(e);
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

// ozimmu handle for the current device, bound to the cuBLAS handle's stream; nullptr if the
// call must go to cuBLAS.
ozimmu_handle_t handle_for(cublasHandle_t ch) {
    State &S = state();
    if (S.disabled) return nullptr;
    using GetMode = cublasStatus_t (*)(cublasHandle_t, cublasPointerMode_t *);
    using GetStream = cublasStatus_t (*)(cublasHandle_t, cudaStream_t *);
    static GetMode get_mode = real<GetMode>("cublasGetPointerMode_v2");
    static GetStream get_stream = real<GetStream>("cublasGetStream_v2");
    if (!get_mode || !get_stream) return nullptr;
    cublasPointerMode_t mode;
    if (get_mode(ch, &mode) != CUBLAS_STATUS_SUCCESS || mode != CUBLAS_POINTER_MODE_HOST)
        return nullptr;
    cudaStream_t stream;
    if (get_stream(ch, &stream) != CUBLAS_STATUS_SUCCESS) return nullptr;
    // the device of the current context, through the driver API the application already
    // loaded (the shim links no CUDA runtime of its own)
    using CtxGetDevice = int (*)(int *);
    static CtxGetDevice ctx_dev = [] {
        void *lib = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
        if (!lib) lib = dlopen("libcuda.so.1", RTLD_NOW);
        return lib ? reinterpret_cast<CtxGetDevice>(dlsym(lib, "cuCtxGetDevice")) : nullptr;
    }();
    int dev = 0;
    if (!ctx_dev || ctx_dev(&dev) != 0 || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lock(S.mu);
    if (!S.h[dev]) {
        if (ozimmu_create(&S.h[dev], dev) != OZIMMU_SUCCESS) {
            S.h[dev] = nullptr;
            return nullptr;
        }
        ozimmu_set_auto(S.h[dev], S.auto_T, 20);
    }
    ozimmu_set_stream(S.h[dev], stream);
    return S.h[dev];
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
    ozimmu_handle_t h = handle_for(handle);
    if (h) {
        std::lock_guard<std::mutex> lock(state().mu);
        ozimmu_status_t st = ozimmu_dgemm(h, op(transa), op(transb), m, n, k, alpha, A, lda, B,
                                          ldb, beta, C, ldc, state().slices);
        log_call("cublasDgemm_v2", transa, transb, m, n, k, 1, st, h);
        if (st == OZIMMU_SUCCESS) return CUBLAS_STATUS_SUCCESS;
    }
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
    ozimmu_handle_t h = handle_for(handle);
    if (h) {
        std::lock_guard<std::mutex> lock(state().mu);
        ozimmu_status_t st = ozimmu_zgemm(
            h, op(transa), op(transb), m, n, k, reinterpret_cast<const double *>(alpha),
            reinterpret_cast<const double *>(A), lda, reinterpret_cast<const double *>(B), ldb,
            reinterpret_cast<const double *>(beta), reinterpret_cast<double *>(C), ldc,
            state().slices);
        log_call("cublasZgemm_v2", transa, transb, m, n, k, 1, st, h);
        if (st == OZIMMU_SUCCESS) return CUBLAS_STATUS_SUCCESS;
    }
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
    ozimmu_handle_t h = handle_for(handle);
    if (h) {
        std::lock_guard<std::mutex> lock(state().mu);
        ozimmu_status_t st = ozimmu_dgemm_strided_batched(
            h, op(transa), op(transb), m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C,
            ldc, strideC, batch, state().slices);
        log_call("cublasDgemmStridedBatched", transa, transb, m, n, k, batch, st, h);
        if (st == OZIMMU_SUCCESS) return CUBLAS_STATUS_SUCCESS;
    }
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
    ozimmu_handle_t h = handle_for(handle);
    if (h) {
        std::lock_guard<std::mutex> lock(state().mu);
        ozimmu_status_t st = ozimmu_zgemm_strided_batched(
            h, op(transa), op(transb), m, n, k, reinterpret_cast<const double *>(alpha),
            reinterpret_cast<const double *>(A), lda, strideA, reinterpret_cast<const double *>(B),
            ldb, strideB, reinterpret_cast<const double *>(beta), reinterpret_cast<double *>(C),
            ldc, strideC, batch, state().slices);
        log_call("cublasZgemmStridedBatched", transa, transb, m, n, k, batch, st, h);
        if (st == OZIMMU_SUCCESS) return CUBLAS_STATUS_SUCCESS;
    }
    return next ? next(handle, transa, transb, m, n, k, alpha, A, lda, strideA, B, ldb, strideB,
                       beta, C, ldc, strideC, batch)
                : CUBLAS_STATUS_NOT_INITIALIZED;
}

}  // extern "C"
