// FP64 pipe throughput on this GPU (development probe): DFMA, I2F.F64.S32, I2F.F64.S64 and
// DMUL rates per SM per clock with 1 and 4 warps per SM sub-partition (independent chains).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_rate tools/fp64_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double *out, int iters, long long *cyc) {
    double a[8];
    int ii[8];
    long long ll[8];
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3 + i; ii[i] = threadIdx.x + i; ll[i] = threadIdx.x * 3 + i; }
    const double b = 1.0000001, c = 1e-9;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) a[i] = fma(a[i], b, c);
            if (OP == 1) { a[i] += (double)ii[i]; ii[i] += 3; }
            if (OP == 2) { a[i] += (double)ll[i]; ll[i] += 3; }
            if (OP == 3) a[i] = a[i] * b;
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    long long *cyc;
    cudaMalloc(&out, sizeof(double) * sms * 1024);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    const int iters = 4096;
    const char *names[4] = {"DFMA", "I2F.F64.S32 + DADD", "I2F.F64.S64 + DADD", "DMUL"};
    for (int op = 0; op < 4; ++op)
        for (int threads : {128, 512}) {
            void (*f)(double *, int, long long *) = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : k<3>;
            f<<<sms, threads>>>(out, iters, cyc);
            cudaDeviceSynchronize();
            long long c = 0;
            cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
            const double ops = (double)threads * iters * 8 * (op == 1 || op == 2 ? 2 : 1);
            printf("%-22s threads/SM %4d: %.2f FP64 ops per SM per clock\n", names[op], threads,
                   ops / (double)c);
        }
    return 0;
}
