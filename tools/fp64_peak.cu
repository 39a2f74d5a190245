// FP64 peaks on this B200 (MEASURED_PEAKS.json has none): DFMA issue peak of
// the CUDA cores and the cuBLAS DGEMM rate (FP64 tensor cores), for the SAI
// setup's FP64 utilisation.  nvcc -gencode arch=compute_100a,code=sm_100a -lcublas
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cstdio>

__global__ void dfma_kernel(double* out, int iters) {
    double a[8];
    for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * 1e-3 + q;
    const double b = 1.0000001, c = 1e-9;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = fma(a[q], b, c);
    double s = 0;
    for (int q = 0; q < 8; ++q) s += a[q];
    if (s == 1234.5) out[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    dfma_kernel<<<blocks, threads>>>(out, 64);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * double(iters) * blocks * threads;
    printf("{\"dfma_tflops\": %.2f, ", flops / (ms * 1e-3) / 1e12);

    const int n = 8192;
    double *A, *B, *Cm;
    cudaMalloc(&A, sizeof(double) * n * n);
    cudaMalloc(&B, sizeof(double) * n * n);
    cudaMalloc(&Cm, sizeof(double) * n * n);
    cudaMemset(A, 0, sizeof(double) * n * n);
    cudaMemset(B, 0, sizeof(double) * n * n);
    cublasHandle_t h;
    cublasCreate(&h);
    const double one = 1.0, zero = 0.0;
    cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, Cm, n);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, Cm, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("\"dgemm_tflops\": %.2f, \"dgemm_n\": %d, \"sms\": %d}\n", 3 * 2.0 * double(n) * n * n / (ms * 1e-3) / 1e12,
           n, sms);
    return 0;
}
