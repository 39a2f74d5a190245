// Micro-test: cost of staging a 46.7 KB table into shared memory per CTA
// (TMA bulk vs plain loads) for tiny grids.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2412_12506_b200/csrc/common.cuh"
using namespace ldgmg_b200;

__global__ void bulk_stage(const double* K, int nK, double* out) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    __syncthreads();
    if (threadIdx.x == 0) { mbar_arrive_expect_tx(&bar, uint32_t(nK) * 8u); bulk_g2s(sm, K, uint32_t(nK) * 8u, &bar); }
    mbar_wait(&bar, 0);
    if (threadIdx.x == 0) out[blockIdx.x] = sm[nK - 1];
}
__global__ void plain_stage(const double* K, int nK, double* out) {
    extern __shared__ __align__(16) double sm[];
    for (int t = threadIdx.x; t < nK; t += blockDim.x) sm[t] = __ldg(K + t);
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = sm[nK - 1];
}
__global__ void empty_kernel(double* out) { if (threadIdx.x == 0) out[blockIdx.x] = 1.0; }
__global__ void dchain(double* out, int n) {  // dependent madd chain of length n
    double s = threadIdx.x * 1e-3, a = 1.0000001, b = 1e-9;
    for (int i = 0; i < n; ++i) s = __dadd_rn(__dmul_rn(s, a), b);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

int probe_main();
int main() {
    probe_main();
    const int nK = 8 * 27 * 27;
    double *K, *out;
    cudaMalloc(&K, nK * 8); cudaMalloc(&out, 4096 * 8);
    cudaMemset(K, 0, nK * 8);
    cudaFuncSetAttribute(bulk_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    cudaFuncSetAttribute(plain_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto time = [&](const char* name, auto launch) {
        for (int i = 0; i < 10; ++i) launch();
        cudaEventRecord(e0);
        for (int i = 0; i < 200; ++i) launch();
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-28s %8.2f us/launch  (%s)\n", name, ms * 1000 / 200, cudaGetErrorString(cudaGetLastError()));
    };
    for (int g : {1, 8, 296}) {
        printf("grid %d\n", g);
        time("empty", [&] { empty_kernel<<<g, 256>>>(out); });
        time("bulk_stage 46.7KB", [&] { bulk_stage<<<g, 256, nK * 8>>>(K, nK, out); });
        time("plain_stage 46.7KB", [&] { plain_stage<<<g, 256, nK * 8>>>(K, nK, out); });
        time("dchain 216", [&] { dchain<<<g, 32>>>(out, 216); });
        time("dchain 2160", [&] { dchain<<<g, 32>>>(out, 2160); });
    }
}
// ---- FP64 issue-rate probes (1 warp): 8 independent chains, with / without smem operands
__global__ void chains8(double* out, int n, long long* t) {
    double s[8];
    for (int q = 0; q < 8; ++q) s[q] = threadIdx.x * 1e-3 + q;
    const double a = 1.0000001, b = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int q = 0; q < 8; ++q) s[q] = __dadd_rn(__dmul_rn(s[q], a), b);
    long long t1 = clock64();
    double r = 0; for (int q = 0; q < 8; ++q) r += s[q];
    if (threadIdx.x == 0) { out[0] = r; t[0] = t1 - t0; }
}
__global__ void chains8_smem(double* out, int n, long long* t) {
    __shared__ double sh[4 * 32 * 32];
    for (int i = threadIdx.x; i < 4 * 32 * 32; i += blockDim.x) sh[i] = 1.0 + i * 1e-9;
    __syncthreads();
    double s[8];
    for (int q = 0; q < 8; ++q) s[q] = 0.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        double kv[8], xv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) { kv[q] = sh[((q & 3) * 32 + (i & 31)) * 32 + threadIdx.x]; xv[q] = sh[q * 27 + (i & 31)]; }
#pragma unroll
        for (int q = 0; q < 8; ++q) s[q] = __dadd_rn(s[q], __dmul_rn(kv[q], xv[q]));
    }
    long long t1 = clock64();
    double r = 0; for (int q = 0; q < 8; ++q) r += s[q];
    if (threadIdx.x == 0) { out[0] = r; t[0] = t1 - t0; }
}
int probe_main();
int probe_main() {
    double* out; long long* t; cudaMalloc(&out, 64); cudaMalloc(&t, 64);
    long long h;
    chains8<<<1, 32>>>(out, 270, t); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
    printf("8 chains x 270 steps (regs): %lld cycles = %.1f cyc/step\n", h, h / 270.0);
    chains8_smem<<<1, 32>>>(out, 270, t); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
    printf("8 chains x 270 steps (smem operands): %lld cycles = %.1f cyc/step\n", h, h / 270.0);
    return 0;
}
