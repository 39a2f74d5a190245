// FP64 dependent-chain latency on the B200 (one warp, clock64):
//   dadd chain, dmul+dadd chain (register operands), dmul+dadd chain with the
//   two operands loaded from shared memory each step, 8 interleaved chains.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_lat tools/fp64_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 1024;

__global__ void lat(double* out, long long* cyc, double a, double b) {
    __shared__ double sm[2 * N + 64];
    for (int i = threadIdx.x; i < 2 * N + 64; i += blockDim.x) sm[i] = 1.0 + 1e-9 * i;
    __syncthreads();
    double s = threadIdx.x;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) s = __dadd_rn(s, a);
    long long t1 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) s = __dadd_rn(s, __dmul_rn(a, b));
    long long t2 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) s = __dadd_rn(s, __dmul_rn(sm[i + threadIdx.x], sm[N + i]));
    long long t3 = clock64();
    double u[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) u[q] = q;
#pragma unroll 4
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int q = 0; q < 8; ++q) u[q] = __dadd_rn(u[q], __dmul_rn(sm[i + q], sm[N + i]));
    }
    long long t4 = clock64();
    for (int q = 0; q < 8; ++q) s += u[q];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0;
        cyc[1] = t2 - t1;
        cyc[2] = t3 - t2;
        cyc[3] = t4 - t3;
    }
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 32 * 8);
    cudaMallocManaged(&cyc, 4 * 8);
    for (int rep = 0; rep < 2; ++rep) {
        lat<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999);
        cudaDeviceSynchronize();
    }
    printf("{\"dadd_chain_cyc_per_op\": %.2f, \"madd_chain_reg\": %.2f, \"madd_chain_smem\": %.2f, "
           "\"madd_8chains_smem_per_step\": %.2f}\n",
           double(cyc[0]) / N, double(cyc[1]) / N, double(cyc[2]) / N, double(cyc[3]) / N);
    return 0;
}
