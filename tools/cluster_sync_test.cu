// Cost of a thread-block-cluster barrier on the B200 (16 CTAs x 256 threads,
// non-portable cluster size) vs a CTA barrier: N iterations, clock64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_sync_test tools/cluster_sync_test.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_cluster(long long* out, int iters, int mode) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (mode == 0)
            asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        else
            __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[mode] = (t1 - t0) / iters;
}

int main() {
    long long* out;
    cudaMallocManaged(&out, 16);
    cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int csize : {2, 8, 16}) {
        for (int mode = 0; mode < 2; ++mode) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(csize);
            cfg.blockDim = dim3(256);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = csize;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_cluster, out, 2000, mode);
            cudaDeviceSynchronize();
            printf("cluster %2d %s: %lld cycles per barrier (%s)\n", csize, mode ? "syncthreads" : "cluster.sync",
                   out[mode], cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
