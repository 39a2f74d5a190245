// Read-bandwidth ceilings on the B200 for the row-pass access pattern
// (exploration tool, not part of the product).  Prints GB/s for:
//   copy      : cudaMemcpy D2D (read+write bytes)
//   ldg128    : grid-stride 16-byte loads, sum reduction (read only)
//   tma(S,NS,G): per-CTA ring of NS stages of S bytes filled by cp.async.bulk,
//              G CTAs per SM, each CTA streams a strided list of chunks.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bwtest tools/bwtest.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void ldg128(const double2* __restrict__ x, size_t n, double* out) {
    double2 acc = {0, 0};
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const double2 v = __ldg(x + i);
        acc.x += v.x;
        acc.y += v.y;
    }
    if (acc.x == 12345.0) out[0] = acc.y;
}

__global__ void tma_stream(const char* __restrict__ base, size_t nchunks, uint32_t chunk, int NS, double* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + size_t(NS) * chunk);
    const int t = threadIdx.x;
    if (t == 0)
        for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bars + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const size_t g = blockIdx.x, ng = gridDim.x;
    size_t issued = 0, q = 0;
    auto issue = [&](size_t item, int st) {
        if (t == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bars + st)), "r"(chunk) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             sa(sm + size_t(st) * chunk)),
                         "l"(base + item * chunk), "r"(chunk), "r"(sa(bars + st))
                         : "memory");
        }
    };
    for (int s = 0; s < NS && g + issued * ng < nchunks; ++s, ++issued) issue(g + issued * ng, s);
    double acc = 0;
    for (size_t item = g; item < nchunks; item += ng, ++q) {
        const int st = int(q % NS);
        const uint32_t ph = uint32_t((q / NS) & 1);
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(ok)
                         : "r"(sa(bars + st)), "r"(ph)
                         : "memory");
        const double* d = reinterpret_cast<const double*>(sm + size_t(st) * chunk);
        acc += d[t];
        __syncthreads();
        if (g + issued * ng < nchunks) {
            if (t == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(g + issued * ng, st);
            ++issued;
        }
    }
    if (acc == 12345.0) out[0] = acc;
}

int main() {
    const size_t bytes = size_t(3) << 30;
    char* buf;
    char* buf2;
    double* out;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&buf2, bytes);
    cudaMalloc(&out, 64);
    cudaMemset(buf, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](auto fn, int reps) {
        fn();
        cudaEventRecord(e0);
        for (int i = 0; i < reps; ++i) fn();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        return ms / reps * 1e-3;
    };
    double t = timeit([&] { cudaMemcpy(buf2, buf, bytes, cudaMemcpyDeviceToDevice); }, 5);
    printf("copy          %8.1f GB/s (r+w)\n", 2.0 * bytes / t / 1e9);
    for (int tpb : {256, 512, 1024}) {
        t = timeit([&] { ldg128<<<sms * 4, tpb>>>((const double2*)buf, bytes / 16, out); }, 5);
        printf("ldg128 tpb=%4d %8.1f GB/s\n", tpb, bytes / t / 1e9);
    }
    cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    for (uint32_t chunk : {5840u, 11680u, 23360u, 40880u}) {
        for (int NS : {2, 3, 4, 6, 8}) {
            const size_t smem = size_t(NS) * chunk + NS * 8;
            if (smem > 227 * 1024) continue;
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tma_stream, 32, smem);
            if (occ < 1) continue;
            const size_t nchunks = bytes / chunk;
            for (int per : {1, 2, occ}) {
                if (per > occ) continue;
                t = timeit([&] { tma_stream<<<sms * per, 32, smem>>>(buf, nchunks, chunk, NS, out); }, 5);
                printf("tma chunk=%6u NS=%d ctas/sm=%2d (occ %2d) %8.1f GB/s  inflight/SM=%6.1f KB\n", chunk, NS, per,
                       occ, nchunks * double(chunk) / t / 1e9, per * NS * chunk / 1024.0);
            }
        }
    }
    cudaError_t err = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(err));
    return 0;
}
