// Shared device/host plumbing for the B200 V-cycle core: error handling that
// maps onto the reference's exception kinds, the launch counter, and the few
// sm_100a PTX primitives the streaming kernels use (mbarrier + 1-D bulk copy
// = TMA `cp.async.bulk`, SASS UBLKCP).
#pragma once

#include <mutex>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/ldgmg_b200.h"

namespace ldgmg_b200 {

/// Exception carrying one of the LDGMG_ERR_* codes; the C ABI converts it to
/// a status + ldgmg_last_error() text.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void require(bool ok, const char* msg) {
    if (!ok) fail(LDGMG_ERR_INVALID_ARGUMENT, msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(LDGMG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define LDGMG_CUDA(call) ::ldgmg_b200::cuda_check((call), #call)

std::atomic<int64_t>& launch_counter();
/// Call right after every kernel launch: counts it and surfaces launch errors.
inline void after_launch(const char* name) {
    launch_counter().fetch_add(1, std::memory_order_relaxed);
    cuda_check(cudaGetLastError(), name);
}

inline int div_up(int64_t a, int64_t b) { return int((a + b - 1) / b); }

/// Programmatic dependent launch (PDL, sm_90+) for the BIG streaming passes
/// (off; the small kernels use it, pdl_small_enabled below): kernels launched with programmatic stream serialization wait for their
/// predecessor (griddepcontrol.wait) only before touching mutable memory, so
/// launch processing and the immutable prologue (barrier init, row pointers,
/// TMA staging of the injection matrices) overlap the previous kernel.
/// Measured on the graph-replayed C2 V-cycle: an early launch_dependents
/// trigger made it 5-10 % SLOWER (dependent CTAs parked on the SMs), the
/// implicit trigger at grid end is neutral (3.295 vs 3.300 ms), so it is off
/// by default and the device-side trigger is not issued.
inline bool pdl_enabled() { return false; }

/// PDL for the SMALL kernels only (split-row passes of the coarse levels,
/// transfers, bottom, projection): they trigger
/// their dependents at entry and issue their immutable prologue (barrier
/// init, TMA of the first row's blocks / injection matrices) before
/// griddepcontrol.wait, so a chain of latency-bound small passes overlaps
/// launch and prologue with its predecessor.  The big streaming passes are
/// launched without the attribute (an early trigger there parked dependent
/// CTAs on the SMs, see pdl_enabled), which also keeps any small kernel from
/// starting before a big pass ends.
inline bool pdl_small_enabled() { return true; }

template <class... KArgs, class... Args>
inline void launch_pdl_small(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                             Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (pdl_enabled() || pdl_small_enabled()) ? 1 : 0;
    cuda_check(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx");
}

template <class... KArgs, class... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cuda_check(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx");
}

/// Raise a kernel's dynamic shared-memory limit only when `bytes` exceeds
/// what was already set on this device: cudaFuncSetAttribute on every launch
/// costs ~15 us of GPU time per following launch (measured), so the
/// attribute is cached per (kernel, device).
template <class K>
inline void ensure_dyn_smem(K* kernel, size_t bytes) {
    struct Entry {
        const void* f;
        int dev;
        size_t bytes;  // current cudaFuncAttributeMaxDynamicSharedMemorySize
    };
    static std::vector<Entry> set;
    static std::mutex mu;  // host threads launch concurrently (SAI batch slots, one context per rank)
    std::lock_guard<std::mutex> lk(mu);
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    const void* f = reinterpret_cast<const void*>(kernel);
    Entry* e = nullptr;
    for (auto& x : set)
        if (x.f == f && x.dev == dev) e = &x;
    if (!e) {  // the default limit is 48 KB minus the kernel's static shared memory
        cudaFuncAttributes fa{};
        cuda_check(cudaFuncGetAttributes(&fa, f), "cudaFuncGetAttributes");
        set.push_back({f, dev, size_t(fa.maxDynamicSharedSizeBytes)});
        e = &set.back();
    }
    if (bytes <= e->bytes) return;
    cuda_check(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)),
               "cudaFuncSetAttribute");
    e->bytes = bytes;
}

/// Pin a kernel's shared-memory carveout to the maximum (once per kernel).
/// The V-cycle alternates the TMA row pass (large carveout) with small
/// kernels; letting the driver pick a smaller carveout for those forces an
/// SM reconfiguration (L1 drain) at every switch, which measured as a
/// ~15 us bubble per small launch on B200.
template <class K>
inline void max_carveout(K* kernel) {
    cuda_check(cudaFuncSetAttribute(reinterpret_cast<const void*>(kernel),
                                             cudaFuncAttributePreferredSharedMemoryCarveout, 100),
                        "carveout");
}

// ------------------------------------------------------------ PTX helpers
#if defined(__CUDACC__)
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
/// arrive + expect `bytes` of async-proxy transactions on the barrier
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    while (!mbar_try_wait(bar, phase)) {
    }
}
/// TMA 1-D bulk copy global -> shared, completion signalled on `bar`.
/// `bytes` must be a multiple of 16, both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
/// PDL device side: let the next kernel in the stream launch now / wait for
/// the previous kernel's completion and memory (no-ops without PDL).
__device__ __forceinline__ void pdl_trigger() {}  // implicit at grid end (see pdl_enabled)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
/// early trigger of the small kernels (no-op when no dependent was launched
/// with programmatic serialization)
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

/// Named barrier over `nthreads` threads (row groups wider than one warp).
__device__ __forceinline__ void group_sync(int id, int nthreads) {
    if (nthreads <= 32)
        __syncwarp();
    else
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

/// Unfused IEEE multiply-add pair: the reference's `s += a * b` compiled for
/// x86-64 without FMA contraction (blockla.hpp:149, smoothers.hpp:508).
__device__ __forceinline__ double madd_rn(double s, double a, double b) {
    return __dadd_rn(s, __dmul_rn(a, b));
}
#endif

}  // namespace ldgmg_b200
