// Host-side objects behind the C ABI handles.  Device layouts:
//   * BSR values: one block per `blk_stride` doubles (rbs*cbs rounded up to an
//     even count so every block starts 16-byte aligned for TMA bulk copies),
//     block stored COLUMN-major: element (r,c) at c*rbs + r.  Lane r of a row
//     group then reads consecutive shared-memory words at every step c.
//   * ptr/col: identical int32 arrays to the reference BlockCsr.
//   * diagonal factors: V per element as bs columns of stride ld = bs|1
//     (odd, conflict-free for both V^T u and V t), padded to an even count.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <vector>

#include "common.cuh"

namespace ldgmg_b200 {

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int num_sms = 148;
    size_t smem_optin = 227 * 1024;
    // scratch for reductions (device) + pinned host slot
    double* d_red = nullptr;
    double* h_red = nullptr;
    // pinned double buffer for large host->device uploads (h2d_staged)
    unsigned char* pin[2] = {nullptr, nullptr};
    cudaEvent_t pin_ev[2] = {nullptr, nullptr};
    size_t pin_bytes = 0;
};

/// Large pageable host -> device copy: threaded memcpy into a pinned double
/// buffer, each slot's DMA overlapping the fill of the other (pageable
/// cudaMemcpy runs at ~2 GB/s on the box; this reaches the PCIe rate).
/// Returns after the copy completed.
void h2d_staged(Ctx& ctx, void* dst, const void* src, size_t bytes);
void ctx_release_staging(Ctx& ctx);

struct LevelProgram;  // setup.hpp
/// Evaluate a deferred-assembly program on the device (assembly_gpu.cu).
std::unique_ptr<struct Bsr> assemble_on_device(Ctx& ctx, const LevelProgram& P);

/// Host<->device copies ordered on the context stream (setup paths; the
/// legacy-stream cudaMemcpy would race with the non-blocking context stream).
inline void h2d(Ctx& ctx, void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    LDGMG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx.stream));
    LDGMG_CUDA(cudaStreamSynchronize(ctx.stream));
}
inline void d2h(Ctx& ctx, void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    LDGMG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx.stream));
    LDGMG_CUDA(cudaStreamSynchronize(ctx.stream));
}

/// Device allocation of the library (devmem.cpp): plain cudaMalloc, or with
/// guard zones checked for out-of-bounds writes (LDGMG_GUARD_BYTES).
void* dev_alloc(size_t bytes);
void dev_free(void* p);
int64_t dev_guard_check();  // corrupted zones so far (-1: guards off)
int64_t dev_guard_live();

/// Stream-ordered allocation scope: DevBufs allocated on this thread while
/// a scope is alive come from cudaMallocAsync on its stream and go back with
/// cudaFreeAsync (no device-wide synchronisation at free), so independent
/// work on several streams keeps overlapping.  Off under guard zones (the
/// guarded path stays synchronous and checked).
cudaStream_t dev_async_stream();
struct DevAsyncScope {
    cudaStream_t prev;
    explicit DevAsyncScope(cudaStream_t s);
    ~DevAsyncScope();
};

/// RAII device allocation.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t astream = nullptr;  // stream-ordered allocation (DevAsyncScope)
    DevBuf() = default;
    explicit DevBuf(size_t n) { alloc(n); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), astream(o.astream) {
        o.p = nullptr;
        o.bytes = 0;
        o.astream = nullptr;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        release();
        p = o.p;
        bytes = o.bytes;
        astream = o.astream;
        o.p = nullptr;
        o.bytes = 0;
        o.astream = nullptr;
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t n) {
        release();
        bytes = n;
        if (!n) return;
        astream = dev_async_stream();
        if (astream)
            LDGMG_CUDA(cudaMallocAsync(&p, n, astream));
        else
            p = dev_alloc(n);
    }
    void release() {
        if (p) {
            if (astream)
                cudaFreeAsync(p, astream);
            else
                dev_free(p);
        }
        p = nullptr;
        bytes = 0;
        astream = nullptr;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

struct Bsr {
    int brows = 0, bcols = 0, rbs = 0, cbs = 0;
    int64_t nnzb = 0;
    int blk_stride = 0;  // doubles per stored block
    int max_row = 0;     // longest block row (split-row kernel scratch)
    DevBuf ptr, col, val;
    std::vector<int> hptr, hcol;
    std::unique_ptr<Bsr> T;  // lazily built transpose (spmv_transpose, B^T sweeps)
    std::unique_ptr<Bsr> TV; // lazily built transpose VIEW (no value copy)
    // set on a transpose view: values live in tbase->val, block q = tbase block tperm[q]
    const Bsr* tbase = nullptr;
    DevBuf tperm;
    // set on a row-prefix view: the first `brows` rows of vbase, its values
    // read in place (ptr/col are copies of vbase's prefix)
    const Bsr* vbase = nullptr;
    std::unique_ptr<Bsr> mat;  // lazily built explicit copy of a transposed view (bsr_materialize)
    DevBuf dpos;  // lazily built: CSR position of each row's diagonal block (-1: none)
    int64_t device_bytes() const { return int64_t(ptr.bytes + col.bytes + val.bytes); }
};

inline int even_up(int64_t n) { return int((n + 1) & ~int64_t(1)); }

inline void set_max_row(Bsr& A) {
    A.max_row = 0;
    for (int i = 0; i < A.brows; ++i) A.max_row = std::max(A.max_row, A.hptr[i + 1] - A.hptr[i]);
}

/// Upload from the reference layout (row-major blocks) to the device layout.
std::unique_ptr<Bsr> bsr_upload(Ctx& ctx, int brows, int bcols, int rbs, int cbs, const int* ptr,
                                const int* col, const double* val, bool require_sorted = true);
/// out[i] = x block idx[i] (ghost-exchange packing)
void launch_gather_blocks(Ctx& ctx, const double* x, const int* idx, int n, int bs, double* out);
/// Device copy of A with the layout of A^T (used for B^T r, bitwise equal to
/// the reference's scatter order, blockla.hpp:163-175).
const Bsr& bsr_transpose(Ctx& ctx, const Bsr& A);
/// A^T as a VIEW of A's values (CSC index + block permutation, no copy): the
/// streaming row pass reads each stored block transposed.  Same bits as
/// bsr_transpose.  Halves the SAI smoother's memory (B^T sweeps at C5 48^3
/// would otherwise need another 72 GB).
const Bsr& bsr_transpose_view(Ctx& ctx, const Bsr& A);
/// The operator a B^T sweep should use: the view when the streaming kernel
/// reads it conflict-free (LDGMG_TVIEW=0 forces the explicit copy).
const Bsr& bsr_transpose_for_sweep(Ctx& ctx, const Bsr& A);
void bsr_download(Ctx& ctx, const Bsr& A, int* ptr, int* col, double* val);
/// Values of blocks [k0, k0 + nb) from the reference layout (row-major blocks).
void bsr_set_values(Ctx& ctx, Bsr& A, int64_t k0, int64_t nb, const double* val);
/// A new matrix with pattern (ptr, col) whose block q is a device copy of
/// src block src_blocks[q] (rank-local operators cut from a device-assembled
/// global-shaped one, without a host round trip of the values).
std::unique_ptr<Bsr> bsr_gather(Ctx& ctx, const Bsr& src, int brows, int bcols, const int* ptr, const int* col,
                                const int64_t* src_blocks);
/// The first `nrows` block rows of `base` (values shared, not copied).
std::unique_ptr<Bsr> bsr_row_prefix_view(Ctx& ctx, const Bsr& base, int nrows);
/// A general transposed view: block q of the result is block perm[q] of
/// `base` read transposed; (ptr, col) its own pattern.  The distributed B^T
/// of a rank (rows = its columns of B, entries from B's own and ghost rows).
std::unique_ptr<Bsr> bsr_transposed_view(Ctx& ctx, const Bsr& base, int brows, int bcols, const int* ptr,
                                         const int* col, const int* perm);
/// Explicit copy of a view (cached on the view): the split-row kernels of
/// small passes read stored blocks only.
const Bsr& bsr_materialize(Ctx& ctx, const Bsr& view);
/// Values pointer the kernels read for A (its own, or the viewed base's).
inline const double* bsr_values(const Bsr& A) {
    return A.tbase ? A.tbase->val.as<double>() : A.vbase ? A.vbase->val.as<double>() : A.val.as<double>();
}

/// Per-element factors of the block-diagonal solve (smoothers.hpp:464-494).
struct DiagFactors {
    int n = 0, bs = 0, ld = 0, vstride = 0;
    DevBuf V, lambda, scale, lmax;  // lmax: max |lambda| per element
};

// ---- streaming row-pass kernels (bsr_kernels.cu) ---------------------------
enum RowMode { MODE_SPMV = 0, MODE_RESIDUAL = 1, MODE_ADD = 2, MODE_RELAX = 3 };

struct RowPass {
    const Bsr* A = nullptr;
    int mode = MODE_SPMV;
    const double* x = nullptr;   // gathered vector (snapshot for Jacobi)
    const double* b = nullptr;   // RESIDUAL / RELAX
    const double* xe = nullptr;  // RELAX: x_e for the damped blend (live x)
    double* y = nullptr;         // output
    const int* rows = nullptr;   // optional row list (colour phase); nullptr = all rows
    int nrows = 0;
    const DiagFactors* F = nullptr;  // RELAX
    const int* part = nullptr;       // RELAX, processor-block GS: partition of each element
    const double* x_alt = nullptr;   //   neighbours in other partitions read from here
    double omega = 1.0;
    double kernel_tol = 1e-12;
};
void launch_rowpass(Ctx& ctx, const RowPass& p);

// ---- transfers / dense / BLAS-1 (vec_kernels.cu) ---------------------------
struct Transfer {
    int n_fine = 0, n_coarse = 0, dim = 2, bss = 0, ncomp = 1, bs = 0;
    int max_children = 0;
    DevBuf parent, orth, child_ptr, child_list, K;
    DevBuf child_orth;  // orth[child_list[q]] in child-list order (restrict_flat_kernel)
    DevBuf Kt;          // K_o transposed, (j, i) at j*bss + i (prolong_flat_kernel)
    bool regular = false;  // every parent p has 2^dim children 2^dim p + o in orthant order o
    std::vector<int> hparent, horth;
};
/// `zero_xc` (optional): also zero this coarse vector (the V-cycle's x_{l+1}).
void launch_restrict(Ctx& ctx, const Transfer& T, const double* rf, double* rc, double* zero_xc = nullptr);
void launch_prolong_add(Ctx& ctx, const Transfer& T, const double* xc, double* xf);

struct DenseEig {  // bottom pseudoinverse: V both layouts + lambda + lmax
    int n = 0;
    DevBuf Vc, Vr, lambda, t;
    double lmax = 0.0;
};
void launch_pinv_apply(Ctx& ctx, const DenseEig& E, double tol, const double* b, double* x);

/// v -= (v.k) k for the constant-mode kernel vectors (multigrid.hpp:243-245).
/// `offs` = entries of the mode-0 coefficient of each kernel component.
/// `scratch` (>= 256 * ncomp doubles) enables the multi-CTA fast path.
void launch_project_constants(Ctx& ctx, double* v, int N, int bs, const int* comp_offsets,
                              int ncomp, double kval, bool strict_order, double* scratch = nullptr);
void launch_project_partials_slice(Ctx& ctx, const double* v, int N, int r0, int r1, int bs, const int* offs,
                                   int ncomp, double kval, double* part);
void launch_project_apply_slice(Ctx& ctx, double* v, int N, int r0, int r1, int bs, const int* offs, int ncomp,
                                double kval, const double* part);
void launch_axpy(Ctx& ctx, int64_t n, double alpha, const double* x, double* y);
/// deterministic fixed-tree dot (partials per CTA, ascending final sum)
void launch_dot(Ctx& ctx, int64_t n, const double* a, const double* b, double* d_out);
void launch_fill(Ctx& ctx, int64_t n, double v, double* y);

}  // namespace ldgmg_b200
