// The C ABI (include/ldgmg_b200.h): status codes + thread-local error text,
// opaque handles over the host objects of core.hpp / mg.hpp.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <unordered_map>

#include "core.hpp"
#include "formats.hpp"
#include "mg.hpp"
#include "dgemm.hpp"
#include "host_eig.hpp"
#include "krylov.hpp"
#include "setup.hpp"

using namespace ldgmg_b200;

struct ldgmg_ctx : Ctx {};
struct ldgmg_bsr : Bsr {};
struct ldgmg_smoother {
    Smoother s;
};
struct ldgmg_transfer {
    std::unique_ptr<Transfer> t;
};
struct ldgmg_mg {
    Mg m;
};
struct ldgmg_problem {
    Problem p;
};

namespace ldgmg_b200 {
std::atomic<int64_t>& launch_counter() {
    static std::atomic<int64_t> c{0};
    return c;
}
}  // namespace ldgmg_b200

namespace {

thread_local std::string g_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return LDGMG_OK;
    } catch (const Error& e) {
        g_error = e.what();
        return e.code;
    } catch (const std::invalid_argument& e) {
        g_error = e.what();
        return LDGMG_ERR_INVALID_ARGUMENT;
    } catch (const std::logic_error& e) {
        g_error = e.what();
        return LDGMG_ERR_LOGIC;
    } catch (const std::bad_alloc&) {
        g_error = "host allocation failed";
        return LDGMG_ERR_RUNTIME;
    } catch (const std::exception& e) {
        g_error = e.what();
        return LDGMG_ERR_RUNTIME;
    }
}

void need(const void* p, const char* what) {
    if (!p) fail(LDGMG_ERR_INVALID_ARGUMENT, std::string(what) + ": null argument");
}

void bind(Ctx& c) { LDGMG_CUDA(cudaSetDevice(c.device)); }

Bsr* own_bsr(std::unique_ptr<Bsr> b) {
    // ldgmg_bsr is layout-identical to Bsr (empty derived struct)
    auto* h = new ldgmg_bsr();
    static_cast<Bsr&>(*h) = std::move(*b);
    return h;
}

}  // namespace

extern "C" {

const char* ldgmg_last_error(void) { return g_error.c_str(); }
int ldgmg_abi_version(void) { return LDGMG_B200_ABI_VERSION; }
int64_t ldgmg_launch_count(void) { return launch_counter().load(); }

int ldgmg_ctx_create(int device, ldgmg_ctx** out) {
    return guarded([&] {
        need(out, "ldgmg_ctx_create");
        int n = 0;
        const cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess || n == 0)
            fail(LDGMG_ERR_CUDA, "no CUDA device visible: the B200 path has no CPU fallback");
        if (device < 0 || device >= n) fail(LDGMG_ERR_INVALID_ARGUMENT, "ldgmg_ctx_create: bad device");
        auto* c = new ldgmg_ctx();
        c->device = device;
        LDGMG_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop{};
        LDGMG_CUDA(cudaGetDeviceProperties(&prop, device));
        c->num_sms = prop.multiProcessorCount;
        c->smem_optin = prop.sharedMemPerBlockOptin;
        LDGMG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
        LDGMG_CUDA(cudaMalloc(&c->d_red, sizeof(double) * 1024));
        LDGMG_CUDA(cudaMallocHost(&c->h_red, sizeof(double) * 8));
        *out = c;
    });
}

int ldgmg_ctx_destroy(ldgmg_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
        cudaFree(ctx->d_red);
        cudaFreeHost(ctx->h_red);
        ctx_release_staging(*ctx);
        delete ctx;
    });
}

int ldgmg_ctx_set_stream(ldgmg_ctx* ctx, void* stream) {
    return guarded([&] {
        need(ctx, "ldgmg_ctx_set_stream");
        if (ctx->own_stream) {
            LDGMG_CUDA(cudaStreamSynchronize(ctx->stream));
            cudaStreamDestroy(ctx->stream);
        }
        ctx->stream = static_cast<cudaStream_t>(stream);
        ctx->own_stream = false;
    });
}

void* ldgmg_ctx_stream(ldgmg_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

int ldgmg_ctx_synchronize(ldgmg_ctx* ctx) {
    return guarded([&] {
        need(ctx, "ldgmg_ctx_synchronize");
        LDGMG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int ldgmg_device_alloc(ldgmg_ctx* ctx, size_t bytes, void** ptr) {
    return guarded([&] {
        need(ctx, "ldgmg_device_alloc");
        bind(*ctx);
        *ptr = dev_alloc(bytes ? bytes : 16);
    });
}
int64_t ldgmg_debug_guard_check(void) { return dev_guard_check(); }
int64_t ldgmg_debug_guard_live(void) { return dev_guard_live(); }
int ldgmg_device_free(ldgmg_ctx* ctx, void* ptr) {
    return guarded([&] {
        need(ctx, "ldgmg_device_free");
        dev_free(ptr);
    });
}
int ldgmg_copy_h2d(ldgmg_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guarded([&] {
        need(ctx, "ldgmg_copy_h2d");
        LDGMG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
        LDGMG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}
int ldgmg_copy_d2h(ldgmg_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guarded([&] {
        need(ctx, "ldgmg_copy_d2h");
        LDGMG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        LDGMG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// ------------------------------------------------------------------ BSR
int ldgmg_bsr_upload(ldgmg_ctx* ctx, int brows, int bcols, int row_bs, int col_bs, const int* ptr,
                     const int* col, const double* val, ldgmg_bsr** out) {
    return guarded([&] {
        need(ctx, "ldgmg_bsr_upload");
        need(ptr, "ldgmg_bsr_upload(ptr)");
        need(out, "ldgmg_bsr_upload(out)");
        bind(*ctx);
        *out = static_cast<ldgmg_bsr*>(own_bsr(bsr_upload(*ctx, brows, bcols, row_bs, col_bs, ptr, col, val)));
    });
}

int ldgmg_bsr_shape(const ldgmg_bsr* A, int* brows, int* bcols, int* row_bs, int* col_bs,
                    int64_t* nnzb) {
    return guarded([&] {
        need(A, "ldgmg_bsr_shape");
        if (brows) *brows = A->brows;
        if (bcols) *bcols = A->bcols;
        if (row_bs) *row_bs = A->rbs;
        if (col_bs) *col_bs = A->cbs;
        if (nnzb) *nnzb = A->nnzb;
    });
}

int ldgmg_bsr_download(ldgmg_ctx* ctx, const ldgmg_bsr* A, int* ptr, int* col, double* val) {
    return guarded([&] {
        need(ctx, "ldgmg_bsr_download");
        need(A, "ldgmg_bsr_download");
        bind(*ctx);
        bsr_download(*ctx, *A, ptr, col, val);
    });
}

int64_t ldgmg_bsr_device_bytes(const ldgmg_bsr* A) { return A ? A->device_bytes() : 0; }

int ldgmg_bsr_destroy(ldgmg_bsr* A) {
    return guarded([&] { delete A; });
}

int ldgmg_bsr_dump_coo(ldgmg_ctx* ctx, const ldgmg_bsr* A, const char* path) {
    return guarded([&] {
        need(ctx, "ldgmg_bsr_dump_coo");
        need(A, "ldgmg_bsr_dump_coo");
        need(path, "ldgmg_bsr_dump_coo(path)");
        bind(*ctx);
        std::vector<int> ptr(A->brows + 1), col(std::max<int64_t>(1, A->nnzb));
        std::vector<double> val(std::max<int64_t>(1, A->nnzb * A->rbs * A->cbs));
        bsr_download(*ctx, *A, ptr.data(), col.data(), val.data());
        coo_write(path, A->brows, A->bcols, A->rbs, A->cbs, ptr.data(), col.data(), val.data());
    });
}

int ldgmg_bsr_load_coo(ldgmg_ctx* ctx, const char* path, ldgmg_bsr** out) {
    return guarded([&] {
        need(ctx, "ldgmg_bsr_load_coo");
        need(path, "ldgmg_bsr_load_coo(path)");
        need(out, "ldgmg_bsr_load_coo(out)");
        bind(*ctx);
        const CooMatrix M = coo_read(path);
        *out = static_cast<ldgmg_bsr*>(
            own_bsr(bsr_upload(*ctx, M.brows, M.bcols, M.rbs, M.cbs, M.ptr.data(), M.col.data(), M.val.data())));
    });
}

int ldgmg_coo_write_host(const char* path, int brows, int bcols, int row_bs, int col_bs, const int* ptr,
                         const int* col, const double* val) {
    return guarded([&] {
        need(ptr, "ldgmg_coo_write_host(ptr)");
        coo_write(path, brows, bcols, row_bs, col_bs, ptr, col, val);
    });
}

int ldgmg_coo_read_host(const char* path, int* brows, int* bcols, int* row_bs, int* col_bs, int64_t* nnzb,
                        int* ptr, int* col, double* val) {
    return guarded([&] {
        const CooMatrix M = coo_read(path);
        if (brows) *brows = M.brows;
        if (bcols) *bcols = M.bcols;
        if (row_bs) *row_bs = M.rbs;
        if (col_bs) *col_bs = M.cbs;
        if (nnzb) *nnzb = int64_t(M.col.size());
        if (ptr) {
            std::memcpy(ptr, M.ptr.data(), sizeof(int) * M.ptr.size());
            if (col) std::memcpy(col, M.col.data(), sizeof(int) * M.col.size());
            if (val) std::memcpy(val, M.val.data(), sizeof(double) * M.val.size());
        }
    });
}

int ldgmg_spmv(ldgmg_ctx* ctx, const ldgmg_bsr* A, const double* x, double* y) {
    return guarded([&] {
        need(ctx, "spmv");
        need(A, "spmv");
        RowPass p;
        p.A = A;
        p.mode = MODE_SPMV;
        p.x = x;
        p.y = y;
        p.nrows = A->brows;
        launch_rowpass(*ctx, p);
    });
}

int ldgmg_spmv_transpose(ldgmg_ctx* ctx, const ldgmg_bsr* A, const double* x, double* y) {
    return guarded([&] {
        need(ctx, "spmv_transpose");
        need(A, "spmv_transpose");
        RowPass p;
        p.A = &bsr_transpose(*ctx, *A);
        p.mode = MODE_SPMV;
        p.x = x;
        p.y = y;
        p.nrows = p.A->brows;
        launch_rowpass(*ctx, p);
    });
}

int ldgmg_residual(ldgmg_ctx* ctx, const ldgmg_bsr* A, const double* b, const double* x, double* r) {
    return guarded([&] {
        need(ctx, "residual");
        need(A, "residual");
        // square blocks; a rank-local slice may have more (ghost) columns than rows
        if (A->rbs != A->cbs || A->bcols < A->brows)
            fail(LDGMG_ERR_INVALID_ARGUMENT, "residual: operator must have square blocks");
        RowPass p;
        p.A = A;
        p.mode = MODE_RESIDUAL;
        p.x = x;
        p.b = b;
        p.y = r;
        p.nrows = A->brows;
        launch_rowpass(*ctx, p);
    });
}

int ldgmg_bsr_upload_ex(ldgmg_ctx* ctx, int brows, int bcols, int row_bs, int col_bs, const int* ptr, const int* col,
                        const double* val, int flags, ldgmg_bsr** out) {
    return guarded([&] {
        need(ctx, "ldgmg_bsr_upload_ex");
        need(ptr, "ldgmg_bsr_upload_ex(ptr)");
        need(out, "ldgmg_bsr_upload_ex(out)");
        bind(*ctx);
        *out = static_cast<ldgmg_bsr*>(own_bsr(bsr_upload(*ctx, brows, bcols, row_bs, col_bs, ptr, col, val,
                                                          (flags & LDGMG_BSR_UNSORTED_COLUMNS) == 0)));
    });
}

int ldgmg_spmv_add(ldgmg_ctx* ctx, const ldgmg_bsr* A, const double* x, double* y) {
    return guarded([&] {
        need(ctx, "spmv_add");
        need(A, "spmv_add");
        RowPass p;
        p.A = A;
        p.mode = MODE_ADD;
        p.x = x;
        p.xe = y;
        p.y = y;
        p.nrows = A->brows;
        launch_rowpass(*ctx, p);
    });
}

int ldgmg_dgemm_nt_batched(ldgmg_ctx* ctx, int M, int N, int K, double alpha, const double* A, int64_t lda,
                           int64_t strideA, const double* B, int64_t ldb, int64_t strideB, double beta, double* D,
                           int64_t ldd, int64_t strideD, int batch) {
    return guarded([&] {
        need(ctx, "dgemm_nt_batched");
        if (M < 0 || N < 0 || K < 0 || batch < 0) fail(LDGMG_ERR_INVALID_ARGUMENT, "dgemm_nt_batched: negative size");
        if ((K > 0 && (lda < K || ldb < K)) || ldd < M)
            fail(LDGMG_ERR_INVALID_ARGUMENT, "dgemm_nt_batched: leading dimension too small");
        bind(*ctx);
        dgemm_nt_batched(*ctx, GemmNT{A, lda, strideA, B, ldb, strideB, D, ldd, strideD, M, N, K, alpha, beta}, batch);
    });
}

int ldgmg_bsr_set_values(ldgmg_ctx* ctx, ldgmg_bsr* A, int64_t first_block, int64_t nblocks, const double* val) {
    return guarded([&] {
        need(ctx, "ldgmg_bsr_set_values");
        need(A, "ldgmg_bsr_set_values");
        bind(*ctx);
        bsr_set_values(*ctx, *A, first_block, nblocks, val);
    });
}

int ldgmg_bsr_gather(ldgmg_ctx* ctx, const ldgmg_bsr* src, int brows, int bcols, const int* ptr, const int* col,
                     const int64_t* src_blocks, ldgmg_bsr** out) {
    return guarded([&] {
        need(ctx, "ldgmg_bsr_gather");
        need(src, "ldgmg_bsr_gather");
        need(ptr, "ldgmg_bsr_gather(ptr)");
        need(out, "ldgmg_bsr_gather(out)");
        bind(*ctx);
        *out = static_cast<ldgmg_bsr*>(own_bsr(bsr_gather(*ctx, *src, brows, bcols, ptr, col, src_blocks)));
    });
}

int ldgmg_bsr_row_prefix_view(ldgmg_ctx* ctx, const ldgmg_bsr* base, int nrows, ldgmg_bsr** out) {
    return guarded([&] {
        need(ctx, "ldgmg_bsr_row_prefix_view");
        need(base, "ldgmg_bsr_row_prefix_view");
        need(out, "ldgmg_bsr_row_prefix_view(out)");
        bind(*ctx);
        *out = static_cast<ldgmg_bsr*>(own_bsr(bsr_row_prefix_view(*ctx, *base, nrows)));
    });
}

int ldgmg_bsr_transposed_view(ldgmg_ctx* ctx, const ldgmg_bsr* base, int brows, int bcols, const int* ptr,
                              const int* col, const int* perm, ldgmg_bsr** out) {
    return guarded([&] {
        need(ctx, "ldgmg_bsr_transposed_view");
        need(base, "ldgmg_bsr_transposed_view");
        need(ptr, "ldgmg_bsr_transposed_view(ptr)");
        need(out, "ldgmg_bsr_transposed_view(out)");
        bind(*ctx);
        *out = static_cast<ldgmg_bsr*>(own_bsr(bsr_transposed_view(*ctx, *base, brows, bcols, ptr, col, perm)));
    });
}

int ldgmg_residual_rows(ldgmg_ctx* ctx, const ldgmg_bsr* A, const double* b, const double* x, double* r,
                        const int* rows, int nrows) {
    return guarded([&] {
        need(ctx, "residual_rows");
        need(A, "residual_rows");
        if (A->rbs != A->cbs) fail(LDGMG_ERR_INVALID_ARGUMENT, "residual: operator must have square blocks");
        if (nrows < 0 || nrows > A->brows) fail(LDGMG_ERR_INVALID_ARGUMENT, "residual_rows: bad row count");
        if (nrows == 0) return;
        need(rows, "residual_rows(rows)");
        RowPass p;
        p.A = A;
        p.mode = MODE_RESIDUAL;
        p.x = x;
        p.b = b;
        p.y = r;
        p.rows = rows;
        p.nrows = nrows;
        launch_rowpass(*ctx, p);
    });
}

int ldgmg_spmv_add_rows(ldgmg_ctx* ctx, const ldgmg_bsr* A, const double* x, double* y, const int* rows,
                        int nrows) {
    return guarded([&] {
        need(ctx, "spmv_add_rows");
        need(A, "spmv_add_rows");
        if (nrows < 0 || nrows > A->brows) fail(LDGMG_ERR_INVALID_ARGUMENT, "spmv_add_rows: bad row count");
        if (nrows == 0) return;
        need(rows, "spmv_add_rows(rows)");
        RowPass p;
        p.A = A;
        p.mode = MODE_ADD;
        p.x = x;
        p.xe = y;
        p.y = y;
        p.rows = rows;
        p.nrows = nrows;
        launch_rowpass(*ctx, p);
    });
}

int ldgmg_pgs_schedule(int n_own, const int* ptr, const int* col, int reverse, int* rows, int* level_ptr,
                       int* nlevels) {
    return guarded([&] {
        need(ptr, "pgs_schedule(ptr)");
        need(nlevels, "pgs_schedule(nlevels)");
        if (n_own < 0) fail(LDGMG_ERR_INVALID_ARGUMENT, "pgs_schedule: negative row count");
        std::vector<int> part(static_cast<size_t>(n_own), 0);
        std::vector<int> hp(ptr, ptr + n_own + 1), hc(col, col + (n_own ? ptr[n_own] : 0));
        std::vector<int> r, lp;
        pgs_wavefronts(n_own, hp.data(), hc.data(), part.data(), n_own, reverse != 0, r, lp);
        *nlevels = int(lp.size()) - 1;
        if (rows) std::copy(r.begin(), r.end(), rows);
        if (level_ptr) std::copy(lp.begin(), lp.end(), level_ptr);
    });
}

struct ldgmg_factors {
    DiagFactors f;
};

int ldgmg_factors_upload(ldgmg_ctx* ctx, int n, int bs, const double* V, const double* lambda, const double* s,
                         ldgmg_factors** out) {
    return guarded([&] {
        need(ctx, "factors_upload");
        need(V, "factors_upload(V)");
        need(lambda, "factors_upload(lambda)");
        need(s, "factors_upload(s)");
        bind(*ctx);
        auto* h = new ldgmg_factors();
        upload_factors(*ctx, h->f, n, bs, V, lambda, s);
        *out = h;
    });
}

int ldgmg_factors_destroy(ldgmg_factors* F) {
    return guarded([&] { delete F; });
}

int ldgmg_relax(ldgmg_ctx* ctx, const ldgmg_bsr* A, const ldgmg_factors* F, const double* b, const double* x_src,
                const double* x_live, double* x_out, double omega) {
    return guarded([&] {
        need(ctx, "relax");
        need(A, "relax");
        need(F, "relax(factors)");
        if (F->f.n != A->brows) fail(LDGMG_ERR_INVALID_ARGUMENT, "relax: factor count != block rows");
        RowPass p;
        p.A = A;
        p.mode = MODE_RELAX;
        p.x = x_src;
        p.b = b;
        p.xe = x_live;
        p.y = x_out;
        p.nrows = A->brows;
        p.F = &F->f;
        p.omega = omega;
        launch_rowpass(*ctx, p);
    });
}

int ldgmg_relax_rows(ldgmg_ctx* ctx, const ldgmg_bsr* A, const ldgmg_factors* F, const double* b,
                     const double* x_src, const double* x_live, double* x_out, double omega, const int* rows,
                     int nrows) {
    return guarded([&] {
        need(ctx, "relax_rows");
        need(A, "relax_rows");
        need(F, "relax_rows(factors)");
        if (F->f.n != A->brows) fail(LDGMG_ERR_INVALID_ARGUMENT, "relax: factor count != block rows");
        if (nrows < 0 || nrows > A->brows) fail(LDGMG_ERR_INVALID_ARGUMENT, "relax: bad row count");
        if (nrows == 0) return;
        need(rows, "relax_rows(rows)");
        RowPass p;
        p.A = A;
        p.mode = MODE_RELAX;
        p.x = x_src;
        p.b = b;
        p.xe = x_live;
        p.y = x_out;
        p.rows = rows;
        p.nrows = nrows;
        p.F = &F->f;
        p.omega = omega;
        launch_rowpass(*ctx, p);
    });
}

int ldgmg_project_partials(ldgmg_ctx* ctx, const double* v_own, int N, int r0, int r1, int bs, const int* offs,
                           int ncomp, double kval, double* partials) {
    return guarded([&] {
        need(ctx, "project_partials");
        launch_project_partials_slice(*ctx, v_own, N, r0, r1, bs, offs, ncomp, kval, partials);
    });
}

int ldgmg_project_apply(ldgmg_ctx* ctx, double* v_own, int N, int r0, int r1, int bs, const int* offs, int ncomp,
                        double kval, const double* partials) {
    return guarded([&] {
        need(ctx, "project_apply");
        launch_project_apply_slice(*ctx, v_own, N, r0, r1, bs, offs, ncomp, kval, partials);
    });
}

int ldgmg_gather_blocks(ldgmg_ctx* ctx, const double* x, const int* idx, int n, int bs, double* out) {
    return guarded([&] {
        need(ctx, "gather_blocks");
        launch_gather_blocks(*ctx, x, idx, n, bs, out);
    });
}

int ldgmg_partition_level(int N, const int* ptr, const int* col, int nranks, int rank, int* r0, int* r1, int* n_ghost,
                          int* n_send, int* local_col, int* ghost_gid, int* recv_count, int* send_count,
                          int* send_idx) {
    return guarded([&] {
        need(ptr, "partition_level(ptr)");
        if (nranks < 1 || nranks > N) fail(LDGMG_ERR_INVALID_ARGUMENT, "partition_ranges: partition count must lie in [1, N]");
        if (rank < 0 || rank >= nranks) fail(LDGMG_ERR_INVALID_ARGUMENT, "partition_level: bad rank");
        auto lo = [&](int p) { return int((long long)p * N / nranks); };
        auto owner = [&](int j) {
            int p = int((long long)j * nranks / N);
            while (p + 1 < nranks && lo(p + 1) <= j) ++p;
            while (p > 0 && lo(p) > j) --p;
            return p;
        };
        const int a = lo(rank), b = lo(rank + 1), nown = b - a;
        // ghost set: non-owned columns of our rows, grouped by owner, ascending gid
        std::vector<std::vector<int>> by(nranks);
        {
            std::vector<char> seen(N, 0);
            for (int i = a; i < b; ++i)
                for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
                    const int j = col[k];
                    if ((j < a || j >= b) && !seen[j]) {
                        seen[j] = 1;
                        by[owner(j)].push_back(j);
                    }
                }
        }
        std::vector<int> ghosts;
        std::vector<int> rc(nranks, 0);
        for (int p = 0; p < nranks; ++p) {
            std::sort(by[p].begin(), by[p].end());
            rc[p] = int(by[p].size());
            ghosts.insert(ghosts.end(), by[p].begin(), by[p].end());
        }
        // send lists: for every other rank q, the owned columns q's rows reference
        std::vector<std::vector<int>> sends(nranks);
        for (int q = 0; q < nranks; ++q) {
            if (q == rank) continue;
            std::vector<char> seen(size_t(nown), 0);
            for (int i = lo(q); i < lo(q + 1); ++i)
                for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
                    const int j = col[k];
                    if (j >= a && j < b && !seen[j - a]) {
                        seen[j - a] = 1;
                        sends[q].push_back(j - a);
                    }
                }
            std::sort(sends[q].begin(), sends[q].end());
        }
        int ns = 0;
        for (auto& s : sends) ns += int(s.size());
        *r0 = a;
        *r1 = b;
        *n_ghost = int(ghosts.size());
        *n_send = ns;
        if (!local_col) return;
        std::unordered_map<int, int> slot;
        for (size_t g = 0; g < ghosts.size(); ++g) slot[ghosts[g]] = nown + int(g);
        for (int i = a, o = 0; i < b; ++i)
            for (int k = ptr[i]; k < ptr[i + 1]; ++k, ++o) {
                const int j = col[k];
                local_col[o] = (j >= a && j < b) ? j - a : slot.at(j);
            }
        if (ghost_gid) std::memcpy(ghost_gid, ghosts.data(), sizeof(int) * ghosts.size());
        if (recv_count) std::memcpy(recv_count, rc.data(), sizeof(int) * nranks);
        if (send_count)
            for (int q = 0; q < nranks; ++q) send_count[q] = int(sends[q].size());
        if (send_idx)
            for (int q = 0, o = 0; q < nranks; ++q)
                for (int v : sends[q]) send_idx[o++] = v;
    });
}

int ldgmg_dot(ldgmg_ctx* ctx, int64_t n, const double* a, const double* b, double* out_host) {
    return guarded([&] {
        need(ctx, "dot");
        launch_dot(*ctx, n, a, b, ctx->d_red);
        LDGMG_CUDA(cudaMemcpyAsync(ctx->h_red, ctx->d_red, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        LDGMG_CUDA(cudaStreamSynchronize(ctx->stream));
        *out_host = ctx->h_red[0];
    });
}

int ldgmg_axpy(ldgmg_ctx* ctx, int64_t n, double alpha, const double* x, double* y) {
    return guarded([&] {
        need(ctx, "axpy");
        launch_axpy(*ctx, n, alpha, x, y);
    });
}

// ------------------------------------------------------------ smoothers
static Smoother& smoother_base(ldgmg_ctx* ctx, const ldgmg_bsr* A, const ldgmg_smoother_config* cfg,
                               ldgmg_smoother*& h) {
    need(ctx, "smoother_create");
    need(A, "smoother_create");
    need(cfg, "smoother_create(cfg)");
    bind(*ctx);
    h = new ldgmg_smoother();
    h->s.A = A;
    h->s.cfg = *cfg;
    return h->s;
}

int ldgmg_smoother_create(ldgmg_ctx* ctx, const ldgmg_bsr* A, int system_kind, int n_velocity,
                          const ldgmg_smoother_config* cfg, ldgmg_smoother** out) {
    ldgmg_smoother* h = nullptr;
    const int rc = guarded([&] {
        Smoother& s = smoother_base(ctx, A, cfg, h);
        s.system_kind = system_kind;
        s.n_velocity = n_velocity;
        s.init_common(*ctx);
        if (s.cfg.kind == LDGMG_SAI) {
            SaiResult r = build_sai_gpu(*ctx, *A, system_kind, n_velocity, s.cfg.level, s.cfg.zeta,
                                        s.cfg.cache != 0, nullptr);
            s.B = std::move(r.B);
            s.stats = r.stats;
        } else {
            compute_factors(*ctx, *A, s.F);
        }
        *out = h;
    });
    if (rc != LDGMG_OK) delete h;
    return rc;
}

int ldgmg_smoother_create_with_factors(ldgmg_ctx* ctx, const ldgmg_bsr* A,
                                       const ldgmg_smoother_config* cfg, const double* V,
                                       const double* lambda, const double* s, ldgmg_smoother** out) {
    ldgmg_smoother* h = nullptr;
    const int rc = guarded([&] {
        need(V, "factors(V)");
        need(lambda, "factors(lambda)");
        need(s, "factors(s)");
        Smoother& sm = smoother_base(ctx, A, cfg, h);
        if (sm.cfg.kind == LDGMG_SAI) fail(LDGMG_ERR_INVALID_ARGUMENT, "factors given to an SAI smoother");
        sm.init_common(*ctx);
        upload_factors(*ctx, sm.F, sm.N, sm.bs, V, lambda, s);
        *out = h;
    });
    if (rc != LDGMG_OK) delete h;
    return rc;
}

int ldgmg_smoother_create_with_sai(ldgmg_ctx* ctx, const ldgmg_bsr* A, const ldgmg_smoother_config* cfg,
                                   const int* Bptr, const int* Bcol, const double* Bval,
                                   ldgmg_smoother** out) {
    ldgmg_smoother* h = nullptr;
    const int rc = guarded([&] {
        Smoother& sm = smoother_base(ctx, A, cfg, h);
        if (sm.cfg.kind != LDGMG_SAI) fail(LDGMG_ERR_INVALID_ARGUMENT, "SAI matrix given to a non-SAI smoother");
        sm.init_common(*ctx);
        sm.B = bsr_upload(*ctx, A->brows, A->bcols, A->rbs, A->cbs, Bptr, Bcol, Bval);
        *out = h;
    });
    if (rc != LDGMG_OK) delete h;
    return rc;
}

int ldgmg_smoother_apply(ldgmg_ctx* ctx, const ldgmg_smoother* S, const double* b, double* x, int sweep) {
    return guarded([&] {
        need(ctx, "Smoother::apply");
        need(S, "Smoother::apply");
        S->s.apply(*ctx, b, x, sweep);
    });
}

int ldgmg_smoother_colours(const ldgmg_smoother* S, int* colour, int* ncolours) {
    return guarded([&] {
        need(S, "colours");
        if (colour && !S->s.colour.empty()) std::memcpy(colour, S->s.colour.data(), sizeof(int) * S->s.colour.size());
        if (ncolours) *ncolours = S->s.ncolours;
    });
}

int ldgmg_smoother_sai_nnzb(const ldgmg_smoother* S, int64_t* nnzb) {
    return guarded([&] {
        need(S, "sai_matrix");
        if (S->s.cfg.kind != LDGMG_SAI || !S->s.B) fail(LDGMG_ERR_LOGIC, "not an SAI smoother");
        *nnzb = S->s.B->nnzb;
    });
}

int ldgmg_smoother_sai_matrix(ldgmg_ctx* ctx, const ldgmg_smoother* S, int* ptr, int* col, double* val) {
    return guarded([&] {
        need(ctx, "sai_matrix");
        need(S, "sai_matrix");
        if (S->s.cfg.kind != LDGMG_SAI || !S->s.B) fail(LDGMG_ERR_LOGIC, "not an SAI smoother");
        bsr_download(*ctx, *S->s.B, ptr, col, val);
    });
}

int ldgmg_smoother_sai_stats(const ldgmg_smoother* S, ldgmg_sai_stats* out) {
    return guarded([&] {
        need(S, "sai_stats");
        *out = S->s.stats;
    });
}

int ldgmg_smoother_diag_factors(ldgmg_ctx* ctx, const ldgmg_smoother* S, double* V, double* lambda,
                                double* s) {
    return guarded([&] {
        need(ctx, "diag_factors");
        need(S, "diag_factors");
        const DiagFactors& F = S->s.F;
        if (!F.n) fail(LDGMG_ERR_LOGIC, "smoother has no diagonal factors");
        const int bs = F.bs;
        if (V) {
            std::vector<double> hv(size_t(F.n) * F.vstride);
            d2h(*ctx, hv.data(), F.V.p, sizeof(double) * hv.size());
            for (int e = 0; e < F.n; ++e)
                for (int a = 0; a < bs; ++a)
                    for (int b = 0; b < bs; ++b)
                        V[(size_t(e) * bs + a) * bs + b] = hv[size_t(e) * F.vstride + size_t(a) * F.ld + b];
        }
        if (lambda) d2h(*ctx, lambda, F.lambda.p, F.lambda.bytes);
        if (s) d2h(*ctx, s, F.scale.p, F.scale.bytes);
    });
}

int ldgmg_smoother_destroy(ldgmg_smoother* S) {
    return guarded([&] { delete S; });
}

// ------------------------------------------------------------ transfers
int ldgmg_transfer_create(ldgmg_ctx* ctx, int n_fine, int n_coarse, const int* parent_of,
                          const int* orthant_of, int dim, int bs_scalar, int n_comp, const double* K,
                          ldgmg_transfer** out) {
    return guarded([&] {
        need(ctx, "transfer_create");
        need(parent_of, "transfer_create(parent_of)");
        need(orthant_of, "transfer_create(orthant_of)");
        need(K, "transfer_create(K)");
        bind(*ctx);
        auto* h = new ldgmg_transfer();
        h->t = transfer_create(*ctx, n_fine, n_coarse, parent_of, orthant_of, dim, bs_scalar, n_comp, K);
        *out = h;
    });
}

int ldgmg_restrict(ldgmg_ctx* ctx, const ldgmg_transfer* T, const double* rf, double* rc) {
    return guarded([&] {
        need(ctx, "restrict_residual");
        need(T, "restrict_residual");
        launch_restrict(*ctx, *T->t, rf, rc);
    });
}

int ldgmg_interpolate_add(ldgmg_ctx* ctx, const ldgmg_transfer* T, const double* xc, double* xf) {
    return guarded([&] {
        need(ctx, "interpolate_add");
        need(T, "interpolate_add");
        launch_prolong_add(*ctx, *T->t, xc, xf);
    });
}

int ldgmg_transfer_destroy(ldgmg_transfer* T) {
    return guarded([&] { delete T; });
}

// ------------------------------------------------------------ multigrid
/// Wall-clock setup phases on stderr when LDGMG_SETUP_TIMING=1 (stream-synchronised).
struct SetupTimer {
    const char* what;
    cudaStream_t s;
    bool on;
    std::chrono::steady_clock::time_point t;
    SetupTimer(const char* w, cudaStream_t st) : what(w), s(st) {
        const char* e = getenv("LDGMG_SETUP_TIMING");
        on = e && atoi(e);
        t = std::chrono::steady_clock::now();
    }
    void stamp(const char* phase) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[setup %s] %-22s %9.3f s\n", what, phase, std::chrono::duration<double>(now - t).count());
        t = now;
    }
};

static void mg_default_smoothers(ldgmg_ctx* ctx, Mg& m) {
    m.sm.assign(m.depth, nullptr);
    if (!m.sai_cache) m.sai_cache = sai_cache_new();
    for (int l = 0; l + 1 < m.depth; ++l) {
        auto s = std::make_unique<Smoother>();
        s->A = m.A[l];
        s->cfg = m.cfg.smoother;
        s->system_kind = m.system_kind;
        s->n_velocity = m.n_velocity;
        s->init_common(*ctx);
        SetupTimer tm("smoother", ctx->stream);
        if (s->cfg.kind == LDGMG_SAI) {
            SaiResult r = build_sai_gpu(*ctx, *m.A[l], m.system_kind, m.n_velocity, s->cfg.level,
                                        s->cfg.zeta, s->cfg.cache != 0, m.sai_cache);
            s->B = std::move(r.B);
            s->stats = r.stats;
            tm.stamp(l == 0 ? "SAI build level 0" : "SAI build coarse");
        } else {
            compute_factors(*ctx, *m.A[l], s->F);
            tm.stamp(l == 0 ? "diag factors level 0" : "diag factors coarse");
        }
        m.sm[l] = s.get();
        m.own_sm.push_back(std::move(s));
    }
}

int ldgmg_mg_create(ldgmg_ctx* ctx, int depth, const ldgmg_bsr* const* A,
                    const ldgmg_transfer* const* transfers, int system_kind, int dim, int n_comp,
                    int bs_scalar, int kernel_constants, int kernel_pressure, const ldgmg_mg_config* cfg,
                    const double* bottom_V, const double* bottom_lambda, ldgmg_mg** out) {
    ldgmg_mg* h = nullptr;
    const int rc = guarded([&] {
        need(ctx, "Multigrid");
        need(A, "Multigrid(A)");
        need(cfg, "Multigrid(cfg)");
        bind(*ctx);
        h = new ldgmg_mg();
        Mg& m = h->m;
        m.depth = depth;
        m.cfg = *cfg;
        m.system_kind = system_kind;
        m.dim = dim;
        m.n_comp = n_comp;
        m.bs_scalar = bs_scalar;
        m.kernel_constants = kernel_constants;
        m.kernel_pressure = kernel_pressure;
        m.n_velocity = system_kind == LDGMG_SYSTEM_STOKES ? dim * bs_scalar : 0;
        for (int l = 0; l < depth; ++l) {
            need(A[l], "Multigrid(A[l])");
            m.A.push_back(A[l]);
        }
        for (int l = 0; l + 1 < depth; ++l) m.T.push_back(transfers ? transfers[l]->t.get() : nullptr);
        m.init(*ctx);
        if (m.bs != n_comp * bs_scalar) fail(LDGMG_ERR_INVALID_ARGUMENT, "multigrid: block size != n_comp*bs_scalar");
        m.set_bottom(*ctx, bottom_V, bottom_lambda);
        m.sm.assign(depth, nullptr);
        *out = h;
    });
    if (rc != LDGMG_OK) delete h;
    return rc;
}

int ldgmg_mg_set_smoother(ldgmg_mg* mg, int level, ldgmg_smoother* S) {
    return guarded([&] {
        need(mg, "mg_set_smoother");
        need(S, "mg_set_smoother");
        if (level < 0 || level + 1 >= mg->m.depth) fail(LDGMG_ERR_LOGIC, "multigrid: the bottom level has no smoother");
        if (S->s.A != mg->m.A[level]) fail(LDGMG_ERR_INVALID_ARGUMENT, "mg_set_smoother: smoother bound to another operator");
        mg->m.sm[level] = &S->s;
        mg->m.invalidate_graphs();
    });
}

static void ensure_smoothers(ldgmg_ctx* ctx, Mg& m) {
    bool any_missing = false;
    for (int l = 0; l + 1 < m.depth; ++l) any_missing |= m.sm[l] == nullptr;
    if (any_missing) {
        std::vector<Smoother*> keep = m.sm;
        mg_default_smoothers(ctx, m);
        for (int l = 0; l + 1 < m.depth; ++l)
            if (keep[l]) m.sm[l] = keep[l];
    }
}

int ldgmg_mg_smoother(ldgmg_mg* mg, int level, ldgmg_smoother** out) {
    return guarded([&] {
        need(mg, "mg_smoother");
        if (level < 0 || level + 1 >= mg->m.depth) fail(LDGMG_ERR_LOGIC, "multigrid: the bottom level has no smoother");
        if (!mg->m.sm[level]) fail(LDGMG_ERR_LOGIC, "multigrid: smoothers not built yet");
        // non-owning view handle sharing the Smoother object
        *out = reinterpret_cast<ldgmg_smoother*>(mg->m.sm[level]);
    });
}

int ldgmg_mg_depth(const ldgmg_mg* mg) { return mg ? mg->m.depth : 0; }

int ldgmg_mg_cycle(ldgmg_ctx* ctx, ldgmg_mg* mg, double* x, const double* b) {
    return guarded([&] {
        need(ctx, "Multigrid::cycle");
        need(mg, "Multigrid::cycle");
        ensure_smoothers(ctx, mg->m);
        mg->m.cycle(*ctx, x, b);
    });
}

int ldgmg_mg_vcycle(ldgmg_ctx* ctx, ldgmg_mg* mg, double* x, const double* b) {
    return guarded([&] {
        need(ctx, "mg_vcycle");
        need(mg, "mg_vcycle");
        ensure_smoothers(ctx, mg->m);
        mg->m.v_cycle(*ctx, 0, x, b);
    });
}

int ldgmg_mg_apply(ldgmg_ctx* ctx, ldgmg_mg* mg, const double* b, double* x) {
    return guarded([&] {
        need(ctx, "Multigrid::apply");
        need(mg, "Multigrid::apply");
        ensure_smoothers(ctx, mg->m);
        mg->m.apply(*ctx, b, x);
    });
}

int ldgmg_mg_cycles(ldgmg_ctx* ctx, ldgmg_mg* mg, double* x, const double* b, int ncycles) {
    return guarded([&] {
        need(ctx, "mg_cycles");
        need(mg, "mg_cycles");
        ensure_smoothers(ctx, mg->m);
        mg->m.cycles(*ctx, x, b, ncycles);
    });
}

namespace {

/// Device state of the graph-resident solve loop: bn, tol, it, maxit, then
/// the relative-residual history (hist[it] after `it` cycles).
struct SolveState {
    double bn, tol;
    int it, maxit;
    int pad[4];
};
constexpr int kSolveHist = int(sizeof(SolveState) / sizeof(double));

/// The device loop copies the final x once after it (copying every iterate
/// inside the loop body measured slower).
constexpr bool solve_snap_in_loop() { return false; }

/// The loop test of ldgmg_mg_solve_host on the device: rr = ||r|| / ||b||
/// (IEEE sqrt and division, the host loop's bits), history entry, and the
/// WHILE node's condition rr > tol && it < maxit.
__global__ void solve_check_kernel(const double* __restrict__ red_b, const double* __restrict__ red_r,
                                   double* st_raw, int first, cudaGraphConditionalHandle h) {
    SolveState* st = reinterpret_cast<SolveState*>(st_raw);
    if (first) {
        st->bn = sqrt(red_b[0]);
        st->it = 0;
    } else {
        st->it += 1;
    }
    const double rn = sqrt(red_r[0]);
    const double rr = st->bn > 0 ? rn / st->bn : rn;
    st_raw[kSolveHist + st->it] = rr;
    cudaGraphSetConditional(h, (rr > st->tol && st->it < st->maxit) ? 1u : 0u);
}

/// Capture the whole stationary solve as ONE graph: prologue (x = 0, ||b||,
/// first residual check) and a conditional WHILE node whose body is one
/// V-cycle, the iterate's device snapshot + copy to pinned host memory (a
/// side branch under the residual check) and the check itself.  No host
/// round trip per iteration.  Returns false (and leaves the host loop in
/// charge) if the driver rejects any piece.
bool build_solve_graph(Ctx& ctx, Mg& m, double* x, const double* b, double* rbuf, bool reuse, int64_t n,
                       int cap, int64_t& n_pro, int64_t& n_body) {
    auto ok = [](cudaError_t e) {
        if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    };
    if (m.solve_exec) {
        cudaGraphExecDestroy(m.solve_exec);
        m.solve_exec = nullptr;
    }
    if (!m.cap_stream) ok(cudaStreamCreateWithFlags(&m.cap_stream, cudaStreamNonBlocking));
    if (!m.cap_side) ok(cudaStreamCreateWithFlags(&m.cap_side, cudaStreamNonBlocking));
    for (auto& e : m.cap_ev)
        if (!e) ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (m.solve_red.bytes < sizeof(double) * 1024) m.solve_red.alloc(sizeof(double) * 1024);
    m.solve_state.alloc(sizeof(double) * (kSolveHist + cap));
    double* red_b = m.solve_red.as<double>();
    double* red_r = red_b + 512;
    double* st = m.solve_state.as<double>();
    if (!m.warm) {  // kernel attributes and lazy transposes outside capture
        m.cycle(ctx, m.solve_xs.as<double>(), b, false);
        ok(cudaStreamSynchronize(ctx.stream));
        m.warm = true;
    }
    ok(cudaStreamSynchronize(ctx.stream));
    Ctx cctx = ctx;
    cctx.stream = m.cap_stream;
    auto check_pass = [&](int first) {
        RowPass p;
        p.A = m.A[0];
        p.mode = MODE_RESIDUAL;
        p.x = x;
        p.b = b;
        p.y = rbuf;
        p.nrows = m.A[0]->brows;
        launch_rowpass(cctx, p);
        launch_dot(cctx, n, rbuf, rbuf, red_r);
        (void)first;
    };
    cudaGraph_t g = nullptr;
    bool capturing = false;
    const int64_t c0 = launch_counter().load();
    try {
        ok(cudaStreamBeginCapture(m.cap_stream, cudaStreamCaptureModeThreadLocal));
        capturing = true;
        ok(cudaMemsetAsync(x, 0, sizeof(double) * n, m.cap_stream));
        launch_dot(cctx, n, b, b, red_b);
        // x = 0: the first residual b - A 0 is b bit for bit (every block
        // product is +0, b - (+0) = b), so it is copied instead of computed
        ok(cudaMemcpyAsync(rbuf, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, m.cap_stream));
        launch_dot(cctx, n, rbuf, rbuf, red_r);
        cudaStreamCaptureStatus status;
        cudaGraph_t cg = nullptr;
        ok(cudaStreamGetCaptureInfo(m.cap_stream, &status, nullptr, &cg, nullptr, nullptr));
        cudaGraphConditionalHandle h;
        ok(cudaGraphConditionalHandleCreate(&h, cg, 0, 0));
        solve_check_kernel<<<1, 1, 0, m.cap_stream>>>(red_b, red_r, st, 1, h);
        ok(cudaGetLastError());
        const cudaGraphNode_t* deps = nullptr;
        size_t ndeps = 0;
        ok(cudaStreamGetCaptureInfo(m.cap_stream, &status, nullptr, &cg, &deps, &ndeps));
        cudaGraphNodeParams cp{};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        ok(cudaGraphAddNode(&node, cg, deps, ndeps, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        ok(cudaStreamUpdateCaptureDependencies(m.cap_stream, &node, 1, cudaStreamSetCaptureDependencies));
        ok(cudaStreamEndCapture(m.cap_stream, &g));
        capturing = false;
        n_pro = launch_counter().load() - c0 + 1;
        const int64_t c1 = launch_counter().load();
        ok(cudaStreamBeginCaptureToGraph(m.cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        capturing = true;
        m.cycle(cctx, x, b, reuse);
        if (solve_snap_in_loop()) {
            ok(cudaMemcpyAsync(m.solve_xs.p, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, m.cap_stream));
            ok(cudaEventRecord(m.cap_ev[0], m.cap_stream));
            ok(cudaStreamWaitEvent(m.cap_side, m.cap_ev[0], 0));
            ok(cudaMemcpyAsync(m.h_stage_x, m.solve_xs.p, sizeof(double) * n, cudaMemcpyDeviceToHost, m.cap_side));
            ok(cudaEventRecord(m.cap_ev[1], m.cap_side));
        }
        check_pass(0);
        solve_check_kernel<<<1, 1, 0, m.cap_stream>>>(red_b, red_r, st, 0, h);
        ok(cudaGetLastError());
        if (solve_snap_in_loop()) ok(cudaStreamWaitEvent(m.cap_stream, m.cap_ev[1], 0));
        cudaGraph_t bout = nullptr;
        ok(cudaStreamEndCapture(m.cap_stream, &bout));
        capturing = false;
        n_body = launch_counter().load() - c1 + 1;
        ok(cudaGraphInstantiate(&m.solve_exec, g, 0));
        ok(cudaGraphDestroy(g));
        g = nullptr;
    } catch (const std::exception& e) {
        if (capturing) {
            cudaGraph_t junk = nullptr;
            cudaStreamEndCapture(m.cap_stream, &junk);
            if (junk) cudaGraphDestroy(junk);
        }
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        if (getenv("LDGMG_SOLVE_TIMING")) fprintf(stderr, "[solve_host] device loop unavailable: %s\n", e.what());
        launch_counter().store(c0);
        m.solve_exec = nullptr;
        return false;
    }
    launch_counter().store(c0);  // captured launches run (and are counted) per graph launch
    m.solve_cap = cap;
    return true;
}

}  // namespace

int ldgmg_mg_solve_host(ldgmg_ctx* ctx, ldgmg_mg* mg, const double* b_host, double* x_host, double tol,
                        int maxit, double* history, int* iters) {
    return guarded([&] {
        need(ctx, "mg_solve_host");
        need(mg, "mg_solve_host");
        need(b_host, "mg_solve_host(b)");
        need(x_host, "mg_solve_host(x)");
        if (maxit < 0) fail(LDGMG_ERR_INVALID_ARGUMENT, "mg_solve_host: maxit must be nonnegative");
        Mg& m = mg->m;
        ensure_smoothers(ctx, m);
        const int64_t n = int64_t(m.A[0]->brows) * m.bs;
        // device vectors and a pinned staging buffer cached on the hierarchy:
        // the same pointers every call keep the captured V-cycle graph valid
        if (m.solve_b.bytes < sizeof(double) * size_t(std::max<int64_t>(1, n))) {
            m.solve_b.alloc(sizeof(double) * std::max<int64_t>(1, n));
            m.solve_x.alloc(sizeof(double) * std::max<int64_t>(1, n));
            m.solve_r.alloc(sizeof(double) * std::max<int64_t>(1, n));
            if (m.h_stage) cudaFreeHost(m.h_stage);
            m.h_stage = nullptr;
            LDGMG_CUDA(cudaMallocHost(&m.h_stage, sizeof(double) * std::max<int64_t>(1, n)));
        }
        if (m.solve_xs.bytes < m.solve_x.bytes) {
            m.solve_xs.alloc(m.solve_x.bytes);
            if (m.h_stage_x) cudaFreeHost(m.h_stage_x);
            m.h_stage_x = nullptr;
            LDGMG_CUDA(cudaMallocHost(&m.h_stage_x, m.solve_x.bytes));
        }
        if (!m.d2h_stream) {
            LDGMG_CUDA(cudaStreamCreateWithFlags(&m.d2h_stream, cudaStreamNonBlocking));
            LDGMG_CUDA(cudaEventCreateWithFlags(&m.ev_snap, cudaEventDisableTiming));
            LDGMG_CUDA(cudaEventCreateWithFlags(&m.ev_d2h, cudaEventDisableTiming));
        }
        DevBuf &b = m.solve_b, &x = m.solve_x, &r = m.solve_r;
        static const bool timing = getenv("LDGMG_SOLVE_TIMING") && atoi(getenv("LDGMG_SOLVE_TIMING"));
        auto tnow = [] { return std::chrono::steady_clock::now(); };
        auto tsec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count() * 1e3; };
        const auto T0 = tnow();
        // pageable -> pinned with host threads, then one DMA
        LDGMG_CUDA(cudaMemcpyAsync(b.p, b_host, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        if (timing) LDGMG_CUDA(cudaStreamSynchronize(ctx->stream));
        const auto T0b = tnow();
        // With an SAI level-0 smoother the residual check of iterate k is the
        // first kernel of cycle k+1 (r = b - A x, same kernel, same bits):
        // compute it into the smoother's residual buffer and let the cycle
        // start from it, one level-0 pass saved per iteration.
        double* rbuf = m.r0_buffer();
        const bool reuse = rbuf != nullptr;
        if (!rbuf) rbuf = r.as<double>();
        static const int dev_loop = getenv("LDGMG_SOLVE_GRAPH") ? atoi(getenv("LDGMG_SOLVE_GRAPH")) : 1;
        if (dev_loop && !m.solve_graph_bad) {
            int64_t& n_pro = m.solve_npro;
            int64_t& n_body = m.solve_nbody;
            const int cap = std::max(maxit + 1, 128);
            if (!m.solve_exec || m.solve_cap < maxit + 1)
                if (!build_solve_graph(*ctx, m, x.as<double>(), b.as<double>(), rbuf, reuse, n, cap, n_pro, n_body))
                    m.solve_graph_bad = true;
            if (m.solve_exec) {
                std::vector<double> hs(kSolveHist + size_t(maxit) + 1, 0.0);
                SolveState* S = reinterpret_cast<SolveState*>(hs.data());
                S->tol = tol;
                S->maxit = maxit;
                LDGMG_CUDA(cudaMemcpyAsync(m.solve_state.p, hs.data(), sizeof(SolveState), cudaMemcpyHostToDevice,
                                           ctx->stream));
                LDGMG_CUDA(cudaGraphLaunch(m.solve_exec, ctx->stream));
                // a page-locked destination takes the iterate by DMA directly
                cudaPointerAttributes xat{};
                const bool x_pinned = cudaPointerGetAttributes(&xat, x_host) == cudaSuccess &&
                                      xat.type == cudaMemoryTypeHost;
                cudaGetLastError();
                if (!solve_snap_in_loop())
                    LDGMG_CUDA(cudaMemcpyAsync(x_pinned ? static_cast<void*>(x_host) : m.h_stage_x, x.p,
                                               sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
                LDGMG_CUDA(cudaMemcpyAsync(hs.data(), m.solve_state.p, sizeof(double) * hs.size(),
                                           cudaMemcpyDeviceToHost, ctx->stream));
                LDGMG_CUDA(cudaStreamSynchronize(ctx->stream));
                const int it = S->it;
                launch_counter().fetch_add(n_pro + int64_t(it) * n_body, std::memory_order_relaxed);
                if (history) std::memcpy(history, hs.data() + kSolveHist, sizeof(double) * (it + 1));
                if (iters) *iters = it;
                const auto T2 = tnow();
                if (it == 0) std::memset(x_host, 0, sizeof(double) * n);  // x = 0 exactly (no cycle ran)
                else if (!(x_pinned && !solve_snap_in_loop())) parallel_memcpy(x_host, m.h_stage_x, sizeof(double) * n);
                if (timing)
                    fprintf(stderr, "[solve_host] device loop: h2d %.3f ms, %d cycles %.3f ms, d2h %.3f ms\n",
                            tsec(T0, T0b), it, tsec(T0b, T2), tsec(T2, tnow()));
                return;
            }
        }
        // host-driven loop (device loop disabled or rejected by the driver)
        LDGMG_CUDA(cudaMemsetAsync(x.p, 0, sizeof(double) * n, ctx->stream));
        launch_dot(*ctx, n, b.as<double>(), b.as<double>(), ctx->d_red);
        LDGMG_CUDA(cudaMemcpyAsync(ctx->h_red, ctx->d_red, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        LDGMG_CUDA(cudaStreamSynchronize(ctx->stream));
        const double bn = std::sqrt(ctx->h_red[0]);
        const auto T1 = tnow();
        auto relres = [&]() {
            RowPass p;
            p.A = m.A[0];
            p.mode = MODE_RESIDUAL;
            p.x = x.as<double>();
            p.b = b.as<double>();
            p.y = rbuf;
            p.nrows = m.A[0]->brows;
            launch_rowpass(*ctx, p);
            launch_dot(*ctx, n, rbuf, rbuf, ctx->d_red);
            LDGMG_CUDA(cudaMemcpyAsync(ctx->h_red, ctx->d_red, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
            LDGMG_CUDA(cudaStreamSynchronize(ctx->stream));
            return bn > 0 ? std::sqrt(ctx->h_red[0]) / bn : std::sqrt(ctx->h_red[0]);
        };
        // Every iterate is snapshotted on the device and its copy to the host
        // runs on a side stream under the next residual check and cycle, so
        // the converged x is already in pinned memory when the loop exits.
        bool snapped = false;
        auto snapshot = [&]() {
            if (snapped) LDGMG_CUDA(cudaStreamWaitEvent(ctx->stream, m.ev_d2h, 0));  // previous copy done
            LDGMG_CUDA(cudaMemcpyAsync(m.solve_xs.p, x.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
            LDGMG_CUDA(cudaEventRecord(m.ev_snap, ctx->stream));
            LDGMG_CUDA(cudaStreamWaitEvent(m.d2h_stream, m.ev_snap, 0));
            LDGMG_CUDA(cudaMemcpyAsync(m.h_stage_x, m.solve_xs.p, sizeof(double) * n, cudaMemcpyDeviceToHost,
                                       m.d2h_stream));
            LDGMG_CUDA(cudaEventRecord(m.ev_d2h, m.d2h_stream));
            snapped = true;
        };
        double rr = relres();
        if (history) history[0] = rr;
        int it = 0;
        while (rr > tol && it < maxit) {
            m.cycles(*ctx, x.as<double>(), b.as<double>(), 1, reuse);
            ++it;
            snapshot();
            rr = relres();
            if (history) history[it] = rr;
        }
        if (iters) *iters = it;
        const auto T2 = tnow();
        if (snapped) {
            LDGMG_CUDA(cudaEventSynchronize(m.ev_d2h));
            parallel_memcpy(x_host, m.h_stage_x, sizeof(double) * n);
        } else {
            std::memset(x_host, 0, sizeof(double) * n);  // x = 0 exactly (no cycle ran)
        }
        if (timing)
            fprintf(stderr, "[solve_host] h2d %.3f norm %.3f ms, %d cycles+checks %.3f ms, d2h %.3f ms\n",
                    tsec(T0, T0b), tsec(T0b, T1), it, tsec(T1, T2), tsec(T2, tnow()));
    });
}

int ldgmg_mg_set_strict_order(ldgmg_mg* mg, int strict) {
    return guarded([&] {
        need(mg, "mg_set_strict_order");
        mg->m.strict_order = strict != 0;
        mg->m.invalidate_graphs();
    });
}

int ldgmg_mg_setup(ldgmg_ctx* ctx, ldgmg_mg* mg) {
    return guarded([&] {
        need(ctx, "mg_setup");
        need(mg, "mg_setup");
        bind(*ctx);
        ensure_smoothers(ctx, mg->m);
    });
}

int ldgmg_mg_cycle_costs(const ldgmg_mg* mg, double* dof_updates, double* alg_bytes) {
    return guarded([&] {
        need(mg, "mg_cycle_costs");
        for (int l = 0; l + 1 < mg->m.depth; ++l)
            if (!mg->m.sm[l]) fail(LDGMG_ERR_LOGIC, "multigrid: smoothers not built yet");
        if (dof_updates) *dof_updates = mg->m.dof_updates_per_cycle();
        if (alg_bytes) *alg_bytes = mg->m.bytes_per_cycle();
    });
}

int ldgmg_mg_destroy(ldgmg_mg* mg) {
    return guarded([&] { delete mg; });
}

// ---------------------------------------------------------------- Krylov
static void report_out(const SolveReport& r, ldgmg_solve_report* rep) {
    rep->n_residuals = int(r.residuals.size());
    if (rep->residuals) {
        if (rep->capacity < rep->n_residuals) fail(LDGMG_ERR_INVALID_ARGUMENT, "solve report: residual buffer too small");
        std::memcpy(rep->residuals, r.residuals.data(), sizeof(double) * r.residuals.size());
    }
    rep->iterations = r.iterations;
    rep->converged = r.converged;
    rep->breakdown = r.breakdown;
    rep->rho = r.rho;
    rep->eta = r.eta;
    rep->classification = r.classification;
    rep->low_confidence = r.low_confidence;
}

int ldgmg_krylov_solve(ldgmg_ctx* ctx, ldgmg_mg* mg, int kind, const double* b, double* x, double tol, int maxit,
                       ldgmg_solve_report* rep) {
    return guarded([&] {
        need(ctx, "krylov_solve");
        need(mg, "krylov_solve");
        need(rep, "krylov_solve(report)");
        ensure_smoothers(ctx, mg->m);
        const SolveReport r = kind == LDGMG_KRYLOV_CG ? pcg(*ctx, mg->m, b, x, tol, maxit)
                                                      : gmres_left(*ctx, mg->m, b, x, tol, maxit);
        report_out(r, rep);
    });
}

int ldgmg_estimate_eta(ldgmg_ctx* ctx, ldgmg_mg* mg, int kind, uint64_t seed, double tol, int maxit,
                       ldgmg_solve_report* rep) {
    return guarded([&] {
        need(ctx, "estimate_eta");
        need(mg, "estimate_eta");
        need(rep, "estimate_eta(report)");
        ensure_smoothers(ctx, mg->m);
        report_out(estimate_eta(*ctx, mg->m, kind, seed, tol, maxit), rep);
    });
}

// ------------------------------------------------------ host setup (L0/L2)
int ldgmg_problem_create(const ldgmg_problem_spec* spec, int min_depth, int bottom_max_elements,
                         ldgmg_problem** out) {
    return guarded([&] {
        need(spec, "problem_create");
        need(out, "problem_create");
        auto* h = new ldgmg_problem();
        try {
            problem_build(*spec, min_depth, bottom_max_elements, h->p);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int ldgmg_problem_create_partial(const ldgmg_problem_spec* spec, int min_depth, int bottom_max_elements,
                                 int nranks, int rank, int halo_hops, int min_rows_per_rank,
                                 ldgmg_problem** out) {
    return guarded([&] {
        need(spec, "problem_create_partial");
        need(out, "problem_create_partial");
        auto* h = new ldgmg_problem();
        try {
            problem_build_partial(*spec, min_depth, bottom_max_elements, nranks, rank, halo_hops, min_rows_per_rank,
                                  h->p);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int ldgmg_problem_create_ex(const ldgmg_problem_spec* spec, int min_depth, int bottom_max_elements, int nranks,
                            int rank, int halo_hops, int min_rows_per_rank, int flags, ldgmg_problem** out) {
    return guarded([&] {
        need(spec, "problem_create_ex");
        need(out, "problem_create_ex");
        auto* h = new ldgmg_problem();
        try {
            problem_build_partial(*spec, min_depth, bottom_max_elements, nranks, rank, halo_hops, min_rows_per_rank,
                                  h->p, (flags & LDGMG_PROBLEM_DEVICE_ASSEMBLY) != 0, (flags & LDGMG_PROBLEM_ANY_N) != 0);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

static std::unique_ptr<Bsr> level_operator(Ctx& ctx, const Problem& p, int l) {
    const auto& L = p.levels[l];
    if (L.deferred) return assemble_on_device(ctx, L.prog);
    return bsr_upload(ctx, L.A.brows, L.A.brows, L.A.bs, L.A.bs, L.A.ptr.data(), L.A.col.data(), L.A.val.data());
}

int ldgmg_problem_device_operator(ldgmg_ctx* ctx, const ldgmg_problem* P, int level, ldgmg_bsr** out) {
    return guarded([&] {
        need(ctx, "problem_device_operator");
        need(P, "problem_device_operator");
        need(out, "problem_device_operator(out)");
        if (level < 0 || level >= int(P->p.levels.size())) fail(LDGMG_ERR_INVALID_ARGUMENT, "problem: bad level");
        bind(*ctx);
        *out = static_cast<ldgmg_bsr*>(own_bsr(level_operator(*ctx, P->p, level)));
    });
}

int ldgmg_problem_level_partial(const ldgmg_problem* P, int level) {
    if (!P || level < 0 || level >= int(P->p.levels.size())) return 0;
    return P->p.levels[level].partial ? 1 : 0;
}

int ldgmg_sai_build(ldgmg_ctx* ctx, const ldgmg_bsr* A, int system_kind, int n_velocity, int level, double zeta,
                    int cache, const int* col_mask, ldgmg_bsr** B, ldgmg_sai_stats* stats) {
    return guarded([&] {
        need(ctx, "build_sai");
        need(A, "build_sai");
        need(B, "build_sai(B)");
        bind(*ctx);
        std::vector<char> mask;
        if (col_mask) {
            mask.resize(A->brows);
            for (int j = 0; j < A->brows; ++j) mask[j] = col_mask[j] != 0;
        }
        SaiResult r = build_sai_gpu(*ctx, *A, system_kind, n_velocity, level, zeta, cache != 0, nullptr,
                                    col_mask ? &mask : nullptr);
        if (stats) *stats = r.stats;
        *B = static_cast<ldgmg_bsr*>(own_bsr(std::move(r.B)));
    });
}

int ldgmg_problem_depth(const ldgmg_problem* P) { return P ? int(P->p.levels.size()) : 0; }

int ldgmg_problem_level_shape(const ldgmg_problem* P, int level, int* n_elements, int* bs, int64_t* nnzb) {
    return guarded([&] {
        need(P, "problem_level_shape");
        if (level < 0 || level >= int(P->p.levels.size())) fail(LDGMG_ERR_INVALID_ARGUMENT, "problem: bad level");
        const auto& L = P->p.levels[level];
        if (n_elements) *n_elements = L.A.brows;
        if (bs) *bs = L.A.bs;
        if (nnzb) *nnzb = int64_t(L.A.col.size());
    });
}

int ldgmg_problem_level_matrix(const ldgmg_problem* P, int level, int* ptr, int* col, double* val) {
    return guarded([&] {
        need(P, "problem_level_matrix");
        if (level < 0 || level >= int(P->p.levels.size())) fail(LDGMG_ERR_INVALID_ARGUMENT, "problem: bad level");
        const auto& A = P->p.levels[level].A;
        if (val && P->p.levels[level].deferred)
            fail(LDGMG_ERR_LOGIC, "problem: operator assembled on the device (use ldgmg_problem_device_operator)");
        if (ptr) std::memcpy(ptr, A.ptr.data(), sizeof(int) * A.ptr.size());
        if (col) std::memcpy(col, A.col.data(), sizeof(int) * A.col.size());
        if (val) std::memcpy(val, A.val.data(), sizeof(double) * A.val.size());
    });
}

int ldgmg_problem_level_transfer(const ldgmg_problem* P, int level, int* parent_of, int* orthant_of) {
    return guarded([&] {
        need(P, "problem_level_transfer");
        if (level < 0 || level + 1 >= int(P->p.levels.size()))
            fail(LDGMG_ERR_INVALID_ARGUMENT, "problem: bottom level has no transfer");
        const auto& L = P->p.levels[level];
        if (parent_of) std::memcpy(parent_of, L.parent_of.data(), sizeof(int) * L.parent_of.size());
        if (orthant_of) std::memcpy(orthant_of, L.orthant_of.data(), sizeof(int) * L.orthant_of.size());
    });
}

int ldgmg_problem_info(const ldgmg_problem* P, int* dim, int* n_comp, int* bs_scalar, int* kernel_constants,
                       int* kernel_pressure, int* n_velocity) {
    return guarded([&] {
        need(P, "problem_info");
        const Problem& p = P->p;
        if (dim) *dim = p.dim;
        if (n_comp) *n_comp = p.n_comp;
        if (bs_scalar) *bs_scalar = p.bs_scalar;
        if (kernel_constants) *kernel_constants = p.kernel_constants;
        if (kernel_pressure) *kernel_pressure = p.kernel_pressure;
        if (n_velocity) *n_velocity = p.kind == LDGMG_SYSTEM_STOKES ? p.dim * p.bs_scalar : 0;
    });
}

int ldgmg_problem_injection(const ldgmg_problem* P, double* K) {
    return guarded([&] {
        need(P, "problem_injection");
        need(K, "problem_injection(K)");
        std::memcpy(K, P->p.inject.data(), sizeof(double) * P->p.inject.size());
    });
}

int ldgmg_mg_create_from_problem(ldgmg_ctx* ctx, const ldgmg_problem* P, const ldgmg_mg_config* cfg,
                                 ldgmg_mg** out) {
    ldgmg_mg* h = nullptr;
    const int rc = guarded([&] {
        need(ctx, "mg_create_from_problem");
        need(P, "mg_create_from_problem");
        need(cfg, "mg_create_from_problem(cfg)");
        bind(*ctx);
        const Problem& p = P->p;
        h = new ldgmg_mg();
        Mg& m = h->m;
        m.depth = int(p.levels.size());
        m.cfg = *cfg;
        m.system_kind = p.kind;
        m.dim = p.dim;
        m.n_comp = p.n_comp;
        m.bs_scalar = p.bs_scalar;
        m.kernel_constants = p.kernel_constants;
        m.kernel_pressure = p.kernel_pressure;
        m.n_velocity = p.kind == LDGMG_SYSTEM_STOKES ? p.dim * p.bs_scalar : 0;
        SetupTimer tm("mg_create_from_problem", ctx->stream);
        for (int l = 0; l < m.depth; ++l) {
            m.own_A.push_back(level_operator(*ctx, p, l));
            m.A.push_back(m.own_A.back().get());
        }
        tm.stamp("operator upload");
        for (int l = 0; l + 1 < m.depth; ++l) {
            const auto& L = p.levels[l];
            m.own_T.push_back(transfer_create(*ctx, L.A.brows, p.levels[l + 1].A.brows, L.parent_of.data(),
                                              L.orthant_of.data(), p.dim, p.bs_scalar, p.n_comp,
                                              p.inject.data()));
            m.T.push_back(m.own_T.back().get());
        }
        tm.stamp("transfers");
        m.init(*ctx);
        tm.stamp("level scratch");
        m.set_bottom(*ctx, nullptr, nullptr);
        tm.stamp("bottom pseudoinverse");
        m.sm.assign(m.depth, nullptr);
        mg_default_smoothers(ctx, m);
        tm.stamp("smoothers");
        *out = h;
    });
    if (rc != LDGMG_OK) delete h;
    return rc;
}

int ldgmg_problem_destroy(ldgmg_problem* P) {
    return guarded([&] { delete P; });
}

int ldgmg_injection_matrices(int dim, int degree, double* K) {
    return guarded([&] {
        need(K, "injection_matrices");
        if (dim != 2 && dim != 3) fail(LDGMG_ERR_INVALID_ARGUMENT, "basis: dim must be 2 or 3");
        const std::vector<double> v = injection_matrices(dim, degree);
        std::memcpy(K, v.data(), sizeof(double) * v.size());
    });
}

int ldgmg_random_rhs(int nblocks, int bs, uint64_t seed, double* out) {
    return guarded([&] {
        need(out, "random_rhs");
        std::mt19937_64 rng(seed);
        const size_t n = size_t(nblocks) * bs;
        for (size_t i = 0; i < n; ++i) {
            const double u = double(rng() >> 11) * 0x1.0p-53;
            out[i] = 2.0 * u - 1.0;
        }
    });
}

}  // extern "C"
