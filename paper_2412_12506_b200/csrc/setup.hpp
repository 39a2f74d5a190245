// Built-in host setup: uniform Morton meshes, the coarsening chain and the
// LDG scalar / Stokes operators per level (the L0/L2 producers the V-cycle
// consumes; the reference's mesh.hpp, basis.hpp, ldg_core.hpp, ldg_scalar.hpp,
// ldg_stokes.hpp and multigrid.hpp:168-241, restated).  Host C++, threaded
// over element rows.  The accumulation order of every block follows the
// reference (BlockBuilder insertion order, accumulate_AtDB source order,
// face_block loop nest), so the operators come out bit-identical to the
// oracle build (tests/test_setup_parity.py).
#pragma once

#include <array>
#include <sys/mman.h>

#include <cstdlib>
#include <memory>
#include <new>
#include <utility>
#include <vector>

#include "../../include/ldgmg_b200.h"

namespace ldgmg_b200 {

/// cudaHostAlloc when a CUDA device is visible and LDGMG_PINNED_SETUP=1
/// (nullptr otherwise); pinned_free returns false for non-pinned pointers.
void* pinned_alloc(size_t bytes);
bool pinned_free(void* p);

/// std::allocator that default-initialises (no zero fill on resize): the
/// operator values are written exactly once by the (threaded) assembly, so
/// zeroing gigabytes first only costs a serial memset and the page faults.
template <class T>
struct DefaultInitAlloc : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = DefaultInitAlloc<U>;
    };
    DefaultInitAlloc() = default;
    template <class U>
    DefaultInitAlloc(const DefaultInitAlloc<U>&) noexcept {}
    template <class U>
    void construct(U* p) noexcept {
        ::new (static_cast<void*>(p)) U;
    }
    template <class U, class... Args>
    void construct(U* p, Args&&... args) {
        ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
    }
    /// large arrays: 2 MiB-aligned and advised for transparent huge pages
    /// (first-touch faults of multi-GB operators dominate the CSR fill)
    T* allocate(size_t n) {
        const size_t bytes = n * sizeof(T);
        if (bytes < (size_t(64) << 20)) return std::allocator<T>::allocate(n);
        // page-locked on request (LDGMG_PINNED_SETUP=1: the operator upload is
        // then a plain DMA); else 2 MiB-aligned, huge-page advised
        if (void* p = pinned_alloc(bytes)) return static_cast<T*>(p);
        const size_t huge = size_t(2) << 20;
        void* p = std::aligned_alloc(huge, (bytes + huge - 1) / huge * huge);
        if (!p) throw std::bad_alloc();
        madvise(p, (bytes + huge - 1) / huge * huge, MADV_HUGEPAGE);
        return static_cast<T*>(p);
    }
    void deallocate(T* p, size_t n) {
        if (n * sizeof(T) < (size_t(64) << 20))
            std::allocator<T>::deallocate(p, n);
        else if (!pinned_free(p))
            std::free(p);
    }
};

struct HostCsr {
    int brows = 0, bs = 0;
    std::vector<int> ptr, col;
    std::vector<double, DefaultInitAlloc<double>> val;
};

/// Device-assembly program of one level operator (problem_build with
/// deferred assembly): every operator block as the host assembly computes it,
/// recorded instead of evaluated so the GPU (assembly_gpu.cu) can evaluate it
/// in the same order, bit for bit.
///   inner block  v = ((0 + d_1 B1_1^T B2_1) + d_2 B1_2^T B2_2 + ...) [+ 1.0 S]
///                (the G_k^T D G_k accumulation of accumulate_AtDB plus the
///                penalty block; bsv x bsv)
///   final block  per sub-block (ncomp x ncomp of bsv x bsv): acc = 0, then
///                per term: acc += scale * X, X an inner block, a stored block
///                or a stored block transposed; kind 3 = the inner block
///                itself (scalar operators); kind 4 = +scale on the diagonal.
struct LevelProgram {
    int n = 0, bs = 0, bsv = 0, ncomp = 1;
    std::vector<int> ptr, col;                          // final pattern
    std::vector<double, DefaultInitAlloc<double>> blocks;  // stored bsv^2 blocks (row-major)
    std::vector<int64_t> inner_ptr{0};                   // prods of inner block i
    std::vector<int> prod_b1, prod_b2, inner_add;        // block ids; add: -1 none
    std::vector<double> prod_d;
    std::vector<int64_t> term_ptr{0};                    // per (cell, sub-block)
    std::vector<int> term_kind, term_idx;
    std::vector<double> term_scale;
};

struct ProblemLevel {
    int n = 0;  // elements per axis
    HostCsr A;
    std::vector<int> phase;
    std::vector<int> parent_of, orthant_of;  // to the next coarser level
    bool partial = false;  // only the rank's rows + halo assembled (others empty)
    bool deferred = false;  // A not built on the host: `prog` holds the device-assembly program
    LevelProgram prog;
};

struct Problem {
    ldgmg_problem_spec spec{};
    int kind = 0, dim = 2, degree = 1, n_comp = 1, bs_scalar = 1;
    int kernel_constants = 0, kernel_pressure = 0;
    std::vector<ProblemLevel> levels;
    std::vector<double> inject;  // 2^dim matrices bs_scalar^2, row-major
};

void problem_build(const ldgmg_problem_spec& spec, int min_depth, int bottom_max_elements,
                   Problem& out);
/// Distributed setup: levels with >= nranks*min_rows_per_rank elements (all
/// but the last) assemble only the rows of rank `rank`'s contiguous range
/// [rank*N/P, (rank+1)*N/P) plus `halo_hops` face layers; every assembled
/// row is bit-identical to problem_build's.  Smaller levels are complete.
void problem_build_partial(const ldgmg_problem_spec& spec, int min_depth, int bottom_max_elements, int nranks,
                           int rank, int halo_hops, int min_rows_per_rank, Problem& out, bool deferred = false,
                           bool any_n = false);

std::vector<double> injection_matrices(int dim, int degree);

}  // namespace ldgmg_b200
