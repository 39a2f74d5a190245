#pragma once

#include <functional>
#include <vector>

namespace ldgmg_b200 {

/// Symmetric eigendecomposition (host, setup only): A n x n column-major;
/// lambda ascending; V column-major eigenvectors.
void sym_eig_host(int n, const double* A, double* lambda, double* V);

/// Split [0, n) over the host threads; body(lo, hi).
void parallel_for(int n, const std::function<void(int, int)>& body);
/// memcpy split over up to 8 host threads (pageable <-> pinned staging)
void parallel_memcpy(void* dst, const void* src, size_t bytes);

}  // namespace ldgmg_b200
