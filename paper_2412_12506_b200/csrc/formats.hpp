// Block-coordinate text format of the reference (dump_block_coo,
// blockla.hpp:253-268): header "blockcoo brows bcols row_bs col_bs nnzb",
// then one "i j v00 v01 ..." line per block in CSR order, row-major block
// values printed with 17 significant digits (bit-exact round trip).
#pragma once

#include <cstdint>
#include <vector>

namespace ldgmg_b200 {

struct CooMatrix {
    int brows = 0, bcols = 0, rbs = 0, cbs = 0;
    std::vector<int> ptr, col;
    std::vector<double> val;  // row-major blocks, CSR order
};

/// Writes the reference's text for a CSR matrix with row-major blocks.
void coo_write(const char* path, int brows, int bcols, int rbs, int cbs, const int* ptr, const int* col,
               const double* val);
/// Parses a dump the way the reference's round-trip test rebuilds it
/// (tests/test_blockla.cpp:207-230): blocks accumulate through a
/// BlockBuilder (zero-initialised, `+= 1.0 * v`, duplicates summed in file
/// order), rows come out with ascending columns.
CooMatrix coo_read(const char* path);

}  // namespace ldgmg_b200
