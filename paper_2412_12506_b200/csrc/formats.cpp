// Block-coordinate text I/O (formats.hpp).
#include "formats.hpp"

#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>

namespace ldgmg_b200 {

namespace {
struct FileCloser {
    void operator()(FILE* f) const {
        if (f) std::fclose(f);
    }
};
using File = std::unique_ptr<FILE, FileCloser>;
}  // namespace

void coo_write(const char* path, int brows, int bcols, int rbs, int cbs, const int* ptr, const int* col,
               const double* val) {
    if (!path) throw std::invalid_argument("dump_block_coo: null path");
    if (brows < 0 || bcols < 0 || rbs <= 0 || cbs <= 0) throw std::invalid_argument("dump_block_coo: bad shape");
    File f(std::fopen(path, "w"));
    if (!f) throw std::runtime_error(std::string("dump_block_coo: cannot open ") + path);
    const size_t nnzb = brows ? size_t(ptr[brows]) : 0;
    std::fprintf(f.get(), "blockcoo %d %d %d %d %zu\n", brows, bcols, rbs, cbs, nnzb);
    const size_t bb = size_t(rbs) * cbs;
    std::string line;
    char buf[40];
    for (int i = 0; i < brows; ++i)
        for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
            line.clear();
            std::snprintf(buf, sizeof buf, "%d %d", i, col[k]);
            line += buf;
            const double* b = val + size_t(k) * bb;
            for (size_t t = 0; t < bb; ++t) {
                // std::ostream with precision(17) and the default float field
                // formats as printf %.17g
                std::snprintf(buf, sizeof buf, " %.17g", b[t]);
                line += buf;
            }
            line += '\n';
            if (std::fwrite(line.data(), 1, line.size(), f.get()) != line.size())
                throw std::runtime_error("dump_block_coo: write failed");
        }
}

namespace {
struct Reader {
    std::string text;
    size_t pos = 0;
    bool token(std::string& out) {
        while (pos < text.size() && std::isspace(static_cast<unsigned char>(text[pos]))) ++pos;
        if (pos >= text.size()) return false;
        const size_t s = pos;
        while (pos < text.size() && !std::isspace(static_cast<unsigned char>(text[pos]))) ++pos;
        out.assign(text, s, pos - s);
        return true;
    }
    long long integer() {
        std::string t;
        if (!token(t)) throw std::runtime_error("blockcoo: truncated input");
        char* end = nullptr;
        errno = 0;
        const long long v = std::strtoll(t.c_str(), &end, 10);
        if (errno || !end || *end) throw std::runtime_error("blockcoo: bad integer '" + t + "'");
        return v;
    }
    double real() {
        std::string t;
        if (!token(t)) throw std::runtime_error("blockcoo: truncated input");
        char* end = nullptr;
        const double v = std::strtod(t.c_str(), &end);
        if (!end || *end) throw std::runtime_error("blockcoo: bad number '" + t + "'");
        return v;
    }
};
}  // namespace

CooMatrix coo_read(const char* path) {
    if (!path) throw std::invalid_argument("blockcoo: null path");
    File f(std::fopen(path, "rb"));
    if (!f) throw std::runtime_error(std::string("blockcoo: cannot open ") + path);
    Reader r;
    char buf[1 << 16];
    size_t n;
    while ((n = std::fread(buf, 1, sizeof buf, f.get())) > 0) r.text.append(buf, n);
    std::string tag;
    if (!r.token(tag) || tag != "blockcoo") throw std::runtime_error("blockcoo: missing header");
    CooMatrix M;
    M.brows = int(r.integer());
    M.bcols = int(r.integer());
    M.rbs = int(r.integer());
    M.cbs = int(r.integer());
    const long long nnzb = r.integer();
    if (M.brows < 0 || M.bcols < 0 || M.rbs <= 0 || M.cbs <= 0 || nnzb < 0)
        throw std::runtime_error("blockcoo: bad header");
    const size_t bb = size_t(M.rbs) * M.cbs;
    std::vector<std::map<int, std::vector<double>>> rows(M.brows);
    std::vector<double> blk(bb);
    for (long long k = 0; k < nnzb; ++k) {
        const long long i = r.integer(), j = r.integer();
        if (i < 0 || i >= M.brows || j < 0 || j >= M.bcols) throw std::runtime_error("blockcoo: index out of range");
        for (auto& v : blk) v = r.real();
        auto& cell = rows[i][int(j)];
        if (cell.empty()) cell.assign(bb, 0.0);
        for (size_t t = 0; t < bb; ++t) cell[t] += 1.0 * blk[t];  // BlockBuilder::add_block
    }
    M.ptr.assign(M.brows + 1, 0);
    for (int i = 0; i < M.brows; ++i) M.ptr[i + 1] = M.ptr[i] + int(rows[i].size());
    M.col.reserve(M.ptr[M.brows]);
    M.val.reserve(size_t(M.ptr[M.brows]) * bb);
    for (int i = 0; i < M.brows; ++i)
        for (auto& [j, b] : rows[i]) {
            M.col.push_back(j);
            M.val.insert(M.val.end(), b.begin(), b.end());
        }
    return M;
}

}  // namespace ldgmg_b200
