// cbg_mm.cpp -- MatrixMarket coordinate I/O for the drop-in CsrMatrix
// (reference interface sparse.hpp:36-38, behaviour of sparse.cpp:113-231:
// 'matrix coordinate real general|symmetric', 1-based indices, symmetric
// off-diagonals mirrored, duplicates summed, columns ascending per row,
// "matrix market: line N: <reason>" runtime errors; values written %.17g).
// Host-side I/O feeding the device solver; rows are bucketed by a counting
// pass instead of a global sort.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <istream>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "cbg/sparse.hpp"

namespace cbg {

namespace {

struct LineReader {
    std::istream& is;
    size_t no = 0;
    bool next(std::string& out) {
        if (!std::getline(is, out)) return false;
        ++no;
        return true;
    }
};

[[noreturn]] void fail_at(size_t line, const std::string& why) {
    throw std::runtime_error("matrix market: line " + std::to_string(line) + ": " + why);
}

bool blank(const std::string& s) { return s.find_first_not_of(" \t\r") == std::string::npos; }

std::string lowered(std::string s) {
    std::transform(s.begin(), s.end(), s.begin(), [](unsigned char c) { return static_cast<char>(std::tolower(c)); });
    return s;
}

double to_double(const std::string& tok, size_t line) {
    double v = 0.0;
    const auto res = std::from_chars(tok.data(), tok.data() + tok.size(), v);
    if (res.ec != std::errc{} || res.ptr != tok.data() + tok.size()) fail_at(line, "bad numeric value '" + tok + "'");
    return v;
}

struct Triple {
    size_t r, c;
    double v;
};

}  // namespace

CsrMatrix parse_matrix_market(std::istream& is) {
    LineReader in{is};
    std::string line;
    if (!in.next(line)) fail_at(1, "empty file");
    {
        std::istringstream hdr(line);
        std::string tag, object, format, field, symmetry;
        hdr >> tag >> object >> format >> field >> symmetry;
        if (tag != "%%MatrixMarket") fail_at(in.no, "missing %%MatrixMarket banner");
        if (lowered(object) != "matrix" || lowered(format) != "coordinate")
            fail_at(in.no, "only 'matrix coordinate' files are supported");
        if (lowered(field) != "real") fail_at(in.no, "unsupported field '" + lowered(field) + "'");
        symmetry = lowered(symmetry);
        if (symmetry != "symmetric" && symmetry != "general") fail_at(in.no, "unsupported symmetry '" + symmetry + "'");
        line = symmetry;  // keep for below
    }
    const bool symmetric = line == "symmetric";
    size_t rows = 0, cols = 0, declared = 0;
    for (;;) {
        if (!in.next(line)) fail_at(in.no + 1, "missing size line");
        if (!line.empty() && line[0] == '%') continue;
        std::istringstream sz(line);
        if (sz >> rows >> cols >> declared) break;
        if (!blank(line)) fail_at(in.no, "bad size line");
    }
    std::vector<Triple> t;
    t.reserve(symmetric ? 2 * declared : declared);
    for (size_t got = 0; got < declared;) {
        if (!in.next(line)) fail_at(in.no + 1, "unexpected end of file");
        if (line.empty() || line[0] == '%' || blank(line)) continue;
        std::istringstream e(line);
        size_t i = 0, j = 0;
        std::string tok;
        if (!(e >> i >> j >> tok)) fail_at(in.no, "bad entry");
        const double v = to_double(tok, in.no);
        if (i < 1 || i > rows || j < 1 || j > cols) fail_at(in.no, "index out of bounds");
        t.push_back({i - 1, j - 1, v});
        if (symmetric && i != j) t.push_back({j - 1, i - 1, v});
        ++got;
    }
    // bucket by row (file order kept), then order each row's columns and
    // sum duplicates in file order
    std::vector<size_t> start(rows + 1, 0);
    for (const Triple& x : t) ++start[x.r + 1];
    for (size_t r = 0; r < rows; ++r) start[r + 1] += start[r];
    std::vector<Triple> byrow(t.size());
    {
        std::vector<size_t> fill(start.begin(), start.end() - 1);
        for (const Triple& x : t) byrow[fill[x.r]++] = x;
    }
    CsrMatrix a;
    a.n_rows = rows;
    a.n_cols = cols;
    a.row_ptrs.assign(rows + 1, 0);
    a.col_idx.reserve(t.size());
    a.values.reserve(t.size());
    for (size_t r = 0; r < rows; ++r) {
        auto first = byrow.begin() + static_cast<std::ptrdiff_t>(start[r]);
        auto last = byrow.begin() + static_cast<std::ptrdiff_t>(start[r + 1]);
        std::stable_sort(first, last, [](const Triple& x, const Triple& y) { return x.c < y.c; });
        for (auto it = first; it != last;) {
            double sum = 0.0;
            const size_t c = it->c;
            for (; it != last && it->c == c; ++it) sum += it->v;
            a.col_idx.push_back(c);
            a.values.push_back(sum);
        }
        a.row_ptrs[r + 1] = a.values.size();
    }
    return a;
}

void write_matrix_market(std::ostream& os, const CsrMatrix& a) {
    os << "%%MatrixMarket matrix coordinate real general\n" << a.n_rows << " " << a.n_cols << " " << a.nnz() << "\n";
    char num[64];
    for (size_t r = 0; r < a.n_rows; ++r)
        for (size_t k = a.row_ptrs[r]; k < a.row_ptrs[r + 1]; ++k) {
            std::snprintf(num, sizeof num, "%.17g", a.values[k]);
            os << r + 1 << " " << a.col_idx[k] + 1 << " " << num << "\n";
        }
    if (!os) throw std::runtime_error("matrix market: write failed");
}

}  // namespace cbg
