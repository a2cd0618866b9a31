// Matrix Market I/O (core/matrix_market.hpp:63-168; instance export
// synth.hpp:152-168): host code, same formats and errors as the reference --
// "array real general" dense files column-major at 17 significant digits,
// "coordinate real general" sparse files with 1-based indices in
// column-major (CSC) order; readers accept real/double/integer fields and
// general symmetry only, skip % comments and blank lines, reject
// non-finite values, out-of-range indices and duplicate entries.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "matrix_market.hpp"

namespace blws {
namespace {

std::string lower(std::string s) {
    std::transform(s.begin(), s.end(), s.begin(), [](unsigned char c) { return static_cast<char>(std::tolower(c)); });
    return s;
}

std::string next_data_line(std::istream& in) {
    std::string line;
    while (std::getline(in, line)) {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty() || line[0] == '%') continue;
        return line;
    }
    throw IoError("matrix market: unexpected end of file");
}

bool read_header(std::istream& in) {  // true: coordinate
    std::string line;
    if (!std::getline(in, line)) throw IoError("matrix market: empty stream");
    std::istringstream hs(line);
    std::string banner, object, format, field, symmetry;
    hs >> banner >> object >> format >> field >> symmetry;
    if (banner != "%%MatrixMarket" || lower(object) != "matrix") throw IoError("matrix market: bad banner");
    format = lower(format);
    field = lower(field);
    symmetry = lower(symmetry);
    if (field != "real" && field != "double" && field != "integer")
        throw IoError("matrix market: only real matrices are supported");
    if (symmetry != "general") throw IoError("matrix market: only general symmetry is supported");
    if (format == "coordinate") return true;
    if (format != "array") throw IoError("matrix market: unknown format '" + format + "'");
    return false;
}

std::ifstream open_in(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw IoError("matrix market: cannot open " + path);
    return f;
}

void put(std::ostream& out, double v) {
    char b[40];
    std::snprintf(b, sizeof(b), "%.17g", v);  // the reference's precision(17)
    out << b;
}

}  // namespace

void mm_write_dense(const std::string& path, Index rows, Index cols, const double* a, Index lda) {
    std::ofstream out(path);
    if (!out) throw IoError("matrix market: cannot open " + path);
    out << "%%MatrixMarket matrix array real general\n" << rows << " " << cols << "\n";
    for (Index j = 0; j < cols; ++j)
        for (Index i = 0; i < rows; ++i) {
            put(out, a[i + j * lda]);
            out << "\n";
        }
    if (!out) throw IoError("matrix market: write failed " + path);
}

void mm_write_sparse(const std::string& path, Index rows, Index cols, Index nnz, const std::int64_t* colptr,
                     const std::int32_t* rowidx, const double* values) {
    std::ofstream out(path);
    if (!out) throw IoError("matrix market: cannot open " + path);
    out << "%%MatrixMarket matrix coordinate real general\n" << rows << " " << cols << " " << nnz << "\n";
    for (Index j = 0; j < cols; ++j)
        for (std::int64_t p = colptr[j]; p < colptr[j + 1]; ++p) {
            out << rowidx[p] + 1 << " " << j + 1 << " ";
            put(out, values[p]);
            out << "\n";
        }
    if (!out) throw IoError("matrix market: write failed " + path);
}

void mm_read_dense(const std::string& path, Index* rows, Index* cols, std::vector<double>* data) {
    std::ifstream in = open_in(path);
    if (read_header(in)) throw IoError("matrix market: expected array format, got coordinate");
    std::istringstream sizes(next_data_line(in));
    Index r = 0, c = 0;
    if (!(sizes >> r >> c) || r <= 0 || c <= 0) throw IoError("matrix market: bad size line");
    *rows = r;
    *cols = c;
    if (!data) return;
    data->resize(static_cast<size_t>(r * c));
    for (Index k = 0; k < r * c; ++k) {
        std::istringstream vs(next_data_line(in));
        double v;
        if (!(vs >> v)) throw IoError("matrix market: bad value");
        if (!std::isfinite(v)) throw IoError("matrix market: non-finite value");
        (*data)[static_cast<size_t>(k)] = v;  // column-major, as written
    }
}

void mm_read_sparse(const std::string& path, Index* rows, Index* cols, std::vector<std::int64_t>* colptr,
                    std::vector<std::int32_t>* rowidx, std::vector<double>* values) {
    std::ifstream in = open_in(path);
    if (!read_header(in)) throw IoError("matrix market: expected coordinate format, got array");
    std::istringstream sizes(next_data_line(in));
    Index r = 0, c = 0, nnz = 0;
    if (!(sizes >> r >> c >> nnz) || r <= 0 || c <= 0 || nnz < 0) throw IoError("matrix market: bad size line");
    *rows = r;
    *cols = c;
    struct E {
        Index j, i;
        double v;
    };
    std::vector<E> es;
    es.reserve(static_cast<size_t>(nnz));
    for (Index k = 0; k < nnz; ++k) {
        std::istringstream ls(next_data_line(in));
        Index i, j;
        double v;
        if (!(ls >> i >> j >> v)) throw IoError("matrix market: bad entry");
        if (i < 1 || i > r || j < 1 || j > c) throw IoError("matrix market: index out of range");
        if (!std::isfinite(v)) throw IoError("matrix market: non-finite value");
        es.push_back({j - 1, i - 1, v});
    }
    std::stable_sort(es.begin(), es.end(), [](const E& a, const E& b) { return a.j != b.j ? a.j < b.j : a.i < b.i; });
    for (size_t k = 1; k < es.size(); ++k)
        if (es[k].j == es[k - 1].j && es[k].i == es[k - 1].i) throw IoError("matrix market: duplicate entry");
    colptr->assign(static_cast<size_t>(c + 1), 0);
    rowidx->resize(es.size());
    values->resize(es.size());
    for (size_t k = 0; k < es.size(); ++k) {
        ++(*colptr)[static_cast<size_t>(es[k].j + 1)];
        (*rowidx)[k] = static_cast<std::int32_t>(es[k].i);
        (*values)[k] = es[k].v;
    }
    for (Index j = 0; j < c; ++j) (*colptr)[static_cast<size_t>(j + 1)] += (*colptr)[static_cast<size_t>(j)];
}

}  // namespace blws
