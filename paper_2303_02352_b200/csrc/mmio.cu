// mmio.cu -- MatrixMarket ingest/distribute and write (host side of the C ABI).
//
// Mirrors read_matrix_market / write_matrix_market (mm_io.cpp:26-110) and
// CsrMatrix::from_triplets (csr.cpp:24-54) plus distribute_matrix
// (dist.cpp:349-363): coordinate real|integer|pattern, general|symmetric|
// skew-symmetric; 1-based entries; symmetric files mirror off-diagonal
// entries (skew negates the mirror and rejects stored diagonals); rows sorted
// by (row, column); duplicates rejected; errors "name:line: msg" as
// parse_error, "cannot open" as io_error.  The parse is one pass over the
// file image (fread + strtoll/strtod, which round like the reference's
// iostream extraction), the CSR build a counting sort by row followed by a
// per-row column sort -- the same unique order as the reference's global
// (row, col) sort, since duplicates are errors.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "common.cuh"
#include "mmio.cuh"

namespace pb {

namespace {

[[noreturn]] void parse_fail(const std::string& name, long line, const std::string& msg) {
    fail(PAIRAMG_PARSE_ERROR, name + ":" + std::to_string(line) + ": " + msg);
}

std::string lower(std::string s) {
    std::transform(s.begin(), s.end(), s.begin(), [](unsigned char c) { return static_cast<char>(std::tolower(c)); });
    return s;
}

// Line cursor over the file image.
struct Lines {
    const char* p;
    const char* end;
    long lineno = 0;
    bool next(const char*& b, const char*& e) {
        if (p >= end) return false;
        b = p;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
        e = nl ? nl : end;
        p = nl ? nl + 1 : end;  // a '\r' stays in the line, as with std::getline
        ++lineno;
        return true;
    }
};

bool blank_or_comment(const char* b, const char* e) { return b == e || *b == '%'; }

// Whitespace-separated integer / real tokens (the reference's `>>`).
bool read_i64(const char*& q, const char* e, int64_t& v) {
    while (q < e && std::isspace(static_cast<unsigned char>(*q))) ++q;
    if (q >= e) return false;
    char buf[64];
    const size_t n = std::min<size_t>(static_cast<size_t>(e - q), sizeof buf - 1);
    std::memcpy(buf, q, n);
    buf[n] = 0;
    char* stop = nullptr;
    errno = 0;
    const long long x = std::strtoll(buf, &stop, 10);
    if (stop == buf || errno) return false;
    q += stop - buf;
    v = x;
    return true;
}

bool read_f64(const char*& q, const char* e, double& v) {
    while (q < e && std::isspace(static_cast<unsigned char>(*q))) ++q;
    if (q >= e) return false;
    char buf[128];
    const size_t n = std::min<size_t>(static_cast<size_t>(e - q), sizeof buf - 1);
    std::memcpy(buf, q, n);
    buf[n] = 0;
    char* stop = nullptr;
    const double x = std::strtod(buf, &stop);
    if (stop == buf) return false;
    q += stop - buf;
    v = x;
    return true;
}

}  // namespace

HostCsr read_matrix_market(const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) fail(PAIRAMG_IO_ERROR, "cannot open " + path);
    std::vector<char> img;
    {
        std::fseek(f, 0, SEEK_END);
        const long sz = std::ftell(f);
        std::fseek(f, 0, SEEK_SET);
        img.resize(sz > 0 ? static_cast<size_t>(sz) : 0);
        const size_t got = sz > 0 ? std::fread(img.data(), 1, img.size(), f) : 0;
        std::fclose(f);
        if (got != img.size()) fail(PAIRAMG_IO_ERROR, "read failure on " + path);
    }
    const std::string& name = path;
    Lines in{img.data(), img.data() + img.size()};
    const char *b, *e;
    if (!in.next(b, e)) parse_fail(name, 1, "empty file");
    std::vector<std::string> tok;
    {
        std::string h(b, e), t;
        size_t i = 0;
        while (tok.size() < 5) {
            while (i < h.size() && std::isspace(static_cast<unsigned char>(h[i]))) ++i;
            size_t j = i;
            while (j < h.size() && !std::isspace(static_cast<unsigned char>(h[j]))) ++j;
            tok.push_back(h.substr(i, j - i));
            i = j;
        }
    }
    if (tok[0] != "%%MatrixMarket") parse_fail(name, in.lineno, "missing %%MatrixMarket banner");
    const std::string object = lower(tok[1]), format = lower(tok[2]), field = lower(tok[3]), symmetry = lower(tok[4]);
    if (object != "matrix") parse_fail(name, in.lineno, "unsupported object '" + object + "'");
    if (format != "coordinate") parse_fail(name, in.lineno, "only coordinate format is supported");
    const bool pattern = field == "pattern";
    if (field != "real" && field != "integer" && !pattern) parse_fail(name, in.lineno, "unsupported field '" + field + "'");
    const bool symmetric = symmetry == "symmetric", skew = symmetry == "skew-symmetric";
    if (!symmetric && !skew && symmetry != "general")
        parse_fail(name, in.lineno, "unsupported symmetry '" + symmetry + "'");

    int64_t nrows = 0, ncols = 0, nstored = 0;
    while (true) {
        if (!in.next(b, e)) parse_fail(name, in.lineno + 1, "missing size line");
        if (blank_or_comment(b, e)) continue;
        const char* q = b;
        if (!read_i64(q, e, nrows) || !read_i64(q, e, ncols) || !read_i64(q, e, nstored))
            parse_fail(name, in.lineno, "malformed size line '" + std::string(b, e) + "'");
        break;
    }
    if (nrows < 0 || ncols < 0 || nstored < 0) parse_fail(name, in.lineno, "negative dimension in size line");

    std::vector<int64_t> ri, ci;
    std::vector<double> vi;
    const size_t cap = static_cast<size_t>(nstored) * ((symmetric || skew) ? 2 : 1);
    ri.reserve(cap);
    ci.reserve(cap);
    vi.reserve(cap);
    int64_t seen = 0;
    while (seen < nstored) {
        if (!in.next(b, e))
            parse_fail(name, in.lineno + 1, "unexpected end of file, expected " + std::to_string(nstored) +
                                                " entries, got " + std::to_string(seen));
        if (blank_or_comment(b, e)) continue;
        const char* q = b;
        int64_t r = 0, c = 0;
        double v = 1.0;
        if (!read_i64(q, e, r) || !read_i64(q, e, c)) parse_fail(name, in.lineno, "malformed entry '" + std::string(b, e) + "'");
        if (!pattern && !read_f64(q, e, v)) parse_fail(name, in.lineno, "missing value in '" + std::string(b, e) + "'");
        if (r < 1 || r > nrows || c < 1 || c > ncols)
            parse_fail(name, in.lineno, "entry (" + std::to_string(r) + ", " + std::to_string(c) + ") out of bounds");
        ri.push_back(r - 1);
        ci.push_back(c - 1);
        vi.push_back(v);
        if ((symmetric || skew) && r != c) {
            ri.push_back(c - 1);
            ci.push_back(r - 1);
            vi.push_back(skew ? -v : v);
        }
        if (skew && r == c) parse_fail(name, in.lineno, "skew-symmetric file stores a diagonal entry");
        ++seen;
    }

    // from_triplets: rows by counting sort, then columns within each row
    HostCsr A;
    A.nrows = nrows;
    A.ncols = ncols;
    const size_t nnz = ri.size();
    A.row_ptr.assign(static_cast<size_t>(nrows) + 1, 0);
    for (int64_t r : ri) ++A.row_ptr[static_cast<size_t>(r) + 1];
    std::partial_sum(A.row_ptr.begin(), A.row_ptr.end(), A.row_ptr.begin());
    std::vector<int64_t> fill(A.row_ptr.begin(), A.row_ptr.end() - 1);
    std::vector<size_t> slot(nnz);
    for (size_t t = 0; t < nnz; ++t) slot[static_cast<size_t>(fill[static_cast<size_t>(ri[t])]++)] = t;
    A.col.resize(nnz);
    A.val.resize(nnz);
    std::vector<std::pair<int64_t, size_t>> rowbuf;
    for (int64_t r = 0; r < nrows; ++r) {
        const int64_t b0 = A.row_ptr[static_cast<size_t>(r)], b1 = A.row_ptr[static_cast<size_t>(r) + 1];
        rowbuf.clear();
        for (int64_t k = b0; k < b1; ++k) rowbuf.push_back({ci[slot[static_cast<size_t>(k)]], slot[static_cast<size_t>(k)]});
        std::sort(rowbuf.begin(), rowbuf.end());
        for (size_t k = 0; k < rowbuf.size(); ++k) {
            if (k > 0 && rowbuf[k].first == rowbuf[k - 1].first)
                fail(PAIRAMG_PARSE_ERROR, name + ": from_triplets: duplicate entry at (" + std::to_string(r) + ", " +
                                              std::to_string(rowbuf[k].first) + ")");
            A.col[static_cast<size_t>(b0) + k] = rowbuf[k].first;
            A.val[static_cast<size_t>(b0) + k] = vi[rowbuf[k].second];
        }
    }
    return A;
}

void write_matrix_market(const std::string& path, int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                         const int64_t* col, const double* val) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) fail(PAIRAMG_IO_ERROR, "cannot open " + path + " for writing");
    const int64_t nnz = nrows > 0 ? row_ptr[nrows] : 0;
    bool ok = std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n",
                           static_cast<long long>(nrows), static_cast<long long>(ncols),
                           static_cast<long long>(nnz)) > 0;
    for (int64_t i = 0; ok && i < nrows; ++i)
        for (int64_t k = row_ptr[i]; ok && k < row_ptr[i + 1]; ++k)
            ok = std::fprintf(f, "%lld %lld %.17g\n", static_cast<long long>(i + 1),
                              static_cast<long long>(col[k] + 1), val[k]) > 0;
    ok = std::fclose(f) == 0 && ok;
    if (!ok) fail(PAIRAMG_IO_ERROR, "write failure");
}

}  // namespace pb
