// Matrix Market ingest / export (host side of the operator layer).
//
// read_matrix_market / write_matrix_market are specified in SPEC.md:442-450 (coordinate or
// array, real, general; other field/symmetry flags -> unsupported-format error; a write-read
// round trip reproduces every entry to full double precision). The coordinate body becomes a
// CSR exactly as SparseCsrMatrix::from_triplets builds it (sparse_csr.cpp:42-64): entries
// ordered by (row, col), duplicate coordinates and out-of-range coordinates are FormatError,
// then the from_parts invariants (sparse_csr.cpp:10-40: finite values, columns < 2^31).
//
// The file is read in one block and its body split at line boundaries over hardware threads,
// each parsing with std::from_chars; triplets are bucketed by row with a counting pass and each
// row's columns sorted, so the host work is O(nnz) apart from short per-row sorts. The device
// upload (and the transposed CSR) reuse make_csr / make_dense.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "mtx.cuh"

namespace qbgpu {

namespace {

struct Header {
    bool coordinate = true;
    std::int64_t m = 0, n = 0, nnz = 0;
    std::size_t body = 0;  // offset of the first entry line
};

std::string lower(std::string s) {
    for (auto& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

std::vector<char> slurp(const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw QbError(kError, "matrix market: cannot open " + path);
    std::fseek(f, 0, SEEK_END);
    const long sz = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    std::vector<char> buf(static_cast<std::size_t>(std::max(sz, 0L)) + 1, '\0');
    const std::size_t got = sz > 0 ? std::fread(buf.data(), 1, static_cast<std::size_t>(sz), f) : 0;
    std::fclose(f);
    if (static_cast<long>(got) != sz) throw QbError(kError, "matrix market: short read of " + path);
    buf[got] = '\n';
    return buf;
}

Header parse_header(const std::vector<char>& buf) {
    Header h;
    std::size_t pos = 0;
    auto next_line = [&](std::string& line) {
        if (pos >= buf.size()) return false;
        std::size_t e = pos;
        while (e < buf.size() && buf[e] != '\n') ++e;
        line.assign(buf.data() + pos, buf.data() + e);
        if (!line.empty() && line.back() == '\r') line.pop_back();
        pos = e + 1;
        return true;
    };
    std::string line;
    if (!next_line(line)) throw QbError(kFormatError, "matrix market: empty file");
    char w[5][64] = {};
    if (std::sscanf(line.c_str(), "%63s %63s %63s %63s %63s", w[0], w[1], w[2], w[3], w[4]) != 5 ||
        lower(w[0]) != "%%matrixmarket" || lower(w[1]) != "matrix")
        throw QbError(kFormatError, "matrix market: malformed banner");
    const std::string fmt = lower(w[2]), field = lower(w[3]), sym = lower(w[4]);
    if (fmt == "coordinate") h.coordinate = true;
    else if (fmt == "array") h.coordinate = false;
    else throw QbError(kFormatError, "matrix market: unsupported format '" + fmt + "'");
    if (field != "real" && field != "integer" && field != "double")
        throw QbError(kFormatError, "matrix market: unsupported field '" + field + "' (real, general only)");
    if (sym != "general")
        throw QbError(kFormatError, "matrix market: unsupported symmetry '" + sym + "' (real, general only)");
    while (next_line(line)) {
        std::size_t i = 0;
        while (i < line.size() && std::isspace(static_cast<unsigned char>(line[i]))) ++i;
        if (i == line.size() || line[i] == '%') continue;
        long long a = 0, b = 0, c = 0;
        const int k = std::sscanf(line.c_str(), "%lld %lld %lld", &a, &b, &c);
        if ((h.coordinate && k != 3) || (!h.coordinate && k < 2) || a < 0 || b < 0 || c < 0)
            throw QbError(kFormatError, "matrix market: malformed size line");
        h.m = a;
        h.n = b;
        h.nnz = h.coordinate ? c : a * b;
        h.body = pos;
        return h;
    }
    throw QbError(kFormatError, "matrix market: missing size line");
}

// Split [begin, end) into ~equal pieces at line starts.
std::vector<std::size_t> split_lines(const std::vector<char>& buf, std::size_t begin, std::size_t end, int parts) {
    std::vector<std::size_t> cut{begin};
    for (int p = 1; p < parts; ++p) {
        std::size_t c = begin + (end - begin) * p / parts;
        while (c < end && buf[c - 1] != '\n') ++c;
        cut.push_back(std::max(c, cut.back()));
    }
    cut.push_back(end);
    return cut;
}

const char* skip_ws(const char* p, const char* e) {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
    return p;
}

int n_threads() {
    const unsigned hc = std::thread::hardware_concurrency();
    return static_cast<int>(std::max(1u, std::min(hc, 64u)));
}

// Parse `want` numbers per non-comment line from [b, e) into out (flat); returns the line count.
template <typename Emit>
void parse_range(const char* b, const char* e, int want, Emit&& emit, std::string& err) {
    double tok[3];
    const char* p = b;
    while (p < e) {
        const char* q = skip_ws(p, e);
        if (q < e && *q == '\n') { p = q + 1; continue; }
        if (q < e && *q == '%') {
            while (q < e && *q != '\n') ++q;
            p = q + 1;
            continue;
        }
        for (int t = 0; t < want; ++t) {
            q = skip_ws(q, e);
            if (q < e && *q == '+') ++q;
            auto r = std::from_chars(q, e, tok[t]);
            if (r.ec != std::errc()) {
                err = "matrix market: malformed entry line";
                return;
            }
            q = r.ptr;
        }
        while (q < e && *q != '\n') ++q;  // ignore trailing tokens (comments)
        p = q + 1;
        emit(tok);
    }
}

}  // namespace

MtxInfo mtx_info(const std::string& path) {
    const auto buf = slurp(path);
    const Header h = parse_header(buf);
    return MtxInfo{h.coordinate, h.m, h.n, h.nnz};
}

void mtx_read_csr(const std::string& path, MtxInfo& info, std::vector<std::int64_t>& rp,
                  std::vector<std::int32_t>& ci, std::vector<double>& v) {
    const auto buf = slurp(path);
    const Header h = parse_header(buf);
    if (!h.coordinate) throw QbError(kFormatError, "matrix market: array file where coordinate expected");
    info = MtxInfo{true, h.m, h.n, h.nnz};
    if (h.n > (std::int64_t{1} << 31) - 1) throw QbError(kFormatError, "csr: column count exceeds int32 index range");
    const int T = n_threads();
    const auto cut = split_lines(buf, h.body, buf.size(), T);
    std::vector<std::vector<std::int64_t>> rows(T), cols(T);
    std::vector<std::vector<double>> vals(T);
    std::vector<std::string> errs(T);
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
            parse_range(buf.data() + cut[t], buf.data() + cut[t + 1], 3, [&](const double* x) {
                // 1-based coordinates; non-integral or out-of-range ones become FormatError below
                const double r = x[0] - 1.0, c = x[1] - 1.0;
                rows[t].push_back(r == std::floor(r) && r >= 0 && r < 9.2e18 ? static_cast<std::int64_t>(r) : -1);
                cols[t].push_back(c == std::floor(c) && c >= 0 && c < 9.2e18 ? static_cast<std::int64_t>(c) : -1);
                vals[t].push_back(x[2]);
            }, errs[t]);
        });
    for (auto& x : th) x.join();
    for (auto& e : errs)
        if (!e.empty()) throw QbError(kFormatError, e);
    std::int64_t total = 0;
    for (int t = 0; t < T; ++t) total += static_cast<std::int64_t>(vals[t].size());
    if (total != h.nnz)
        throw QbError(kFormatError, "matrix market: " + std::to_string(total) + " entries, header says " +
                                        std::to_string(h.nnz));
    // counting pass by row (from_triplets order: row, then column)
    rp.assign(static_cast<std::size_t>(h.m) + 1, 0);
    for (int t = 0; t < T; ++t)
        for (std::size_t i = 0; i < rows[t].size(); ++i) {
            const std::int64_t r = rows[t][i], c = cols[t][i];
            if (r < 0 || r >= h.m || c < 0 || c >= h.n) throw QbError(kFormatError, "csr: triplet coordinate out of range");
            ++rp[static_cast<std::size_t>(r) + 1];
        }
    for (std::int64_t i = 0; i < h.m; ++i) rp[i + 1] += rp[i];
    std::vector<std::pair<std::int32_t, double>> ent(static_cast<std::size_t>(total));
    std::vector<std::int64_t> fill(rp.begin(), rp.end() - 1);
    for (int t = 0; t < T; ++t)
        for (std::size_t i = 0; i < rows[t].size(); ++i)
            ent[static_cast<std::size_t>(fill[rows[t][i]]++)] = {static_cast<std::int32_t>(cols[t][i]), vals[t][i]};
    ci.resize(static_cast<std::size_t>(total));
    v.resize(static_cast<std::size_t>(total));
    std::vector<std::thread> th2;
    std::vector<std::string> err2(T);
    for (int t = 0; t < T; ++t)
        th2.emplace_back([&, t] {
            const std::int64_t r0 = h.m * t / T, r1 = h.m * (t + 1) / T;
            for (std::int64_t r = r0; r < r1; ++r) {
                auto* b = ent.data() + rp[r];
                auto* e = ent.data() + rp[r + 1];
                std::stable_sort(b, e, [](const auto& x, const auto& y) { return x.first < y.first; });
                for (auto* p = b; p < e; ++p) {
                    if (p > b && p[-1].first == p->first) { err2[t] = "csr: duplicate coordinate"; return; }
                    if (!std::isfinite(p->second)) { err2[t] = "csr: non-finite value"; return; }
                    ci[p - ent.data()] = p->first;
                    v[p - ent.data()] = p->second;
                }
            }
        });
    for (auto& x : th2) x.join();
    for (auto& e : err2)
        if (!e.empty()) throw QbError(e == "csr: non-finite value" ? kError : kFormatError, e);
}

void mtx_read_dense(const std::string& path, MtxInfo& info, std::vector<double>& a) {
    const auto buf = slurp(path);
    const Header h = parse_header(buf);
    if (h.coordinate) throw QbError(kFormatError, "matrix market: coordinate file where array expected");
    info = MtxInfo{false, h.m, h.n, h.nnz};
    std::vector<double> vals;
    vals.reserve(static_cast<std::size_t>(h.m * h.n));
    std::string err;
    parse_range(buf.data() + h.body, buf.data() + buf.size(), 1, [&](const double* x) { vals.push_back(x[0]); }, err);
    if (!err.empty()) throw QbError(kFormatError, err);
    if (static_cast<std::int64_t>(vals.size()) != h.m * h.n)
        throw QbError(kFormatError, "matrix market: array entry count does not match the size line");
    for (double x : vals)
        if (!std::isfinite(x)) throw QbError(kError, "dense: non-finite value");  // dense_matrix.cpp:17-18
    a = std::move(vals);  // array format is column-major, the DenseMatrix layout
}

namespace {
void put_double(std::string& out, double x) {
    char tmp[40];
    const auto r = std::to_chars(tmp, tmp + sizeof(tmp), x);  // shortest round-trip representation
    out.append(tmp, r.ptr);
}
void write_all(const std::string& path, const std::string& s) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw QbError(kError, "matrix market: cannot create " + path);
    const std::size_t put = std::fwrite(s.data(), 1, s.size(), f);
    std::fclose(f);
    if (put != s.size()) throw QbError(kError, "matrix market: short write to " + path);
}
}  // namespace

void mtx_write_csr(const std::string& path, std::int64_t m, std::int64_t n, std::int64_t nnz, const std::int64_t* rp,
                   const std::int32_t* ci, const double* v) {
    std::string s = "%%MatrixMarket matrix coordinate real general\n";
    s += std::to_string(m) + " " + std::to_string(n) + " " + std::to_string(nnz) + "\n";
    s.reserve(s.size() + static_cast<std::size_t>(nnz) * 40);
    for (std::int64_t i = 0; i < m; ++i)
        for (std::int64_t t = rp[i]; t < rp[i + 1]; ++t) {
            s += std::to_string(i + 1);
            s += ' ';
            s += std::to_string(static_cast<std::int64_t>(ci[t]) + 1);
            s += ' ';
            put_double(s, v[t]);
            s += '\n';
        }
    write_all(path, s);
}

void mtx_write_dense(const std::string& path, std::int64_t m, std::int64_t n, const double* a, std::int64_t lda) {
    std::string s = "%%MatrixMarket matrix array real general\n";
    s += std::to_string(m) + " " + std::to_string(n) + "\n";
    s.reserve(s.size() + static_cast<std::size_t>(m * n) * 24);
    for (std::int64_t j = 0; j < n; ++j)
        for (std::int64_t i = 0; i < m; ++i) {
            put_double(s, a[i + j * lda]);
            s += '\n';
        }
    write_all(path, s);
}

}  // namespace qbgpu
