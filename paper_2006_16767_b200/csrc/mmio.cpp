// mmio.cpp -- host-side matrix load/convert with the reference's semantics:
//   load_matrix_market  matrix_market.hpp:38-127 (real/integer/pattern,
//                       general/symmetric; 1-based -> 0-based; duplicates summed)
//   write_matrix_market matrix_market.hpp:132-146 (canonical, %.17g)
//   save/load_binary    matrix_market.hpp:148-225 (ASPMVBIN v1, little-endian)
//   load_matrix         matrix_market.hpp:228-238 (sniffs the binary magic)
//   from_triplets       sparse.hpp:220-258 (bucket by row, sort by column,
//                       sum duplicates; values narrowed to the dtype first)
// Errors: ParseError(line) -> ADASPMV_ERR_PARSE with "(line N)" appended as in
// types.hpp:23-25; FormatError -> ADASPMV_ERR_FORMAT; structure violations
// -> ADASPMV_ERR_INVALID_ARGUMENT (CsrMatrix::validate, sparse.hpp:44-63).
#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "internal.hpp"

namespace ada {

namespace {

[[noreturn]] void parse_error(const std::string& what, long line) {
    throw Error(ADASPMV_ERR_PARSE, line > 0 ? what + " (line " + std::to_string(line) + ")" : what);
}
[[noreturn]] void format_error(const std::string& what) { throw Error(ADASPMV_ERR_FORMAT, what); }

std::string lower(std::string s) {
    for (auto& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

bool blank(const std::string& s) {
    return std::all_of(s.begin(), s.end(), [](unsigned char c) { return std::isspace(c); });
}

constexpr char kMagic[8] = {'A', 'S', 'P', 'M', 'V', 'B', 'I', 'N'};
constexpr uint32_t kVersion = 1;

void validate_csr(const HostCsr& m) {
    const auto& ro = m.row_offsets;
    const auto& ci = m.col_indices;
    if (ro.size() != static_cast<size_t>(m.rows) + 1) invalid("csr: row_offsets length != rows+1");
    if (ro.front() != 0) invalid("csr: row_offsets[0] != 0");
    for (int64_t r = 0; r < m.rows; ++r) {
        if (ro[r + 1] < ro[r]) invalid("csr: row_offsets not nondecreasing");
        for (int64_t k = ro[r]; k < ro[r + 1]; ++k) {
            if (ci[k] < 0 || ci[k] >= m.cols) invalid("csr: column index out of range");
            if (k > ro[r] && ci[k] <= ci[k - 1])
                invalid("csr: columns not strictly increasing in row " + std::to_string(r));
        }
    }
    if (ci.size() != static_cast<size_t>(ro.back()) || m.values.size() != static_cast<size_t>(ro.back()))
        invalid("csr: array lengths inconsistent with nnz");
}

}  // namespace

namespace {

// Serial parser: the reference's line-by-line semantics and error messages
// (matrix_market.hpp:38-127).  Used for the header, and for the data
// section whenever the parallel pass below finds anything irregular, so
// every error is reported exactly as the reference reports it.
HostTriplets load_mm_serial(const std::string& path) {
    std::ifstream in(path);
    if (!in) format_error("cannot open file: " + path);
    std::string line;
    long lineno = 0;
    if (!std::getline(in, line)) parse_error("empty file", 1);
    ++lineno;
    std::istringstream banner(lower(line));
    std::string tag, object, format, field, symmetry;
    banner >> tag >> object >> format >> field >> symmetry;
    if (tag != "%%matrixmarket" || object != "matrix") parse_error("malformed Matrix Market banner", lineno);
    if (format != "coordinate")
        parse_error("only coordinate format is supported, got '" + format + "'", lineno);
    if (field != "real" && field != "integer" && field != "pattern")
        parse_error("unsupported field '" + field + "'", lineno);
    if (symmetry != "general" && symmetry != "symmetric")
        parse_error("unsupported symmetry '" + symmetry + "'", lineno);
    const bool pattern = field == "pattern";
    const bool symmetric = symmetry == "symmetric";
    int64_t rows = 0, cols = 0;
    long long declared = -1;
    for (;;) {
        if (!std::getline(in, line)) parse_error("missing size line", lineno);
        ++lineno;
        if (!line.empty() && line[0] == '%') continue;
        if (blank(line)) continue;
        std::istringstream ss(line);
        long long r = 0, c = 0, e = 0;
        if (!(ss >> r >> c >> e) || r < 0 || c < 0 || e < 0) parse_error("malformed size line", lineno);
        std::string rest;
        if (ss >> rest) parse_error("trailing tokens on size line", lineno);
        rows = r;
        cols = c;
        declared = e;
        break;
    }
    if (rows == 0 || cols == 0)
        parse_error("degenerate matrix dimensions (" + std::to_string(rows) + " x " +
                        std::to_string(cols) + ")",
                    lineno);
    std::vector<int64_t> tr, tc;
    std::vector<double> tv;
    const size_t reserve = static_cast<size_t>(symmetric ? 2 * declared : declared);
    tr.reserve(reserve);
    tc.reserve(reserve);
    tv.reserve(reserve);
    long long seen = 0;
    while (std::getline(in, line)) {
        ++lineno;
        if (line.empty() || line[0] == '%' || blank(line)) continue;
        const char* p = line.c_str();
        char* end = nullptr;
        long long r = std::strtoll(p, &end, 10);
        if (end == p) parse_error("expected row coordinate", lineno);
        p = end;
        long long c = std::strtoll(p, &end, 10);
        if (end == p) parse_error("expected column coordinate", lineno);
        p = end;
        double v = 1.0;
        if (!pattern) {
            v = std::strtod(p, &end);
            if (end == p) parse_error("expected value", lineno);
            p = end;
        }
        while (*p != '\0' && std::isspace(static_cast<unsigned char>(*p))) ++p;
        if (*p != '\0') parse_error("trailing tokens on entry line", lineno);
        if (r < 1 || r > rows) parse_error("row coordinate " + std::to_string(r) + " out of range", lineno);
        if (c < 1 || c > cols)
            parse_error("column coordinate " + std::to_string(c) + " out of range", lineno);
        ++seen;
        if (seen > declared) parse_error("more entries than declared in size line", lineno);
        tr.push_back(r - 1);
        tc.push_back(c - 1);
        tv.push_back(v);
        if (symmetric && r != c) {
            tr.push_back(c - 1);
            tc.push_back(r - 1);
            tv.push_back(v);
        }
    }
    if (seen != declared)
        parse_error("entry count " + std::to_string(seen) + " does not match declared " +
                        std::to_string(declared),
                    lineno);
    HostTriplets t;
    t.rows = rows;
    t.cols = cols;
    t.r = std::move(tr);
    t.c = std::move(tc);
    t.v = std::move(tv);
    return t;
}

HostCsr load_bin(const std::string& path, int dtype) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) format_error("cannot open file: " + path);
    auto rd = [&](void* p, size_t bytes) {
        if (std::fread(p, 1, bytes, f) != bytes) {
            std::fclose(f);
            format_error("truncated binary matrix file: " + path);
        }
    };
    char magic[8];
    rd(magic, 8);
    if (std::memcmp(magic, kMagic, 8) != 0) {
        std::fclose(f);
        format_error("not a binary matrix file: " + path);
    }
    uint32_t version = 0, width = 0;
    rd(&version, 4);
    rd(&width, 4);
    if (version != kVersion) {
        std::fclose(f);
        format_error("unsupported binary matrix version " + std::to_string(version));
    }
    if (width != static_cast<uint32_t>(value_bytes(dtype))) {
        std::fclose(f);
        format_error("binary matrix value width " + std::to_string(width) + " does not match this build");
    }
    uint64_t dims[3];
    rd(dims, sizeof dims);
    HostCsr m;
    m.rows = static_cast<int64_t>(dims[0]);
    m.cols = static_cast<int64_t>(dims[1]);
    m.row_offsets.resize(static_cast<size_t>(dims[0]) + 1);
    m.col_indices.resize(static_cast<size_t>(dims[2]));
    m.values.resize(static_cast<size_t>(dims[2]));
    rd(m.row_offsets.data(), m.row_offsets.size() * sizeof(int64_t));
    rd(m.col_indices.data(), m.col_indices.size() * sizeof(int64_t));
    if (dtype == ADASPMV_F64) {
        rd(m.values.data(), m.values.size() * sizeof(double));
    } else {
        std::vector<float> tmp(m.values.size());
        rd(tmp.data(), tmp.size() * sizeof(float));
        std::copy(tmp.begin(), tmp.end(), m.values.begin());
    }
    std::fclose(f);
    validate_csr(m);
    return m;
}

}  // namespace

namespace {

// Parallel parser of the coordinate section (ingestion at scale, SURVEY.md
// 8(f)3): the file is read once, the entry lines are split into one chunk
// per host thread at line boundaries and parsed concurrently with the serial
// parser's conversions (strtoll / strtod), and the chunks are concatenated in
// file order, so the triplet sequence is the serial one.  Anything the fast
// path does not accept verbatim (a malformed or out-of-range entry, a count
// mismatch, an unusual header, an embedded NUL) returns false and the caller
// re-parses serially, which raises the reference's error with its line.
struct Chunk {
    std::vector<int64_t> r, c;
    std::vector<double> v;
    long long seen = 0;
    bool ok = true;
};

void parse_chunk(const char* b, const char* e, bool pattern, bool symmetric, int64_t rows, int64_t cols,
                 Chunk& out) {
    out.r.reserve(static_cast<size_t>((e - b) / 12 + 16));
    out.c.reserve(out.r.capacity());
    out.v.reserve(out.r.capacity());
    const char* p = b;
    while (p < e) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(e - p)));
        const char* le = nl ? nl : e;
        const char* q = p;
        while (q < le && std::isspace(static_cast<unsigned char>(*q))) ++q;
        if (q == le || *p == '%') {  // blank or comment line
            p = le + 1;
            continue;
        }
        char* end = nullptr;
        const long long r = std::strtoll(p, &end, 10);
        if (end == p || end > le) { out.ok = false; return; }
        const char* t = end;
        const long long c = std::strtoll(t, &end, 10);
        if (end == t || end > le) { out.ok = false; return; }
        t = end;
        double v = 1.0;
        if (!pattern) {
            v = std::strtod(t, &end);
            if (end == t || end > le) { out.ok = false; return; }
            t = end;
        }
        while (t < le && std::isspace(static_cast<unsigned char>(*t))) ++t;
        if (t != le || r < 1 || r > rows || c < 1 || c > cols) { out.ok = false; return; }
        ++out.seen;
        out.r.push_back(r - 1);
        out.c.push_back(c - 1);
        out.v.push_back(v);
        if (symmetric && r != c) {
            out.r.push_back(c - 1);
            out.c.push_back(r - 1);
            out.v.push_back(v);
        }
        p = le + 1;
    }
}

bool load_mm_parallel(const std::string& path, HostTriplets& t) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) return false;
    std::string buf;
    if (std::fseek(f, 0, SEEK_END) == 0) {
        const long size = std::ftell(f);
        if (size > 0) {
            buf.resize(static_cast<size_t>(size));
            std::rewind(f);
            if (std::fread(&buf[0], 1, buf.size(), f) != buf.size()) buf.clear();
        }
    }
    std::fclose(f);
    if (buf.size() < (size_t(1) << 20)) return false;  // small files: the serial parser is as fast
    if (std::memchr(buf.data(), '\0', buf.size())) return false;
    // header: banner, comments / blank lines, size line (as load_mm_serial)
    size_t pos = 0;
    auto next_line = [&](std::string& line) {
        if (pos >= buf.size()) return false;
        const size_t nl = buf.find('\n', pos);
        const size_t e = nl == std::string::npos ? buf.size() : nl;
        line.assign(buf, pos, e - pos);
        pos = e + 1;
        return true;
    };
    std::string line;
    if (!next_line(line)) return false;
    std::istringstream banner(lower(line));
    std::string tag, object, format, field, symmetry;
    banner >> tag >> object >> format >> field >> symmetry;
    if (tag != "%%matrixmarket" || object != "matrix" || format != "coordinate") return false;
    if (field != "real" && field != "integer" && field != "pattern") return false;
    if (symmetry != "general" && symmetry != "symmetric") return false;
    const bool pattern = field == "pattern", symmetric = symmetry == "symmetric";
    long long rows = 0, cols = 0, declared = -1;
    for (;;) {
        if (!next_line(line)) return false;
        if ((!line.empty() && line[0] == '%') || blank(line)) continue;
        std::istringstream ss(line);
        if (!(ss >> rows >> cols >> declared) || rows <= 0 || cols <= 0 || declared < 0) return false;
        std::string rest;
        if (ss >> rest) return false;
        break;
    }
    const size_t data = std::min(pos, buf.size());
    const unsigned hw = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    const size_t len = buf.size() - data;
    const unsigned nt = static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>(hw, len / (256 << 10))));
    std::vector<size_t> cut(nt + 1, buf.size());
    cut[0] = data;
    for (unsigned i = 1; i < nt; ++i) {  // chunk starts right after a newline
        const size_t want = data + len * i / nt;
        const size_t nl = buf.find('\n', std::max(want, cut[i - 1]));
        cut[i] = nl == std::string::npos ? buf.size() : nl + 1;
    }
    std::vector<Chunk> chunks(nt);
    {
        std::vector<std::thread> th;
        for (unsigned i = 0; i < nt; ++i)
            th.emplace_back(parse_chunk, buf.data() + cut[i], buf.data() + cut[i + 1], pattern, symmetric,
                            static_cast<int64_t>(rows), static_cast<int64_t>(cols), std::ref(chunks[i]));
        for (auto& x : th) x.join();
    }
    long long seen = 0;
    size_t total = 0;
    std::vector<size_t> at(nt + 1, 0);
    for (unsigned i = 0; i < nt; ++i) {
        if (!chunks[i].ok) return false;
        seen += chunks[i].seen;
        at[i + 1] = at[i] + chunks[i].r.size();
    }
    total = at[nt];
    if (seen != declared) return false;
    t.rows = rows;
    t.cols = cols;
    t.r.resize(total);
    t.c.resize(total);
    t.v.resize(total);
    {
        std::vector<std::thread> th;
        for (unsigned i = 0; i < nt; ++i)
            th.emplace_back([&, i] {
                std::copy(chunks[i].r.begin(), chunks[i].r.end(), t.r.begin() + static_cast<std::ptrdiff_t>(at[i]));
                std::copy(chunks[i].c.begin(), chunks[i].c.end(), t.c.begin() + static_cast<std::ptrdiff_t>(at[i]));
                std::copy(chunks[i].v.begin(), chunks[i].v.end(), t.v.begin() + static_cast<std::ptrdiff_t>(at[i]));
                Chunk().r.swap(chunks[i].r);
            });
        for (auto& x : th) x.join();
    }
    return true;
}

}  // namespace

HostTriplets load_mm(const std::string& path) {
    HostTriplets t;
    if (load_mm_parallel(path, t)) return t;
    return load_mm_serial(path);
}

HostMatrixFile load_matrix_file(const std::string& path, int dtype) {
    HostMatrixFile out;
    {
        std::ifstream probe(path, std::ios::binary);
        if (!probe) format_error("cannot open file: " + path);
        char magic[8] = {};
        probe.read(magic, 8);
        if (probe.gcount() == 8 && std::memcmp(magic, kMagic, 8) == 0) {
            out.is_csr = true;
            out.csr = load_bin(path, dtype);
            return out;
        }
    }
    out.trip = load_mm(path);
    return out;
}

void write_matrix_market_file(const std::string& path, int64_t rows, int64_t cols,
                              const std::vector<int64_t>& ro, const std::vector<int64_t>& ci,
                              const std::vector<double>& vals) {
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) format_error("cannot open file for writing: " + path);
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n");
    std::fprintf(f, "%lld %lld %lld\n", static_cast<long long>(rows), static_cast<long long>(cols),
                 static_cast<long long>(ro.empty() ? 0 : ro.back()));
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t k = ro[r]; k < ro[r + 1]; ++k)
            std::fprintf(f, "%lld %lld %.17g\n", static_cast<long long>(r + 1),
                         static_cast<long long>(ci[k] + 1), vals[k]);
    std::fclose(f);
}

void save_binary_file(const std::string& path, int64_t rows, int64_t cols,
                      const std::vector<int64_t>& ro, const std::vector<int64_t>& ci,
                      const void* vals, int dtype) {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) format_error("cannot open file for writing: " + path);
    auto wr = [&](const void* p, size_t bytes) {
        if (std::fwrite(p, 1, bytes, f) != bytes) {
            std::fclose(f);
            format_error("short write to " + path);
        }
    };
    wr(kMagic, 8);
    const uint32_t version = kVersion, width = static_cast<uint32_t>(value_bytes(dtype));
    wr(&version, 4);
    wr(&width, 4);
    const uint64_t dims[3] = {static_cast<uint64_t>(rows), static_cast<uint64_t>(cols),
                              static_cast<uint64_t>(ro.empty() ? 0 : ro.back())};
    wr(dims, sizeof dims);
    wr(ro.data(), ro.size() * sizeof(int64_t));
    wr(ci.data(), ci.size() * sizeof(int64_t));
    wr(vals, ci.size() * static_cast<size_t>(width));
    std::fclose(f);
}

}  // namespace ada
