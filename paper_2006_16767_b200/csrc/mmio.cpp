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

HostCsr csr_from_triplets(int64_t rows, int64_t cols, int64_t count, const int64_t* tr,
                          const int64_t* tc, const double* tv, bool round_f32) {
    if (rows < 0 || cols < 0) invalid("negative matrix dimension");
    HostCsr m;
    m.rows = rows;
    m.cols = cols;
    std::vector<int64_t> off(static_cast<size_t>(rows) + 1, 0);
    for (int64_t i = 0; i < count; ++i) {
        if (tr[i] < 0 || tr[i] >= rows || tc[i] < 0 || tc[i] >= cols)
            invalid("triplet coordinate out of range");
        off[static_cast<size_t>(tr[i]) + 1]++;
    }
    for (int64_t r = 0; r < rows; ++r) off[r + 1] += off[r];
    std::vector<std::pair<int64_t, double>> slots(static_cast<size_t>(count));
    {
        std::vector<int64_t> cur(off.begin(), off.end() - 1);
        for (int64_t i = 0; i < count; ++i) {
            double v = round_f32 ? static_cast<double>(static_cast<float>(tv[i])) : tv[i];
            slots[static_cast<size_t>(cur[static_cast<size_t>(tr[i])]++)] = {tc[i], v};
        }
    }
    m.row_offsets.assign(static_cast<size_t>(rows) + 1, 0);
    m.col_indices.reserve(slots.size());
    m.values.reserve(slots.size());
    for (int64_t r = 0; r < rows; ++r) {
        auto first = slots.begin() + off[r];
        auto last = slots.begin() + off[r + 1];
        std::stable_sort(first, last, [](const auto& a, const auto& b) { return a.first < b.first; });
        for (auto it = first; it != last;) {
            const int64_t col = it->first;
            if (round_f32) {
                float sum = 0;
                for (; it != last && it->first == col; ++it) sum += static_cast<float>(it->second);
                m.values.push_back(sum);
            } else {
                double sum = 0;
                for (; it != last && it->first == col; ++it) sum += it->second;
                m.values.push_back(sum);
            }
            m.col_indices.push_back(col);
        }
        m.row_offsets[static_cast<size_t>(r) + 1] = static_cast<int64_t>(m.col_indices.size());
    }
    return m;
}

namespace {

HostCsr load_mm(const std::string& path, int dtype) {
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
    return csr_from_triplets(rows, cols, static_cast<int64_t>(tr.size()), tr.data(), tc.data(),
                             tv.data(), dtype == ADASPMV_F32);
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

HostCsr load_matrix_file(const std::string& path, int dtype) {
    {
        std::ifstream probe(path, std::ios::binary);
        if (!probe) format_error("cannot open file: " + path);
        char magic[8] = {};
        probe.read(magic, 8);
        if (probe.gcount() == 8 && std::memcmp(magic, kMagic, 8) == 0) return load_bin(path, dtype);
    }
    return load_mm(path, dtype);
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
