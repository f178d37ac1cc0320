// selector.cpp -- features and the cascaded decision-tree
// selector hook.
//
// Matrix features (ids 0..8) are computed once on the device at matrix
// creation (matrix.cu).  Vector features (ids 9..12) are lazy: nnz_x of a
// sparse input is known on the host for free; nnz_s / m_sparsity (and nnz_x
// of a dense input) take one device reduction and a scalar D2H -- the only
// per-iteration device round trip of the selection.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>

#include "internal.hpp"

namespace ada {

// FNV-1a of the frozen feature order, written into model files.
std::string feature_order_hash() {
    const char* order =
        "m,n,nnz,max_row,min_row,avg_row,relative_range,var_nnz_row,gc,nnz_x,x_sparsity,nnz_s,"
        "m_sparsity";
    uint64_t h = 1469598103934665603ull;
    for (const char* p = order; *p; ++p) {
        h ^= static_cast<unsigned char>(*p);
        h *= 1099511628211ull;
    }
    char buf[32];
    std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(h));
    return buf;
}

void features(Context& ctx, const Matrix& m, Vector& v, uint32_t mask, double* out) {
    for (int i = 0; i < 9; ++i)
        if (mask & (1u << i)) out[i] = m.feat[i];
    if (mask & ((1u << 9) | (1u << 10))) {
        // a dense-only x gets nnz_x and nnz_s from one pass (vector_nnz_s)
        if (v.nnz < 0 && v.has_dense && !v.has_sparse && v.n == m.cols) vector_nnz_s(ctx, v, m);
        const double nx = static_cast<double>(vector_nnz(ctx, v));
        if (mask & (1u << 9)) out[9] = nx;
        if (mask & (1u << 10)) out[10] = v.n > 0 ? nx / static_cast<double>(v.n) : 0.0;
    }
    if (mask & ((1u << 11) | (1u << 12))) {
        const double ns = static_cast<double>(vector_nnz_s(ctx, v, m));
        if (mask & (1u << 11)) out[11] = ns;
        if (mask & (1u << 12)) out[12] = m.nnz > 0 ? ns / static_cast<double>(m.nnz) : 0.0;
    }
}

namespace {

// Walks one tree (routing "value <= threshold -> left"),
// pulling features lazily into `f` / `have`.
int walk(Context& ctx, const Matrix& m, Vector& v, const Tree& t, double* f, uint32_t& have,
         uint32_t& consulted, double* feature_s) {
    int32_t i = 0;
    for (int guard = 0; guard < 1 << 20; ++guard) {
        const int32_t feat = t.feature[static_cast<size_t>(i)];
        if (feat < 0) return t.leaf[static_cast<size_t>(i)];
        if (!(have & (1u << feat)) && (feat == 11 || feat == 12) && v.nnz >= 0 && v.n == m.cols &&
            !(v.nnz_s >= 0 && v.nnz_s_matrix == m.id)) {
            // nnz_s of k = nnz_x distinct columns lies between the sums of the
            // k smallest and the k largest column degrees: when the whole
            // interval is on one side of the split, route without the device
            // reduction (the walk is the one the exact value would take)
            double lo = static_cast<double>(m.nnz_s_lower(v.nnz));
            double hi = static_cast<double>(m.nnz_s_upper(v.nnz));
            if (feat == 12) {
                const double nz = m.nnz > 0 ? static_cast<double>(m.nnz) : 1.0;
                lo = m.nnz > 0 ? lo / nz : 0.0;
                hi = m.nnz > 0 ? hi / nz : 0.0;
            }
            const double thr = t.threshold[static_cast<size_t>(i)];
            if (hi <= thr || lo > thr) consulted |= 1u << feat;
            if (hi <= thr) {
                i = t.left[static_cast<size_t>(i)];
                continue;
            }
            if (lo > thr) {
                i = t.right[static_cast<size_t>(i)];
                continue;
            }
        }
        if (!(have & (1u << feat))) {
            const auto t0 = std::chrono::steady_clock::now();
            features(ctx, m, v, 1u << feat, f);
            if (feature_s)
                *feature_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            have |= 1u << feat;
        }
        i = f[feat] <= t.threshold[static_cast<size_t>(i)] ? t.left[static_cast<size_t>(i)]
                                                          : t.right[static_cast<size_t>(i)];
    }
    throw Error(ADASPMV_ERR_INTERNAL, "decision tree walk did not terminate");
}

}  // namespace

// predict_kernel: pattern -> workload -> write-back iff
// ColSpMSpV.  Classes: pattern {0 ColSpMSpV, 1 RowSpMSpV, 2 SpMV}
// (kernels.hpp:34), workload {0 Direct, 1 LoadBalanced}, write-back
// {0 Atomic, 1 Sort}; returns KernelId::index() (kernels.hpp:52-60).
int predict(Context& ctx, const Matrix& m, Vector& v, const Bundle& b, uint32_t* used, int* trees,
            double* feature_s) {
    double f[ADASPMV_NUM_FEATURES] = {0};
    uint32_t have = 0, consulted = 0;  // computed / routed on their bounds
    int nt = 0;
    const int pattern = walk(ctx, m, v, b.trees[0], f, have, consulted, feature_s);
    ++nt;
    // schema 2: the column family reads its own workload tree
    const Tree& wt = pattern == 0 && b.has_col ? b.trees[3] : b.trees[1];
    const int lb = walk(ctx, m, v, wt, f, have, consulted, feature_s) == 1 ? 1 : 0;
    ++nt;
    int k;
    switch (pattern) {
        case 2: k = lb; break;      // SpMV
        case 1: k = 2 + lb; break;  // RowSpMSpV
        case 0: {
            const int sort = walk(ctx, m, v, b.trees[2], f, have, consulted, feature_s) == 1 ? 1 : 0;
            ++nt;
            k = 4 + 2 * lb + sort;
            break;
        }
        default: throw Error(ADASPMV_ERR_FORMAT, "pattern tree produced an invalid class");
    }
    if (used) *used = have | consulted;
    if (trees) *trees = nt;
    return k;
}

namespace {

[[noreturn]] void bad(const std::string& why) { throw Error(ADASPMV_ERR_FORMAT, "model file: " + why); }

void check_tree(const Tree& t, int nclasses) {
    const size_t n = t.feature.size();
    if (n == 0) bad("empty tree");
    for (size_t i = 0; i < n; ++i) {
        const int32_t f = t.feature[i];
        if (f < 0) {
            if (t.leaf[i] < 0 || t.leaf[i] >= nclasses) bad("leaf class out of range");
            continue;
        }
        if (f >= ADASPMV_NUM_FEATURES) bad("feature id out of range");
        if (!(t.mask & (1u << f))) bad("node reads a feature outside the tree's mask");
        // children after the parent: acyclic, single root at 0
        if (t.left[i] <= static_cast<int32_t>(i) || t.right[i] <= static_cast<int32_t>(i) ||
            t.left[i] >= static_cast<int32_t>(n) || t.right[i] >= static_cast<int32_t>(n))
            bad("child index out of order or range");
    }
}

}  // namespace

void validate_bundle(const Bundle& b) {
    check_tree(b.trees[0], 3);
    check_tree(b.trees[1], 2);
    check_tree(b.trees[2], 2);
    if (b.has_col) check_tree(b.trees[3], 2);
}

// Text form of the SPEC.md:383 model file:
//   adaspmv-bundle <schema_version>
//   hardware_tag <tag>
//   feature_order_hash <hex>
//   tree <pattern|workload|writeback> mask <u32> nodes <N>
//   <feature> <threshold> <left> <right> <leaf>      (N lines; leaf: feature -1)
//   ... (three trees) ...
//   end
// Schema 2 (an extension, not in SPEC.md): a fourth tree `workload_col`, the
// LB-vs-Direct decision of the ColSpMSpV family (the row patterns keep
// `workload`); both workload trees may read every feature.
Bundle* bundle_load(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw Error(ADASPMV_ERR_FORMAT, "cannot open file: " + path);
    auto* b = new Bundle();
    try {
        std::string tag;
        if (!(in >> tag >> b->schema_version) || tag != "adaspmv-bundle") bad("missing header");
        if (b->schema_version != 1 && b->schema_version != 2)
            bad("unsupported schema_version " + std::to_string(b->schema_version));
        const int ntrees = b->schema_version == 2 ? 4 : 3;
        b->has_col = ntrees == 4;
        std::string key;
        if (!(in >> key >> b->hardware_tag) || key != "hardware_tag") bad("missing hardware_tag");
        if (!(in >> key >> b->feature_order_hash) || key != "feature_order_hash")
            bad("missing feature_order_hash");
        if (b->feature_order_hash != feature_order_hash()) bad("feature order hash mismatch");
        bool seen[4] = {false, false, false, false};
        for (int k = 0; k < ntrees; ++k) {
            std::string tw, target, mw, nw;
            uint32_t mask = 0;
            long long n = 0;
            if (!(in >> tw >> target >> mw >> mask >> nw >> n) || tw != "tree" || mw != "mask" ||
                nw != "nodes" || n <= 0 || n > (1 << 22))
                bad("truncated or malformed tree header");
            int idx = target == "pattern"                     ? 0
                      : target == "workload"                  ? 1
                      : target == "writeback"                 ? 2
                      : target == "workload_col" && ntrees == 4 ? 3
                                                              : -1;
            if (idx < 0 || seen[idx]) bad("unknown or repeated tree target '" + target + "'");
            seen[idx] = true;
            Tree& t = b->trees[idx];
            t.target = idx;
            t.mask = mask;
            t.feature.resize(static_cast<size_t>(n));
            t.threshold.resize(static_cast<size_t>(n));
            t.left.resize(static_cast<size_t>(n));
            t.right.resize(static_cast<size_t>(n));
            t.leaf.resize(static_cast<size_t>(n));
            for (long long i = 0; i < n; ++i) {
                std::string th;
                if (!(in >> t.feature[i] >> th >> t.left[i] >> t.right[i] >> t.leaf[i]))
                    bad("truncated node list");
                t.threshold[i] = std::strtod(th.c_str(), nullptr);  // %.17g round trip
            }
        }
        std::string end;
        if (!(in >> end) || end != "end") bad("missing end marker");
        validate_bundle(*b);
        return b;
    } catch (...) {
        delete b;
        throw;
    }
}

}  // namespace ada
