// dropin_vs_ref.cpp -- TEST INFRASTRUCTURE: one program that includes BOTH the
// unmodified reference headers (<adaspmv/kernels.hpp>, <adaspmv/matrix_market.hpp>,
// compiled from /root/reference/proj/include where they lie) and the drop-in
// C++ header (include/adaspmv_cuda.hpp over libadaspmv_cuda.so), loads the
// same Matrix Market file through both `load_matrix`s (matrix_market.hpp:228)
// and runs every KernelId through both `run_kernel`s (kernels.hpp:520-535) on
// the same operands.  It is the check a caller switching from
// `adaspmv::run_kernel` to `adaspmv::cuda::run_kernel` would write.
//
//   dropin_vs_ref <file.mtx> <seed> <density>...
//
// Pass criteria: |y_gpu - y_ref|_i <= rtol * (|A||x|)_i with
// rtol 1e-12 (fp64) / 1e-5 (ADASPMV_REAL32); the sort write-back's sparse
// index sets equal the reference's exactly; dims equal.  Prints one line per
// (density, kernel) and "DROPIN OK" / "DROPIN FAIL"; exit status 0 / 1.
// Built by oracle/Makefile into oracle/_ref/ (the GPU box has no /root/reference).
#include <adaspmv/kernels.hpp>
#include <adaspmv/matrix_market.hpp>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "adaspmv_cuda.hpp"

namespace ref = adaspmv;
namespace gpu = adaspmv::cuda;

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: %s file.mtx seed density...\n", argv[0]);
        return 2;
    }
    const std::string path = argv[1];
    const unsigned seed = static_cast<unsigned>(std::strtoul(argv[2], nullptr, 10));
#ifdef ADASPMV_REAL32
    const double rtol = 1e-5;
#else
    const double rtol = 1e-12;
#endif
    bool ok = true;
    try {
        const ref::DualMatrix A = ref::load_matrix(path);
        gpu::Context ctx(0);
        const gpu::DualMatrix G = gpu::load_matrix(ctx, path);
        if (G.rows() != A.rows() || G.cols() != A.cols() || G.nnz() != A.nnz()) {
            std::printf("dims differ: ref %lld x %lld (%lld) gpu %lld x %lld (%lld)\n", (long long)A.rows(),
                        (long long)A.cols(), (long long)A.nnz(), (long long)G.rows(), (long long)G.cols(),
                        (long long)G.nnz());
            std::printf("DROPIN FAIL\n");
            return 1;
        }
        // |A| for the magnitude-scaled tolerance
        ref::CsrMatrix abs_csr = A.csr;
        for (auto& v : abs_csr.values) v = std::fabs(v);
        const ref::DualMatrix absA = ref::DualMatrix::from_csr(std::move(abs_csr));
        std::mt19937_64 rng(seed);
        for (int di = 3; di < argc; ++di) {
            const double dens = std::strtod(argv[di], nullptr);
            const ref::index_t n = A.cols();
            // support: each column kept with probability dens, values in [-1, 1)
            ref::SparseVector xs;
            xs.length = n;
            std::uniform_real_distribution<double> u01(0.0, 1.0);
            for (ref::index_t j = 0; j < n; ++j)
                if (u01(rng) < dens) {
                    xs.indices.push_back(j);
                    xs.values.push_back(static_cast<ref::real_t>(2.0 * u01(rng) - 1.0));
                }
            const ref::DenseVector xd = ref::sparse_to_dense(xs);
            const ref::BitMask xm = ref::build_bitmask(xs);
            ref::DenseVector xa = xd;
            for (auto& v : xa.values) v = std::fabs(v);
            const ref::DenseVector bound = ref::reference_multiply(absA, xa);
            // the same operands in the drop-in's host value types
            gpu::SparseVector gs;
            gs.length = xs.length;
            gs.indices.assign(xs.indices.begin(), xs.indices.end());
            gs.values.assign(xs.values.begin(), xs.values.end());
            gpu::DenseVector gd(std::vector<gpu::real_t>(xd.values.begin(), xd.values.end()));
            gpu::BitMask gm(xm.length);
            gm.words.assign(xm.words.begin(), xm.words.end());
            ref::OperandViews rv;
            rv.dense = &xd;
            rv.sparse = &xs;
            rv.mask = &xm;
            gpu::OperandViews gv;
            gv.dense = &gd;
            gv.sparse = &gs;
            gv.mask = &gm;
            for (int k = 0; k < ref::KernelId::kCount; ++k) {
                const ref::KernelId rid = ref::KernelId::from_index(k);
                const gpu::KernelId gid = gpu::KernelId::from_index(k);
                const ref::MultiplyOutput ry = ref::run_kernel(A, rid, rv, ref::KernelConfig{});
                const gpu::MultiplyOutput gy = gpu::run_kernel(G, gid, gv, gpu::KernelConfig{});
                const auto& rd = ry.dense();
                const auto& gdv = gy.dense();
                double worst = 0;  // max |diff| / allowed
                bool good = rd.size() == gdv.size();
                for (ref::index_t i = 0; good && i < rd.size(); ++i) {
                    const double diff = std::fabs(static_cast<double>(gdv[i]) - static_cast<double>(rd[i]));
                    const double allowed = rtol * static_cast<double>(bound[i]) + 1e-300;
                    worst = std::max(worst, diff / allowed);
                    if (diff > allowed) good = false;
                }
                bool same_index = true;
                if (rid.writeback == ref::Writeback::Sort) {  // sparse outputs: index sets exact
                    const auto& ri = ry.sparse().indices;
                    const auto& gi = gy.sparse().indices;
                    same_index = ri.size() == gi.size() && std::equal(ri.begin(), ri.end(), gi.begin());
                }
                std::printf("density %-8g nnz_x %-9lld kernel %-20s %s  worst/allowed %.3g%s\n", dens,
                            (long long)xs.nnz(), std::string(rid.name()).c_str(), good && same_index ? "ok" : "MISMATCH",
                            worst, same_index ? "" : "  (sparse index set differs)");
                ok = ok && good && same_index;
            }
        }
    } catch (const std::exception& e) {
        std::printf("exception: %s\nDROPIN FAIL\n", e.what());
        return 1;
    }
    std::printf(ok ? "DROPIN OK\n" : "DROPIN FAIL\n");
    return ok ? 0 : 1;
}
