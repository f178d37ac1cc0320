"""ctypes front end of the CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this module.  The
product (``paper_2006_16767_b200``) never does; it fails loudly when its CUDA
library is missing instead of falling back here.

Two checkers are exposed:

* :class:`Port` -- ``oracle/liboracle.so``, the plain-C restatement
  (``adaspmv_oracle.c``), each function citing the reference file:line.
* :class:`Ref`  -- ``oracle/_ref/libadaspmv_ref_{f64,f32}.so``, the unmodified
  reference headers compiled by ``oracle/Makefile`` behind ``ref_capi.cpp``.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_dp = C.POINTER(C.c_double)


def _as(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _nullable(dt):
    """ndpointer that also accepts None."""
    base = np.ctypeslib.ndpointer(dtype=dt, flags="C_CONTIGUOUS")

    class _N(base):  # type: ignore[misc, valid-type]
        @classmethod
        def from_param(cls, obj):
            if obj is None:
                return None
            return base.from_param(obj)

    return _N


class OracleMissing(RuntimeError):
    pass


# --------------------------------------------------------------------------
# The plain-C port
# --------------------------------------------------------------------------
class Port:
    """oracle/liboracle.so (plain-C restatement)."""

    def __init__(self, path: Path | None = None):
        path = path or HERE / "liboracle.so"
        if not path.exists():
            raise OracleMissing(f"{path} not built (run `make -C oracle`)")
        L = self.lib = C.CDLL(str(path))
        L.or_segment_of.restype = C.c_int64
        L.or_segment_of.argtypes = [_i64p, C.c_int64, C.c_int64]
        L.or_make_partition.restype = C.c_int
        L.or_make_partition.argtypes = [_i64p, C.c_int64, C.c_int64, C.c_int, _i64p]
        L.or_build_bitmask_sparse.argtypes = [C.c_int64, C.c_int64, _i64p, _u64p]
        L.or_effective_nnz.restype = C.c_int64
        L.or_effective_nnz.argtypes = [_i64p, C.c_int64, _i64p]
        L.or_csr_validate.restype = C.c_int
        L.or_csr_validate.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p]
        L.or_gini_coefficient.restype = C.c_double
        L.or_gini_coefficient.argtypes = [C.c_int64, _i64p]
        L.or_gini_pairwise.restype = C.c_double
        L.or_gini_pairwise.argtypes = [C.c_int64, _i64p]
        L.or_matrix_features.restype = C.c_int
        L.or_matrix_features.argtypes = [C.c_int64, C.c_int64, _i64p, _f64p]
        L.or_tree_predict.restype = C.c_int
        L.or_tree_predict.argtypes = [_i32p, _f64p, _i32p, _i32p, _i32p, _f64p]
        L.or_bfs_queue.restype = C.c_int64
        L.or_bfs_queue.argtypes = [C.c_int64, _i64p, _i64p, C.c_int64, _i64p]
        L.or_bfs_queue_i32.restype = C.c_int64
        L.or_bfs_queue_i32.argtypes = [C.c_int64, _i64p, _i32p, C.c_int64, _i64p]
        L.or_pagerank_incremental.restype = C.c_int64
        L.or_pagerank_incremental.argtypes = [C.c_int64, _i64p, _i64p, C.c_double, C.c_double, C.c_int64,
                                              _f64p]
        L.or_vector_features_sparse.argtypes = [C.c_int64, C.c_int64, _i64p, C.c_int64, _i64p, _f64p]
        for sfx, rp in (("_f64", _f64p), ("_f32", _f32p)):
            nr = _nullable(np.float64 if sfx == "_f64" else np.float32)
            f = getattr(L, "or_reference_multiply" + sfx)
            f.argtypes = [C.c_int64, _i64p, _i64p, rp, rp, rp]
            f = getattr(L, "or_semiring_multiply" + sfx)
            f.argtypes = [C.c_int64, _i64p, _i64p, rp, rp, C.c_int, rp]
            f = getattr(L, "or_row_major_multiply" + sfx)
            f.argtypes = [C.c_int64, _i64p, _i64p, rp, rp, _nullable(np.uint64), C.c_int, C.c_int, rp]
            f = getattr(L, "or_spmspv_col" + sfx)
            f.restype = C.c_int64
            f.argtypes = [C.c_int64, _i64p, _i64p, rp, C.c_int64, _i64p, rp, C.c_int, C.c_int,
                          C.c_int, C.c_int, nr, _nullable(np.int64), nr]
            f = getattr(L, "or_sort_reduce_pairs" + sfx)
            f.restype = C.c_int64
            f.argtypes = [C.c_int64, _i64p, rp, _i64p, rp]
            f = getattr(L, "or_csr_to_csc" + sfx)
            f.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, rp, _i64p, _i64p, rp]
            f = getattr(L, "or_dense_to_sparse" + sfx)
            f.restype = C.c_int64
            f.argtypes = [C.c_int64, rp, _i64p, rp]
            f = getattr(L, "or_sparse_to_dense" + sfx)
            f.restype = C.c_int
            f.argtypes = [C.c_int64, C.c_int64, _i64p, rp, rp]
            f = getattr(L, "or_build_bitmask_dense" + sfx)
            f.argtypes = [C.c_int64, rp, _u64p]
            f = getattr(L, "or_vector_features_dense" + sfx)
            f.argtypes = [C.c_int64, C.c_int64, _i64p, rp, _f64p]

    @staticmethod
    def _sfx(dt):
        return "_f64" if np.dtype(dt) == np.float64 else "_f32"

    # --- partition / index helpers --------------------------------------
    def segment_of(self, offsets, pos):
        o = _as(offsets, np.int64)
        return int(self.lib.or_segment_of(o, len(o), int(pos)))

    def make_partition(self, offsets, total, workers):
        o = _as(offsets, np.int64)
        out = np.zeros(4 * max(workers, 1), np.int64)
        rc = self.lib.or_make_partition(o, len(o), int(total), int(workers), out)
        if rc != 0:
            raise ValueError("make_partition: invalid arguments")
        return out.reshape(-1, 4)

    def build_bitmask_sparse(self, n, idx):
        idx = _as(idx, np.int64)
        w = np.zeros((n + 63) // 64, np.uint64)
        self.lib.or_build_bitmask_sparse(n, len(idx), idx, w)
        return w

    def build_bitmask_dense(self, x):
        x = np.ascontiguousarray(x)
        w = np.zeros((len(x) + 63) // 64, np.uint64)
        getattr(self.lib, "or_build_bitmask_dense" + self._sfx(x.dtype))(len(x), x, w)
        return w

    def effective_nnz(self, col_offsets, idx):
        idx = _as(idx, np.int64)
        return int(self.lib.or_effective_nnz(_as(col_offsets, np.int64), len(idx), idx))

    def csr_validate(self, rows, cols, ro, ci):
        return int(self.lib.or_csr_validate(rows, cols, _as(ro, np.int64), _as(ci, np.int64)))

    # --- features / selector / BFS (SPEC-only) -----------------------------
    def gini(self, degrees):
        d = _as(degrees, np.int64)
        return float(self.lib.or_gini_coefficient(len(d), d))

    def gini_pairwise(self, degrees):
        d = _as(degrees, np.int64)
        return float(self.lib.or_gini_pairwise(len(d), d))

    def matrix_features(self, rows, cols, ro):
        out = np.zeros(9, np.float64)
        if self.lib.or_matrix_features(rows, cols, _as(ro, np.int64), out) != 0:
            raise ValueError("matrix features: zero rows")
        return out

    def vector_features_sparse(self, n, col_offsets, idx):
        co = _as(col_offsets, np.int64)
        idx = _as(idx, np.int64)
        out = np.zeros(4, np.float64)
        self.lib.or_vector_features_sparse(n, int(co[-1]), co, len(idx), idx, out)
        return out

    def vector_features_dense(self, col_offsets, x):
        co = _as(col_offsets, np.int64)
        x = np.ascontiguousarray(x)
        out = np.zeros(4, np.float64)
        getattr(self.lib, "or_vector_features_dense" + self._sfx(x.dtype))(len(x), int(co[-1]), co, x, out)
        return out

    def tree_predict(self, feature, threshold, left, right, leaf, f13):
        return int(self.lib.or_tree_predict(_as(feature, np.int32), _as(threshold, np.float64),
                                            _as(left, np.int32), _as(right, np.int32),
                                            _as(leaf, np.int32), _as(f13, np.float64)))

    def bfs_queue_i32(self, n, col_offsets, row_indices, source):
        lv = np.zeros(n, np.int64)
        nl = self.lib.or_bfs_queue_i32(n, _as(col_offsets, np.int64), _as(row_indices, np.int32), int(source), lv)
        return lv, int(nl)

    def bfs_queue(self, n, col_offsets, row_indices, source):
        lv = np.zeros(n, np.int64)
        nl = self.lib.or_bfs_queue(n, _as(col_offsets, np.int64), _as(row_indices, np.int64), int(source), lv)
        return lv, int(nl)

    def pagerank_incremental(self, n, col_offsets, row_indices, damping=0.85, prune=1e-6, max_iters=300):
        """SPEC.md:498-506; pass A's CSR (row_offsets, col_indices): out-edges per source."""
        rank = np.zeros(n, np.float64)
        it = self.lib.or_pagerank_incremental(n, _as(col_offsets, np.int64), _as(row_indices, np.int64),
                                              float(damping), float(prune), int(max_iters), rank)
        return rank, int(it)

    # --- value-typed kernels ---------------------------------------------
    def reference_multiply(self, rows, ro, ci, vals, x):
        vals = np.ascontiguousarray(vals)
        dt = vals.dtype
        y = np.zeros(rows, dt)
        getattr(self.lib, "or_reference_multiply" + self._sfx(dt))(
            rows, _as(ro, np.int64), _as(ci, np.int64), vals, _as(x, dt), y)
        return y

    def semiring_multiply(self, rows, ro, ci, vals, x, sr):
        """y = A x under semiring sr (0 plus-times, 1 or-and, 2 min-plus); dense x,
        absent entries 0 (or-and) / +inf (min-plus)."""
        vals = np.ascontiguousarray(vals)
        dt = vals.dtype
        y = np.zeros(rows, dt)
        getattr(self.lib, "or_semiring_multiply" + self._sfx(dt))(
            rows, _as(ro, np.int64), _as(ci, np.int64), vals, _as(x, dt), int(sr), y)
        return y

    def row_major_multiply(self, rows, ro, ci, vals, x, mask=None, load_balanced=False, workers=1):
        vals = np.ascontiguousarray(vals)
        dt = vals.dtype
        y = np.zeros(rows, dt)
        getattr(self.lib, "or_row_major_multiply" + self._sfx(dt))(
            rows, _as(ro, np.int64), _as(ci, np.int64), vals, _as(x, dt),
            None if mask is None else _as(mask, np.uint64), int(load_balanced), int(workers), y)
        return y

    def spmspv_col(self, rows, co, ri, vals, xi, xv, load_balanced=False, sort=False, workers=1,
                   private_acc=False):
        """Returns dense y (atomic) or (idx, val) sparse y (sort)."""
        vals = np.ascontiguousarray(vals)
        dt = vals.dtype
        xi = _as(xi, np.int64)
        xv = _as(xv, dt)
        f = getattr(self.lib, "or_spmspv_col" + self._sfx(dt))
        if not sort:
            y = np.zeros(rows, dt)
            f(rows, _as(co, np.int64), _as(ri, np.int64), vals, len(xi), xi, xv, int(load_balanced),
              0, int(workers), int(private_acc), y, None, None)
            return y
        yi = np.zeros(max(rows, 1), np.int64)
        yv = np.zeros(max(rows, 1), dt)
        k = f(rows, _as(co, np.int64), _as(ri, np.int64), vals, len(xi), xi, xv, int(load_balanced),
              1, int(workers), 0, None, yi, yv)
        return yi[:k].copy(), yv[:k].copy()

    def sort_reduce_pairs(self, rows_in, vals_in):
        vals_in = np.ascontiguousarray(vals_in)
        dt = vals_in.dtype
        n = len(vals_in)
        oi = np.zeros(max(n, 1), np.int64)
        ov = np.zeros(max(n, 1), dt)
        k = getattr(self.lib, "or_sort_reduce_pairs" + self._sfx(dt))(n, _as(rows_in, np.int64), vals_in, oi, ov)
        return oi[:k].copy(), ov[:k].copy()

    def csr_to_csc(self, rows, cols, ro, ci, vals):
        vals = np.ascontiguousarray(vals)
        dt = vals.dtype
        nnz = int(ro[rows])
        co = np.zeros(cols + 1, np.int64)
        ri = np.zeros(max(nnz, 1), np.int64)
        cv = np.zeros(max(nnz, 1), dt)
        getattr(self.lib, "or_csr_to_csc" + self._sfx(dt))(rows, cols, _as(ro, np.int64), _as(ci, np.int64),
                                                          vals, co, ri, cv)
        return co, ri[:nnz].copy(), cv[:nnz].copy()

    def dense_to_sparse(self, v):
        v = np.ascontiguousarray(v)
        idx = np.zeros(max(len(v), 1), np.int64)
        val = np.zeros(max(len(v), 1), v.dtype)
        k = getattr(self.lib, "or_dense_to_sparse" + self._sfx(v.dtype))(len(v), v, idx, val)
        return idx[:k].copy(), val[:k].copy()

    def sparse_to_dense(self, n, idx, val):
        val = np.ascontiguousarray(val)
        out = np.zeros(n, val.dtype)
        rc = getattr(self.lib, "or_sparse_to_dense" + self._sfx(val.dtype))(n, len(val), _as(idx, np.int64), val, out)
        if rc != 0:
            raise IndexError("sparse vector index out of bounds")
        return out

    # --- the reference kernels, restated: all 8 by KernelId::index() ------
    def run_kernel(self, kernel_index, rows, cols, ro, ci, vals, csc, x_dense=None, x_sparse=None,
                   workers=1, private_acc=False):
        """Mirror of run_kernel (kernels.hpp:520-535) over host arrays.

        ``csc`` = (col_offsets, row_indices, values).  Returns ("dense", y) or
        ("sparse", (idx, val)) in the representation the reference kernel
        produces (sort write-back -> sparse, kernels.hpp:113-115).
        """
        vals = np.ascontiguousarray(vals)
        dt = vals.dtype
        if x_dense is None:
            xi, xv = x_sparse
            x_dense = self.sparse_to_dense(cols, xi, _as(xv, dt))
        if x_sparse is None:
            x_sparse = self.dense_to_sparse(_as(x_dense, dt))
        k = int(kernel_index)
        if k in (0, 1):
            return "dense", self.row_major_multiply(rows, ro, ci, vals, x_dense, None, k == 1, workers)
        if k in (2, 3):
            mask = self.build_bitmask_sparse(cols, x_sparse[0])
            return "dense", self.row_major_multiply(rows, ro, ci, vals, x_dense, mask, k == 3, workers)
        co, ri, cv = csc
        lb = k in (6, 7)
        sort = k in (5, 7)
        r = self.spmspv_col(rows, co, ri, cv, x_sparse[0], x_sparse[1], lb, sort, workers, private_acc)
        return ("sparse", r) if sort else ("dense", r)


# --------------------------------------------------------------------------
# The reference itself (compiled headers behind ref_capi.cpp)
# --------------------------------------------------------------------------
class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def host_isa() -> str:
    """x86-64 ISA level of this host for the timed reference build: v4 when the
    CPU has AVX-512 (avx512f/bw/dq/vl), else v3."""
    try:
        flags = Path("/proc/cpuinfo").read_text().split("flags", 2)[1].split("\n", 1)[0].split()
    except Exception:
        return "v3"
    return "v4" if all(f in flags for f in ("avx512f", "avx512bw", "avx512dq", "avx512vl")) else "v3"


def host_cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class Ref:
    """oracle/_ref/libadaspmv_ref_{f64,f32}[_cnt].so (checker build: -ffp-contract=off)
    or, bench=True, libadaspmv_ref_bench_{f64,f32}_{v3,v4}.so: the reference's
    own ref_bench flags (-O3, contraction allowed) at this host's ISA level."""

    def __init__(self, dtype=np.float64, counters=False, path: Path | None = None, bench: bool = False):
        self.dtype = np.dtype(dtype)
        sfx = "f64" if self.dtype == np.float64 else "f32"
        name = f"libadaspmv_ref_{'cnt_' if counters else ''}{sfx}.so"
        if bench:
            name = f"libadaspmv_ref_bench_{sfx}_{host_isa()}.so"
        self.variant = name
        path = path or HERE / "_ref" / name
        if not path.exists():
            raise OracleMissing(f"{path} not built (run `make -C oracle ref` where the reference is mounted)")
        L = self.lib = C.CDLL(str(path))
        rp = _f64p if self.dtype == np.float64 else _f32p
        nr = _nullable(self.dtype)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_real_bytes.restype = C.c_int
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_threads.restype = C.c_int
        L.ref_matrix_create.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, nr, C.POINTER(vp)]
        L.ref_matrix_destroy.argtypes = [vp]
        L.ref_matrix_dims.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.ref_matrix_export.argtypes = [vp, _nullable(np.int64), _nullable(np.int64), nr,
                                        _nullable(np.int64), _nullable(np.int64), nr]
        L.ref_matrix_transpose.argtypes = [vp, C.POINTER(vp)]
        L.ref_run_kernel.argtypes = [vp, C.c_int, nr, C.c_int64, _nullable(np.int64), nr, C.c_int, C.c_int,
                                     nr, _nullable(np.int64), nr, C.POINTER(C.c_int64), _nullable(np.uint64)]
        L.ref_bench_kernel.argtypes = [vp, C.c_int, nr, C.c_int64, _nullable(np.int64), nr, C.c_int, C.c_int, _f64p]
        L.ref_reference_multiply.argtypes = [vp, rp, rp]
        L.ref_effective_nnz.argtypes = [vp, C.c_int64, _i64p, C.POINTER(C.c_int64)]
        L.ref_dense_to_sparse.argtypes = [C.c_int64, rp, _i64p, rp, C.POINTER(C.c_int64)]
        L.ref_sparse_to_dense.argtypes = [C.c_int64, C.c_int64, _i64p, rp, rp]
        L.ref_build_bitmask_sparse.argtypes = [C.c_int64, C.c_int64, _i64p, _u64p]
        L.ref_build_bitmask_dense.argtypes = [C.c_int64, rp, _u64p]
        L.ref_make_partition.argtypes = [_i64p, C.c_int64, C.c_int64, C.c_int, _i64p]
        L.ref_segment_of.restype = C.c_int64
        L.ref_segment_of.argtypes = [_i64p, C.c_int64, C.c_int64]
        L.ref_sort_reduce_pairs.argtypes = [C.c_int64, _i64p, rp, C.c_int64, _i64p, rp, C.POINTER(C.c_int64)]
        L.ref_load_matrix.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.ref_write_matrix_market.argtypes = [vp, C.c_char_p]
        L.ref_save_binary.argtypes = [vp, C.c_char_p]
        L.ref_from_triplets.argtypes = [C.c_int64, C.c_int64, C.c_int64, _i64p, _i64p, rp, C.POINTER(vp)]
        L.ref_bfs.argtypes = [vp, C.c_int64, C.c_int, _i64p, C.POINTER(C.c_int64), C.POINTER(C.c_double)]

    def _check(self, rc):
        if rc != 0:
            raise RefError(rc, self.lib.ref_last_error().decode())

    def set_threads(self, n):
        self.lib.ref_set_threads(int(n))

    def threads(self):
        return int(self.lib.ref_threads())

    # matrix handles ------------------------------------------------------
    def matrix(self, rows, cols, ro, ci, vals=None):
        h = C.c_void_p()
        self._check(self.lib.ref_matrix_create(rows, cols, _as(ro, np.int64), _as(ci, np.int64),
                                               None if vals is None else _as(vals, self.dtype), C.byref(h)))
        return RefMatrix(self, h)

    def from_triplets(self, rows, cols, tr, tc, tv):
        h = C.c_void_p()
        tr = _as(tr, np.int64)
        self._check(self.lib.ref_from_triplets(rows, cols, len(tr), tr, _as(tc, np.int64),
                                               _as(tv, self.dtype), C.byref(h)))
        return RefMatrix(self, h)

    def load_matrix(self, path):
        h = C.c_void_p()
        self._check(self.lib.ref_load_matrix(str(path).encode(), C.byref(h)))
        return RefMatrix(self, h)

    # free functions --------------------------------------------------------
    def dense_to_sparse(self, v):
        v = _as(v, self.dtype)
        idx = np.zeros(max(len(v), 1), np.int64)
        val = np.zeros(max(len(v), 1), self.dtype)
        k = C.c_int64()
        self._check(self.lib.ref_dense_to_sparse(len(v), v, idx, val, C.byref(k)))
        return idx[:k.value].copy(), val[:k.value].copy()

    def sparse_to_dense(self, n, idx, val):
        out = np.zeros(n, self.dtype)
        idx = _as(idx, np.int64)
        self._check(self.lib.ref_sparse_to_dense(n, len(idx), idx, _as(val, self.dtype), out))
        return out

    def build_bitmask_sparse(self, n, idx):
        idx = _as(idx, np.int64)
        w = np.zeros((n + 63) // 64, np.uint64)
        self._check(self.lib.ref_build_bitmask_sparse(n, len(idx), idx, w))
        return w

    def build_bitmask_dense(self, v):
        v = _as(v, self.dtype)
        w = np.zeros((len(v) + 63) // 64, np.uint64)
        self._check(self.lib.ref_build_bitmask_dense(len(v), v, w))
        return w

    def make_partition(self, offsets, total, workers):
        o = _as(offsets, np.int64)
        out = np.zeros(4 * max(workers, 1), np.int64)
        self._check(self.lib.ref_make_partition(o, len(o), int(total), int(workers), out))
        return out.reshape(-1, 4)

    def segment_of(self, offsets, pos):
        o = _as(offsets, np.int64)
        return int(self.lib.ref_segment_of(o, len(o), int(pos)))

    def sort_reduce_pairs(self, rows_in, vals_in, nrows):
        rows_in = _as(rows_in, np.int64)
        n = len(rows_in)
        oi = np.zeros(max(n, 1), np.int64)
        ov = np.zeros(max(n, 1), self.dtype)
        k = C.c_int64()
        self._check(self.lib.ref_sort_reduce_pairs(n, rows_in, _as(vals_in, self.dtype), nrows, oi, ov, C.byref(k)))
        return oi[:k.value].copy(), ov[:k.value].copy()


class RefMatrix:
    def __init__(self, ref: Ref, handle):
        self.ref = ref
        self.h = handle
        r, c, z = C.c_int64(), C.c_int64(), C.c_int64()
        ref.lib.ref_matrix_dims(handle, C.byref(r), C.byref(c), C.byref(z))
        self.rows, self.cols, self.nnz = r.value, c.value, z.value

    def __del__(self):
        try:
            if self.h:
                self.ref.lib.ref_matrix_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def export(self):
        """-> (row_offsets, col_indices, values, col_offsets, row_indices, csc_values)."""
        dt = self.ref.dtype
        ro = np.zeros(self.rows + 1, np.int64)
        ci = np.zeros(max(self.nnz, 1), np.int64)
        cv = np.zeros(max(self.nnz, 1), dt)
        co = np.zeros(self.cols + 1, np.int64)
        ri = np.zeros(max(self.nnz, 1), np.int64)
        rv = np.zeros(max(self.nnz, 1), dt)
        self.ref.lib.ref_matrix_export(self.h, ro, ci, cv, co, ri, rv)
        z = self.nnz
        return ro, ci[:z].copy(), cv[:z].copy(), co, ri[:z].copy(), rv[:z].copy()

    def transpose(self):
        h = C.c_void_p()
        self.ref._check(self.ref.lib.ref_matrix_transpose(self.h, C.byref(h)))
        return RefMatrix(self.ref, h)

    def run_kernel(self, kernel_index, x_dense=None, x_sparse=None, workers=0, private_acc=False):
        """-> (dense y, (sparse idx, val), counters[3])."""
        dt = self.ref.dtype
        yd = np.zeros(self.rows, dt)
        yi = np.zeros(max(self.rows, 1), np.int64)
        yv = np.zeros(max(self.rows, 1), dt)
        k = C.c_int64()
        cnt = np.zeros(3, np.uint64)
        if x_dense is not None:
            args = (_as(x_dense, dt), 0, None, None)
        else:
            xi, xv = x_sparse
            xi = _as(xi, np.int64)
            args = (None, len(xi), xi, _as(xv, dt))
        self.ref._check(self.ref.lib.ref_run_kernel(self.h, int(kernel_index), *args, int(workers),
                                                    int(private_acc), yd, yi, yv, C.byref(k), cnt))
        return yd, (yi[:k.value].copy(), yv[:k.value].copy()), cnt

    def bfs(self, source=0, kernel=-1):
        """SPEC.md:489-497 plus-times BFS with the reference's run_kernel
        (ref_capi.cpp ref_bfs) -> (levels int64[n], n_levels, wall seconds)."""
        n = self.rows
        lv = np.empty(n, np.int64)
        nl, sec = C.c_int64(), C.c_double()
        self.ref._check(self.ref.lib.ref_bfs(self.h, int(source), int(kernel), lv, C.byref(nl), C.byref(sec)))
        return lv, int(nl.value), float(sec.value)

    def bench_kernel(self, kernel_index, x_dense=None, x_sparse=None, warmup=1, repeats=10):
        dt = self.ref.dtype
        times = np.zeros(repeats, np.float64)
        if x_dense is not None:
            args = (_as(x_dense, dt), 0, None, None)
        else:
            xi, xv = x_sparse
            xi = _as(xi, np.int64)
            args = (None, len(xi), xi, _as(xv, dt))
        self.ref._check(self.ref.lib.ref_bench_kernel(self.h, int(kernel_index), *args, int(warmup),
                                                      int(repeats), times))
        return times

    def reference_multiply(self, x):
        y = np.zeros(self.rows, self.ref.dtype)
        self.ref._check(self.ref.lib.ref_reference_multiply(self.h, _as(x, self.ref.dtype), y))
        return y

    def effective_nnz(self, idx):
        idx = _as(idx, np.int64)
        k = C.c_int64()
        self.ref._check(self.ref.lib.ref_effective_nnz(self.h, len(idx), idx, C.byref(k)))
        return k.value

    def write_matrix_market(self, path):
        self.ref._check(self.ref.lib.ref_write_matrix_market(self.h, str(path).encode()))

    def save_binary(self, path):
        self.ref._check(self.ref.lib.ref_save_binary(self.h, str(path).encode()))


def have_ref(dtype=np.float64) -> bool:
    sfx = "f64" if np.dtype(dtype) == np.float64 else "f32"
    return (HERE / "_ref" / f"libadaspmv_ref_{sfx}.so").exists()


def build(quiet=True) -> None:
    """Builds liboracle.so and, where the reference is mounted, _ref/ (make)."""
    import subprocess
    subprocess.run(["make", "-C", str(HERE), "all"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


if os.environ.get("ADASPMV_ORACLE_AUTOBUILD") == "1":  # pragma: no cover
    build()
