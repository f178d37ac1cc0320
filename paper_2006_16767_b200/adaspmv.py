"""Python mirror of the reference's ``namespace adaspmv`` API over the CUDA C-ABI.

The reference (arXiv 2006.16767, ``proj/include/adaspmv/*.hpp``) is a C++
header library; its hot path is ``run_kernel(DualMatrix, KernelId,
OperandViews, KernelConfig) -> MultiplyOutput`` (kernels.hpp:520-535).  This
module keeps those names, argument meanings and error behaviour, and calls
``libadaspmv_cuda.so`` (include/adaspmv_cuda.h) through ctypes:

====================  ===============================================
reference             here
====================  ===============================================
Pattern/Workload/...  :class:`Pattern`, :class:`Workload`, :class:`Writeback`
KernelId              :class:`KernelId` (index/from_index/name/parse)
CsrMatrix/DualMatrix  :class:`DualMatrix` (device resident CSR + CSC)
DenseVector           :class:`DenseVector` (host numpy values)
SparseVector          :class:`SparseVector` (host indices + values)
KernelConfig          :class:`KernelConfig`
OperandViews          :class:`OperandViews`
MultiplyOutput        :class:`MultiplyOutput` (lazy dense()/sparse())
run_kernel/spmv/...   :func:`run_kernel`, :func:`spmv`, :func:`spmspv_row`,
                      :func:`spmspv_col`
std::invalid_argument :class:`InvalidArgument` (a ``ValueError``)
std::out_of_range     :class:`OutOfRange` (an ``IndexError``)
ParseError/FormatError :class:`ParseError` / :class:`FormatError`
====================  ===============================================

There is no CPU fallback: importing works without a GPU, but every call that
needs the library raises :class:`LibraryMissing` if ``libadaspmv_cuda.so`` is
absent, and CUDA errors surface as :class:`CudaError`.
"""
from __future__ import annotations

import ctypes as C
import threading
import enum
import os
import re
from dataclasses import dataclass
from pathlib import Path
from typing import Optional

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libadaspmv_cuda.so"

F64, F32 = 0, 1
PLUS_TIMES, OR_AND, MIN_PLUS = 0, 1, 2
# adaspmv_iteration_report::exec_mode: how BFS ran the selected kernel
EXEC_AS_SELECTED, EXEC_MASKED_PULL, EXEC_FUSED_PUSH_LB = 0, 1, 2
FEATURE_NAMES = ("m", "n", "nnz", "max_row", "min_row", "avg_row", "relative_range",
                 "var_nnz_row", "gc", "nnz_x", "x_sparsity", "nnz_s", "m_sparsity")


# --------------------------------------------------------------------------
# errors (types.hpp:21-36 + std exceptions used by the reference)
# --------------------------------------------------------------------------
class AdaspmvError(RuntimeError):
    code = 7


class InvalidArgument(AdaspmvError, ValueError):
    code = 1


class OutOfRange(AdaspmvError, IndexError):
    code = 2


class ParseError(AdaspmvError):
    code = 3

    @property
    def line(self) -> int:
        m = re.search(r"\(line (\d+)\)$", str(self))
        return int(m.group(1)) if m else 0


class FormatError(AdaspmvError):
    code = 4


class CudaError(AdaspmvError):
    code = 5


class OutOfMemory(AdaspmvError, MemoryError):
    code = 6


class LibraryMissing(RuntimeError):
    pass


_ERRORS = {1: InvalidArgument, 2: OutOfRange, 3: ParseError, 4: FormatError, 5: CudaError,
           6: OutOfMemory, 7: AdaspmvError}


class _IterReport(C.Structure):
    _fields_ = [("iteration", C.c_int64), ("nnz_x", C.c_int64), ("kernel", C.c_int32),
                ("exec_mode", C.c_int32), ("feature_s", C.c_double), ("predict_s", C.c_double),
                ("convert_s", C.c_double), ("kernel_s", C.c_double)]


class _Config(C.Structure):
    _fields_ = [("workers", C.c_int32), ("atomic_private_accumulators", C.c_int32),
                ("semiring", C.c_int32), ("lanes_per_row", C.c_int32),
                ("row_layout", C.c_int32), ("bin_rows", C.c_int32),
                ("bin_tile_nnz", C.c_int64), ("bin_cluster", C.c_int32), ("bin_panel_kib", C.c_int32)]


class _HostOperand(C.Structure):
    _fields_ = [("nnz", C.c_int64), ("indices", C.c_void_p), ("values", C.c_void_p)]


class _HostResult(C.Structure):
    _fields_ = [("form", C.c_int32), ("kernel", C.c_int32), ("capacity", C.c_int64),
                ("indices", C.c_void_p), ("values", C.c_void_p), ("nnz_y", C.c_int64)]


RESULT_DENSE, RESULT_SPARSE, RESULT_AUTO = 0, 1, 2

_lib = None
# adaspmv_allgather_fn (host transport of the dist mode)
_ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)


def load(path: Optional[os.PathLike] = None):
    """Loads libadaspmv_cuda.so (once).  Raises LibraryMissing if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise LibraryMissing(f"{p} is not built; run __graft_entry__.build() "
                             "(make -C paper_2006_16767_b200/csrc)")
    L = C.CDLL(str(p))
    vp, i64, i32, u32 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint32
    P = C.POINTER
    sigs = {
        "adaspmv_ctx_create": [C.c_int, vp, P(vp)],
        "adaspmv_ctx_destroy": [vp],
        "adaspmv_ctx_synchronize": [vp],
        "adaspmv_ctx_stream": [vp],
        "adaspmv_ctx_launch_count": [vp],
        "adaspmv_ctx_set_timing": [vp, C.c_int],
        "adaspmv_ctx_set_bfs_loop": [vp, C.c_int],
        "adaspmv_output_elapsed": [vp, vp, P(C.c_double)],
        "adaspmv_ctx_set_counters": [vp, C.c_int],
        "adaspmv_output_counters": [vp, vp, vp],
        "adaspmv_matrix_create_csr": [vp, i64, i64, vp, vp, vp, C.c_int, P(vp)],
        "adaspmv_matrix_create_csr_device": [vp, i64, i64, i64, vp, vp, vp, C.c_int, P(vp)],
        "adaspmv_matrix_from_triplets": [vp, i64, i64, i64, vp, vp, vp, C.c_int, P(vp)],
        "adaspmv_matrix_load": [vp, C.c_char_p, C.c_int, P(vp)],
        "adaspmv_matrix_write_matrix_market": [vp, vp, C.c_char_p],
        "adaspmv_matrix_save_binary": [vp, vp, C.c_char_p],
        "adaspmv_matrix_transpose": [vp, vp, P(vp)],
        "adaspmv_matrix_destroy": [vp],
        "adaspmv_matrix_dims": [vp, P(i64), P(i64), P(i64), P(C.c_int)],
        "adaspmv_matrix_download": [vp, vp, vp, vp, vp, vp, vp, vp],
        "adaspmv_matrix_features": [vp, vp],
        "adaspmv_matrix_gather_spread": [vp, vp],
        "adaspmv_vector_create": [vp, i64, C.c_int, P(vp)],
        "adaspmv_vector_destroy": [vp],
        "adaspmv_vector_set_sparse": [vp, vp, i64, vp, vp],
        "adaspmv_vector_set_dense": [vp, vp, vp],
        "adaspmv_vector_set_sparse_device": [vp, vp, i64, vp, vp],
        "adaspmv_vector_set_dense_device": [vp, vp, vp],
        "adaspmv_vector_set_output": [vp, vp, vp],
        "adaspmv_vector_prepare": [vp, vp, C.c_int],
        "adaspmv_vector_nnz": [vp, vp, P(i64)],
        "adaspmv_vector_get_sparse": [vp, vp, i64, vp, vp, P(i64)],
        "adaspmv_vector_get_dense": [vp, vp, vp],
        "adaspmv_vector_get_bitmask": [vp, vp, vp],
        "adaspmv_effective_nnz": [vp, vp, vp, P(i64)],
        "adaspmv_features": [vp, vp, vp, u32, vp],
        "adaspmv_bundle_load": [C.c_char_p, P(vp)],
        "adaspmv_bundle_create": [vp, vp, vp, vp, vp, vp, P(vp)],
        "adaspmv_bundle_destroy": [vp],
        "adaspmv_select": [vp, vp, vp, vp, P(C.c_int), P(u32), P(C.c_int)],
        "adaspmv_output_create": [vp, P(vp)],
        "adaspmv_output_destroy": [vp],
        "adaspmv_run": [vp, vp, vp, C.c_int, vp, vp],
        "adaspmv_run_adaptive": [vp, vp, vp, vp, vp, vp, P(C.c_int)],
        "adaspmv_output_info": [vp, P(i64), P(C.c_int), P(C.c_int), P(C.c_int)],
        "adaspmv_output_dense": [vp, vp, vp],
        "adaspmv_output_sparse": [vp, vp, i64, vp, vp, P(i64)],
        "adaspmv_output_device_dense": [vp, vp, P(vp)],
        "adaspmv_output_device_sparse": [vp, vp, P(vp), P(vp), P(i64)],
        "adaspmv_make_partition": [vp, i64, i64, C.c_int, vp],
        "adaspmv_sort_reduce_pairs": [vp, i64, vp, vp, C.c_int, i64, vp, vp, P(i64)],
        "adaspmv_shard_rows": [vp, i64, C.c_int, vp],
        "adaspmv_bfs": [vp, vp, i64, C.c_int, vp, C.c_int, vp, P(i64), vp, i64],
        "adaspmv_pagerank": [vp, vp, C.c_double, C.c_double, i64, vp, C.c_int, vp, P(i64), vp, i64],
        "adaspmv_execute_iteration": [vp, vp, vp, vp, C.c_int, vp, vp, vp],
        "adaspmv_run_batch": [vp, vp, vp, C.c_int, vp, i64, vp, vp, C.c_int],
        "adaspmv_multi_create": [C.c_int, vp, i64, i64, vp, vp, vp, C.c_int, P(vp)],
        "adaspmv_multi_cuts": [vp, vp],
        "adaspmv_multi_run": [vp, vp, C.c_int, vp, i64, vp, vp, vp, vp],
        "adaspmv_multi_destroy": [vp],
        "adaspmv_dist_unique_id": [vp],
        "adaspmv_dist_create_nccl": [vp, C.c_int, C.c_int, vp, P(vp)],
        "adaspmv_dist_create_host": [vp, C.c_int, C.c_int, _ALLGATHER_FN, vp, P(vp)],
        "adaspmv_dist_destroy": [vp],
        "adaspmv_dist_bcast_vector": [vp, vp, C.c_int],
        "adaspmv_dist_allgather_output": [vp, vp, vp, P(i64)],
        "adaspmv_dist_alloc_peer_output": [vp, i64, P(vp)],
        "adaspmv_dist_run_allgather": [vp, vp, vp, C.c_int, vp, vp, vp, P(i64), P(C.c_int)],
        "adaspmv_dist_bfs": [vp, vp, i64, i64, C.c_int, vp, C.c_int, vp, P(i64), vp, i64],
    }
    for name, args in sigs.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    L.adaspmv_ctx_stream.restype = C.c_void_p
    L.adaspmv_ctx_launch_count.restype = C.c_int64
    L.adaspmv_last_error.restype = C.c_char_p
    L.adaspmv_last_error.argtypes = []
    L.adaspmv_version.restype = C.c_char_p
    L.adaspmv_version.argtypes = []
    if path is None:
        _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        msg = _lib.adaspmv_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, AdaspmvError)(msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _dtype_code(dt) -> int:
    dt = np.dtype(dt)
    if dt == np.float64:
        return F64
    if dt == np.float32:
        return F32
    raise InvalidArgument(f"unsupported value dtype {dt}")


def _np_dtype(code: int):
    return np.float64 if code == F64 else np.float32


# --------------------------------------------------------------------------
# kernel identity (kernels.hpp:35-100), kept bit-for-bit
# --------------------------------------------------------------------------
class Pattern(enum.IntEnum):
    ColSpMSpV = 0
    RowSpMSpV = 1
    SpMV = 2


class Workload(enum.IntEnum):
    Direct = 0
    LoadBalanced = 1


class Writeback(enum.IntEnum):
    Atomic = 0
    Sort = 1


_NAMES = ("spmv_direct", "spmv_lb", "row_direct", "row_lb", "col_direct_atomic",
          "col_direct_sort", "col_lb_atomic", "col_lb_sort")  # kernels.hpp:77-79


@dataclass(frozen=True, eq=False)
class KernelId:
    pattern: Pattern = Pattern.SpMV
    workload: Workload = Workload.Direct
    writeback: Writeback = Writeback.Atomic

    kCount = 8

    def index(self) -> int:  # kernels.hpp:52-60
        lb = 1 if self.workload == Workload.LoadBalanced else 0
        if self.pattern == Pattern.SpMV:
            return lb
        if self.pattern == Pattern.RowSpMSpV:
            return 2 + lb
        return 4 + 2 * lb + (1 if self.writeback == Writeback.Sort else 0)

    @staticmethod
    def from_index(i: int) -> "KernelId":  # kernels.hpp:62-74
        table = {
            0: (Pattern.SpMV, Workload.Direct, Writeback.Atomic),
            1: (Pattern.SpMV, Workload.LoadBalanced, Writeback.Atomic),
            2: (Pattern.RowSpMSpV, Workload.Direct, Writeback.Atomic),
            3: (Pattern.RowSpMSpV, Workload.LoadBalanced, Writeback.Atomic),
            4: (Pattern.ColSpMSpV, Workload.Direct, Writeback.Atomic),
            5: (Pattern.ColSpMSpV, Workload.Direct, Writeback.Sort),
            6: (Pattern.ColSpMSpV, Workload.LoadBalanced, Writeback.Atomic),
            7: (Pattern.ColSpMSpV, Workload.LoadBalanced, Writeback.Sort),
        }
        if i not in table:
            raise InvalidArgument("kernel index out of range")
        return KernelId(*table[i])

    def name(self) -> str:
        return _NAMES[self.index()]

    @staticmethod
    def parse(s: str) -> Optional["KernelId"]:
        for i in range(8):
            if _NAMES[i] == s:
                return KernelId.from_index(i)
        return None

    def __eq__(self, o):  # kernels.hpp:89-92: write-back only matters for ColSpMSpV
        if not isinstance(o, KernelId):
            return NotImplemented
        if self.pattern != o.pattern or self.workload != o.workload:
            return False
        return self.pattern != Pattern.ColSpMSpV or self.writeback == o.writeback

    def __hash__(self):
        return hash(self.index())

    def __repr__(self):
        return f"KernelId({self.name()})"


def all_kernels():
    return [KernelId.from_index(i) for i in range(8)]


# --------------------------------------------------------------------------
# host value types (sparse.hpp:99-151)
# --------------------------------------------------------------------------
class DenseVector:
    def __init__(self, values):
        self.values = np.ascontiguousarray(values)

    def size(self) -> int:
        return len(self.values)

    def __len__(self):
        return len(self.values)


class SparseVector:
    def __init__(self, length: int, indices=(), values=(), dtype=np.float64):
        self.length = int(length)
        self.indices = np.ascontiguousarray(indices, dtype=np.int64)
        self.values = np.ascontiguousarray(values, dtype=dtype if len(values) == 0 else None)
        if self.values.dtype not in (np.float32, np.float64):
            self.values = self.values.astype(np.float64)

    def nnz(self) -> int:
        return len(self.indices)

    def validate(self):  # sparse.hpp:120-129
        if len(self.indices) != len(self.values):
            raise InvalidArgument("sparse vector: indices/values length mismatch")
        if len(self.indices):
            if self.indices.min() < 0 or self.indices.max() >= self.length:
                raise InvalidArgument("sparse vector: index out of range")
            if np.any(np.diff(self.indices) <= 0):
                raise InvalidArgument("sparse vector: indices not strictly increasing")


class BitMask:
    """Packed LSB-first u64 words (sparse.hpp:133-151)."""

    def __init__(self, length: int, words=None):
        self.length = int(length)
        self.words = (np.zeros((length + 63) // 64, np.uint64) if words is None
                      else np.ascontiguousarray(words, dtype=np.uint64))

    def test(self, i: int) -> bool:
        return bool((int(self.words[i >> 6]) >> (i & 63)) & 1)

    def popcount(self) -> int:
        return int(sum(bin(int(w)).count("1") for w in self.words))


@dataclass
class KernelConfig:  # kernels.hpp:154-162 (+ device knobs)
    workers: int = 0
    atomic_private_accumulators: bool = False
    semiring: int = PLUS_TIMES
    lanes_per_row: int = 0
    row_layout: int = 0       # K0/K2: 0 auto, 1 CSR gather, 2 row bins
    bin_rows: int = 0         # rows per bin override (0 = auto)
    bin_tile_nnz: int = 0     # entries per bin tile override (0 = auto)
    bin_cluster: int = 0      # CTAs per bin tile: 1 single, 2 cluster pair, 0 auto
    bin_panel_kib: int = 0    # x KiB per column panel of the row bins (<= 0: one panel)

    def _c(self) -> _Config:
        c = _Config()
        c.workers = int(self.workers)
        c.atomic_private_accumulators = int(bool(self.atomic_private_accumulators))
        c.semiring = int(self.semiring)
        c.lanes_per_row = int(self.lanes_per_row)
        c.row_layout = int(self.row_layout)
        c.bin_rows = int(self.bin_rows)
        c.bin_tile_nnz = int(self.bin_tile_nnz)
        c.bin_cluster = int(self.bin_cluster)
        c.bin_panel_kib = int(self.bin_panel_kib)
        return c


@dataclass
class OperandViews:  # kernels.hpp:171-175
    dense: Optional[DenseVector] = None
    sparse: Optional[SparseVector] = None
    mask: Optional[BitMask] = None


# --------------------------------------------------------------------------
# device objects
# --------------------------------------------------------------------------
class Context:
    """One device + one stream (replaces the reference ThreadPool)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        load()
        h = C.c_void_p()
        _check(_lib.adaspmv_ctx_create(int(device), C.c_void_p(stream) if stream else None, C.byref(h)))
        self.h = h
        self.device = device

    def synchronize(self):
        _check(_lib.adaspmv_ctx_synchronize(self.h))

    @property
    def stream(self) -> int:
        return int(_lib.adaspmv_ctx_stream(self.h) or 0)

    @property
    def launches(self) -> int:
        return int(_lib.adaspmv_ctx_launch_count(self.h))

    def set_counters(self, enable: bool = True):
        """KernelCounters for every following run (kernels.hpp:106-111)."""
        _check(_lib.adaspmv_ctx_set_counters(self.h, 1 if enable else 0))

    def set_bfs_loop(self, host_loop: bool = True):
        """adaspmv_ctx_set_bfs_loop: True = host-driven level loop, False (the
        context default) = the device-resident BFS graph where it applies."""
        _check(_lib.adaspmv_ctx_set_bfs_loop(self.h, int(bool(host_loop))))

    def set_timing(self, enable: bool = True):
        """Bracket every multiply with CUDA events (MultiplyOutput.elapsed())."""
        _check(_lib.adaspmv_ctx_set_timing(self.h, int(bool(enable))))

    def close(self):
        if getattr(self, "h", None):
            _lib.adaspmv_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


class DualMatrix:
    """Device-resident CSR + CSC (sparse.hpp:204-259)."""

    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx
        r, c, z, d = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int()
        _check(_lib.adaspmv_matrix_dims(handle, C.byref(r), C.byref(c), C.byref(z), C.byref(d)))
        self._rows, self._cols, self._nnz, self.dtype_code = r.value, c.value, z.value, d.value

    def rows(self) -> int:
        return self._rows

    def cols(self) -> int:
        return self._cols

    def nnz(self) -> int:
        return self._nnz

    @property
    def dtype(self):
        return _np_dtype(self.dtype_code)

    @staticmethod
    def from_csr(rows, cols, row_offsets, col_indices, values=None, dtype=None,
                 ctx: Optional[Context] = None) -> "DualMatrix":
        """DualMatrix::from_csr (sparse.hpp:212-217); values=None -> pattern (1.0)."""
        ctx = ctx or default_context()
        ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
        ci = np.ascontiguousarray(col_indices, dtype=np.int64)
        if dtype is None:
            dtype = np.float64 if values is None else np.asarray(values).dtype
        code = _dtype_code(dtype)
        vals = None if values is None else np.ascontiguousarray(values, dtype=_np_dtype(code))
        if len(ro) != rows + 1:
            raise InvalidArgument("csr: row_offsets length != rows+1")
        if ro[-1] != len(ci) or (vals is not None and len(vals) != len(ci)):
            raise InvalidArgument("csr: array lengths inconsistent with nnz")
        h = C.c_void_p()
        _check(_lib.adaspmv_matrix_create_csr(ctx.h, int(rows), int(cols), _ptr(ro), _ptr(ci), _ptr(vals),
                                              code, C.byref(h)))
        return DualMatrix(h, ctx)

    @staticmethod
    def from_triplets(rows, cols, t_rows, t_cols, t_values, dtype=np.float64,
                      ctx: Optional[Context] = None) -> "DualMatrix":
        """DualMatrix::from_triplets (sparse.hpp:220-258)."""
        ctx = ctx or default_context()
        code = _dtype_code(dtype)
        tr = np.ascontiguousarray(t_rows, dtype=np.int64)
        tc = np.ascontiguousarray(t_cols, dtype=np.int64)
        tv = np.ascontiguousarray(t_values, dtype=_np_dtype(code))
        if not (len(tr) == len(tc) == len(tv)):
            raise InvalidArgument("triplet arrays differ in length")
        h = C.c_void_p()
        _check(_lib.adaspmv_matrix_from_triplets(ctx.h, int(rows), int(cols), len(tr), _ptr(tr), _ptr(tc),
                                                 _ptr(tv), code, C.byref(h)))
        return DualMatrix(h, ctx)

    @staticmethod
    def from_device(rows, cols, nnz, d_row_offsets: int, d_col_indices: int, d_values: Optional[int],
                    dtype=np.float32, ctx: Optional[Context] = None) -> "DualMatrix":
        """From device-resident CSR (int64 offsets, int32 indices; raw pointers)."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(_lib.adaspmv_matrix_create_csr_device(ctx.h, int(rows), int(cols), int(nnz),
                                                     C.c_void_p(d_row_offsets), C.c_void_p(d_col_indices),
                                                     C.c_void_p(d_values) if d_values else None,
                                                     _dtype_code(dtype), C.byref(h)))
        return DualMatrix(h, ctx)

    def download(self):
        """-> (row_offsets, col_indices, values, col_offsets, row_indices, csc_values)."""
        z = self._nnz
        dt = self.dtype
        ro = np.zeros(self._rows + 1, np.int64)
        ci = np.zeros(max(z, 1), np.int64)
        cv = np.zeros(max(z, 1), dt)
        co = np.zeros(self._cols + 1, np.int64)
        ri = np.zeros(max(z, 1), np.int64)
        rv = np.zeros(max(z, 1), dt)
        _check(_lib.adaspmv_matrix_download(self.ctx.h, self.h, _ptr(ro), _ptr(ci), _ptr(cv), _ptr(co),
                                            _ptr(ri), _ptr(rv)))
        return ro, ci[:z], cv[:z], co, ri[:z], rv[:z]

    def features(self) -> np.ndarray:
        out = np.zeros(9, np.float64)
        _check(_lib.adaspmv_matrix_features(self.h, _ptr(out)))
        return out

    def gather_spread(self) -> float:
        out = C.c_double()
        _check(_lib.adaspmv_matrix_gather_spread(self.h, C.byref(out)))
        return out.value

    def transpose(self) -> "DualMatrix":
        h = C.c_void_p()
        _check(_lib.adaspmv_matrix_transpose(self.ctx.h, self.h, C.byref(h)))
        return DualMatrix(h, self.ctx)

    def write_matrix_market(self, path):
        _check(_lib.adaspmv_matrix_write_matrix_market(self.ctx.h, self.h, str(path).encode()))

    def save_binary(self, path):
        _check(_lib.adaspmv_matrix_save_binary(self.ctx.h, self.h, str(path).encode()))

    def close(self):
        if getattr(self, "h", None):
            _lib.adaspmv_matrix_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def load_matrix(path, dtype=np.float64, ctx: Optional[Context] = None) -> DualMatrix:
    """load_matrix (matrix_market.hpp:228-238)."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    _check(_lib.adaspmv_matrix_load(ctx.h, str(path).encode(), _dtype_code(dtype), C.byref(h)))
    return DualMatrix(h, ctx)


def transpose(m: DualMatrix) -> DualMatrix:
    return m.transpose()


class DeviceVector:
    """One operand x on the device with its lazily built representations."""

    def __init__(self, length: int, dtype=np.float64, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.length = int(length)
        self.dtype = np.dtype(dtype)
        h = C.c_void_p()
        _check(_lib.adaspmv_vector_create(self.ctx.h, self.length, _dtype_code(dtype), C.byref(h)))
        self.h = h
        self._keep = None

    def set_sparse(self, indices, values):
        idx = np.ascontiguousarray(indices, dtype=np.int64)
        val = np.ascontiguousarray(values, dtype=self.dtype)
        if len(idx) != len(val):
            raise InvalidArgument("sparse vector: indices/values length mismatch")
        self._keep = (idx, val)  # async H2D source must outlive the copy
        _check(_lib.adaspmv_vector_set_sparse(self.ctx.h, self.h, len(idx), _ptr(idx), _ptr(val)))
        return self

    def set_dense(self, values):
        val = np.ascontiguousarray(values, dtype=self.dtype)
        if len(val) != self.length:
            raise InvalidArgument("dense vector length mismatch")
        self._keep = val
        _check(_lib.adaspmv_vector_set_dense(self.ctx.h, self.h, _ptr(val)))
        return self

    def set_sparse_device(self, nnz, d_indices: int, d_values: int):
        _check(_lib.adaspmv_vector_set_sparse_device(self.ctx.h, self.h, int(nnz), C.c_void_p(d_indices),
                                                     C.c_void_p(d_values)))
        return self

    def set_dense_device(self, d_values: int):
        _check(_lib.adaspmv_vector_set_dense_device(self.ctx.h, self.h, C.c_void_p(d_values)))
        return self

    def set_output(self, y: "MultiplyOutput"):
        _check(_lib.adaspmv_vector_set_output(self.ctx.h, self.h, y.h))
        return self

    def prepare(self, kernel: int | KernelId):
        k = kernel.index() if isinstance(kernel, KernelId) else int(kernel)
        _check(_lib.adaspmv_vector_prepare(self.ctx.h, self.h, k))

    def nnz(self) -> int:
        n = C.c_int64()
        _check(_lib.adaspmv_vector_nnz(self.ctx.h, self.h, C.byref(n)))
        return n.value

    def sparse(self) -> SparseVector:
        n = C.c_int64()
        _check(_lib.adaspmv_vector_get_sparse(self.ctx.h, self.h, 0, None, None, C.byref(n)))
        idx = np.zeros(max(n.value, 1), np.int64)
        val = np.zeros(max(n.value, 1), self.dtype)
        _check(_lib.adaspmv_vector_get_sparse(self.ctx.h, self.h, n.value, _ptr(idx), _ptr(val), C.byref(n)))
        return SparseVector(self.length, idx[:n.value], val[:n.value])

    def dense(self) -> DenseVector:
        out = np.zeros(self.length, self.dtype)
        _check(_lib.adaspmv_vector_get_dense(self.ctx.h, self.h, _ptr(out)))
        return DenseVector(out)

    def bitmask(self) -> BitMask:
        b = BitMask(self.length)
        _check(_lib.adaspmv_vector_get_bitmask(self.ctx.h, self.h, _ptr(b.words)))
        return b

    def close(self):
        if getattr(self, "h", None):
            _lib.adaspmv_vector_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MultiplyOutput:
    """y in the representation the kernel produced (kernels.hpp:116-152)."""

    def __init__(self, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        _check(_lib.adaspmv_output_create(self.ctx.h, C.byref(h)))
        self.h = h

    def _info(self):
        n, hd, hs, dt = C.c_int64(), C.c_int(), C.c_int(), C.c_int()
        _check(_lib.adaspmv_output_info(self.h, C.byref(n), C.byref(hd), C.byref(hs), C.byref(dt)))
        return n.value, bool(hd.value), bool(hs.value), _np_dtype(dt.value)

    def size(self) -> int:
        return self._info()[0]

    def has_dense(self) -> bool:
        return self._info()[1]

    def has_sparse(self) -> bool:
        return self._info()[2]

    def dense(self) -> DenseVector:
        n, _, _, dt = self._info()
        out = np.zeros(n, dt)
        _check(_lib.adaspmv_output_dense(self.ctx.h, self.h, _ptr(out)))
        return DenseVector(out)

    def nnz(self) -> int:
        k = C.c_int64()
        _check(_lib.adaspmv_output_sparse(self.ctx.h, self.h, 0, None, None, C.byref(k)))
        return k.value

    def sparse(self) -> SparseVector:
        n, _, _, dt = self._info()
        k = self.nnz()
        idx = np.empty(max(k, 1), np.int64)
        val = np.empty(max(k, 1), dt)
        kk = C.c_int64()
        _check(_lib.adaspmv_output_sparse(self.ctx.h, self.h, k, _ptr(idx), _ptr(val), C.byref(kk)))
        return SparseVector(n, idx[:k], val[:k])

    def counters(self) -> dict:
        """KernelCounters of the run that produced this output (the context
        must count): values_read, pairs_emitted, cas_retries."""
        c = np.zeros(3, np.uint64)
        _check(_lib.adaspmv_output_counters(self.ctx.h, self.h, _ptr(c)))
        return dict(values_read=int(c[0]), pairs_emitted=int(c[1]), cas_retries=int(c[2]))

    def elapsed(self) -> float:
        """Device seconds of the last timed run (Context.set_timing)."""
        s = C.c_double()
        _check(_lib.adaspmv_output_elapsed(self.ctx.h, self.h, C.byref(s)))
        return s.value

    def device_dense(self) -> int:
        p = C.c_void_p()
        _check(_lib.adaspmv_output_device_dense(self.ctx.h, self.h, C.byref(p)))
        return int(p.value or 0)

    def device_sparse(self):
        pi, pv, k = C.c_void_p(), C.c_void_p(), C.c_int64()
        _check(_lib.adaspmv_output_device_sparse(self.ctx.h, self.h, C.byref(pi), C.byref(pv), C.byref(k)))
        return int(pi.value or 0), int(pv.value or 0), k.value

    def close(self):
        if getattr(self, "h", None):
            _lib.adaspmv_output_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------------
# selector
# --------------------------------------------------------------------------
class SelectorBundle:
    def __init__(self, handle):
        self.h = handle

    @staticmethod
    def load(path) -> "SelectorBundle":
        load()
        h = C.c_void_p()
        _check(_lib.adaspmv_bundle_load(str(path).encode(), C.byref(h)))
        return SelectorBundle(h)

    @staticmethod
    def from_trees(trees) -> "SelectorBundle":
        """trees = [pattern, workload, writeback], each a dict of node arrays
        feature/threshold/left/right/leaf (feature < 0 = leaf)."""
        load()
        keep = []
        arrs = {k: (C.c_void_p * 3)() for k in ("feature", "threshold", "left", "right", "leaf")}
        n = (C.c_int32 * 3)()
        for t, tree in enumerate(trees):
            n[t] = len(tree["feature"])
            for k in arrs:
                a = np.ascontiguousarray(tree[k], dtype=np.float64 if k == "threshold" else np.int32)
                keep.append(a)
                arrs[k][t] = a.ctypes.data
        h = C.c_void_p()
        _check(_lib.adaspmv_bundle_create(C.cast(n, C.c_void_p), C.cast(arrs["feature"], C.c_void_p),
                                          C.cast(arrs["threshold"], C.c_void_p), C.cast(arrs["left"], C.c_void_p),
                                          C.cast(arrs["right"], C.c_void_p), C.cast(arrs["leaf"], C.c_void_p),
                                          C.byref(h)))
        return SelectorBundle(h)

    @staticmethod
    def constant(pattern: int, workload: int, writeback: int = 0) -> "SelectorBundle":
        """Stub bundle with constant leaves."""
        leaf = lambda c: {"feature": [-1], "threshold": [0.0], "left": [-1], "right": [-1], "leaf": [c]}
        return SelectorBundle.from_trees([leaf(pattern), leaf(workload), leaf(writeback)])

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.adaspmv_bundle_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _as_device_vector(m: DualMatrix, views) -> DeviceVector:
    if isinstance(views, DeviceVector):
        return views
    v = DeviceVector(m.cols(), m.dtype, m.ctx)
    if isinstance(views, DenseVector):
        return v.set_dense(views.values)
    if isinstance(views, SparseVector):
        return v.set_sparse(views.indices, views.values)
    if isinstance(views, OperandViews):
        if views.sparse is not None:
            return v.set_sparse(views.sparse.indices, views.sparse.values)
        if views.dense is not None:
            return v.set_dense(views.dense.values)
    raise InvalidArgument("no operand given")


def features(m: DualMatrix, x, mask: int = 0x1FFF) -> np.ndarray:
    """The 13 Table-1 features; NaN where not requested."""
    v = _as_device_vector(m, x) if mask >> 9 else None
    out = np.full(13, np.nan)
    _check(_lib.adaspmv_features(m.ctx.h, m.h, v.h if v else None, int(mask), _ptr(out)))
    return out


def predict_kernel(m: DualMatrix, x, bundle: SelectorBundle):
    """-> (KernelId, features_used_mask, trees_evaluated)."""
    v = _as_device_vector(m, x)
    k, used, nt = C.c_int(), C.c_uint32(), C.c_int()
    _check(_lib.adaspmv_select(m.ctx.h, m.h, v.h, bundle.h, C.byref(k), C.byref(used), C.byref(nt)))
    return KernelId.from_index(k.value), used.value, nt.value


# --------------------------------------------------------------------------
# run_kernel and the direct entries (kernels.hpp:290-535)
# --------------------------------------------------------------------------
def run_kernel(m: DualMatrix, kid: KernelId | int, views, cfg: Optional[KernelConfig] = None,
               out: Optional[MultiplyOutput] = None) -> MultiplyOutput:
    """run_kernel (kernels.hpp:520-535).  `views` is an OperandViews, a
    DenseVector/SparseVector, or a DeviceVector.  Like the reference, the
    pattern's operand must be present in an OperandViews (:524-534)."""
    k = kid.index() if isinstance(kid, KernelId) else int(kid)
    if isinstance(views, OperandViews):
        pat = KernelId.from_index(k).pattern
        if pat == Pattern.SpMV and views.dense is None:
            raise InvalidArgument("SpMV requires a dense operand")
        if pat == Pattern.RowSpMSpV and (views.dense is None or views.mask is None):
            raise InvalidArgument("RowSpMSpV requires dense values and a bitmask")
        if pat == Pattern.ColSpMSpV and views.sparse is None:
            raise InvalidArgument("ColSpMSpV requires a sparse operand")
        if pat != Pattern.ColSpMSpV:
            views = views.dense
        else:
            views = views.sparse
    if isinstance(views, (DenseVector,)) and views.size() != m.cols():
        raise InvalidArgument("multiply: vector length != matrix columns")
    if isinstance(views, SparseVector) and views.length != m.cols():
        raise InvalidArgument("multiply: vector length != matrix columns")
    v = _as_device_vector(m, views)
    out = out or MultiplyOutput(m.ctx)
    c = (cfg or KernelConfig())._c()
    _check(_lib.adaspmv_run(m.ctx.h, m.h, v.h, k, C.byref(c), out.h))
    out._operand = v  # keep x alive while the output may be lazily converted
    return out


def spmv(m: DualMatrix, x: DenseVector, workload: Workload, cfg: Optional[KernelConfig] = None):
    return run_kernel(m, KernelId(Pattern.SpMV, workload), x, cfg)


def spmspv_row(m: DualMatrix, x: SparseVector | DenseVector, workload: Workload,
               cfg: Optional[KernelConfig] = None):
    return run_kernel(m, KernelId(Pattern.RowSpMSpV, workload), x, cfg)


def spmspv_col(m: DualMatrix, x: SparseVector, workload: Workload, writeback: Writeback,
               cfg: Optional[KernelConfig] = None):
    return run_kernel(m, KernelId(Pattern.ColSpMSpV, workload, writeback), x, cfg)


def run_adaptive(m: DualMatrix, x, bundle: SelectorBundle, cfg: Optional[KernelConfig] = None,
                 out: Optional[MultiplyOutput] = None):
    """Select then run; -> (MultiplyOutput, KernelId)."""
    v = _as_device_vector(m, x)
    out = out or MultiplyOutput(m.ctx)
    c = (cfg or KernelConfig())._c()
    k = C.c_int()
    _check(_lib.adaspmv_run_adaptive(m.ctx.h, m.h, v.h, bundle.h, C.byref(c), out.h, C.byref(k)))
    out._operand = v
    return out, KernelId.from_index(k.value)


class BatchResult:
    """One result of run_batch: `kernel` (KernelId), `is_sparse`, and
    `dense` (DenseVector) or `sparse` (SparseVector, int64 indices)."""

    def __init__(self, kernel, is_sparse, dense=None, sparse=None):
        self.kernel, self.is_sparse, self.dense, self.sparse = kernel, is_sparse, dense, sparse


def run_batch(m: DualMatrix, xs, bundle: Optional[SelectorBundle] = None, force_kernel: int = -1,
              form: int = RESULT_AUTO, cfg: Optional[KernelConfig] = None, lanes: int = 0,
              buffers=None):
    """adaspmv_run_batch: y_k = A x_k for every host operand in `xs`
    (DenseVector, SparseVector, or numpy arrays: 1-D values = dense, a pair
    (indices, values) = sparse), selected by `bundle` (else `force_kernel`),
    pipelined over `lanes` streams.  `buffers` (optional, one (indices int64,
    values) pair of length rows per operand, ideally pinned) receive the
    results without allocation; the returned BatchResults view them."""
    ops = (_HostOperand * max(len(xs), 1))()
    res = (_HostResult * max(len(xs), 1))()
    keep = []
    rows = m.rows()
    vdt = m.dtype
    bufs = []
    for k, x in enumerate(xs):
        if isinstance(x, DenseVector):
            x = np.ascontiguousarray(x.values, dtype=vdt)
        elif isinstance(x, SparseVector):
            x = (x.indices, x.values)
        if isinstance(x, tuple):
            xi = np.ascontiguousarray(x[0], dtype=np.int64)
            xv = np.ascontiguousarray(x[1], dtype=vdt)
            keep += [xi, xv]
            ops[k].nnz, ops[k].indices, ops[k].values = len(xi), xi.ctypes.data, xv.ctypes.data
        else:
            xd = np.ascontiguousarray(x, dtype=vdt)
            if len(xd) != m.cols():
                raise InvalidArgument("run_batch: vector length != matrix columns")
            keep.append(xd)
            ops[k].nnz, ops[k].indices, ops[k].values = -1, None, xd.ctypes.data
        if buffers is not None:
            bi, bv = buffers[k]
        else:
            bi = np.empty(rows if form != RESULT_DENSE else 0, np.int64)
            bv = np.empty(rows, vdt)
        bufs.append((bi, bv))
        res[k].form = int(form)
        res[k].capacity = len(bi) if form != RESULT_DENSE else 0
        res[k].indices = bi.ctypes.data if form != RESULT_DENSE and len(bi) else None
        res[k].values = bv.ctypes.data
    c = (cfg or KernelConfig())._c()
    _check(_lib.adaspmv_run_batch(m.ctx.h, m.h, bundle.h if bundle else None, int(force_kernel), C.byref(c),
                                  len(xs), C.cast(ops, C.c_void_p), C.cast(res, C.c_void_p), int(lanes)))
    out = []
    for k in range(len(xs)):
        bi, bv = bufs[k]
        kid = KernelId.from_index(res[k].kernel)
        if res[k].form == RESULT_SPARSE:
            nz = int(res[k].nnz_y)
            out.append(BatchResult(kid, True, sparse=SparseVector(rows, bi[:nz], bv[:nz], dtype=vdt)))
        else:
            out.append(BatchResult(kid, False, dense=DenseVector(bv[:rows])))
    return out


class MultiMatrix:
    """adaspmv_multi: the row-partitioned mode in one process -- G row blocks
    of ~nnz/G nonzeros, block g on devices[g]."""

    def __init__(self, rows, cols, row_offsets, col_indices, values=None, devices=(0,), dtype=None):
        load()
        ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
        ci = np.ascontiguousarray(col_indices, dtype=np.int64)
        if dtype is None:
            dtype = np.float64 if values is None else np.asarray(values).dtype
        self.dtype = np.dtype(dtype)
        vals = None if values is None else np.ascontiguousarray(values, dtype=self.dtype)
        dev = np.ascontiguousarray(devices, dtype=np.int32)
        self.rows, self.cols, self.ngpu = int(rows), int(cols), len(dev)
        self.h = C.c_void_p()
        _check(_lib.adaspmv_multi_create(self.ngpu, _ptr(dev), self.rows, self.cols, _ptr(ro), _ptr(ci),
                                         _ptr(vals), _dtype_code(self.dtype), C.byref(self.h)))

    def cuts(self) -> np.ndarray:
        c = np.zeros(self.ngpu + 1, np.int64)
        _check(_lib.adaspmv_multi_cuts(self.h, _ptr(c)))
        return c

    def multiply(self, x, bundle: Optional["SelectorBundle"] = None, force_kernel: int = -1,
                 cfg: Optional[KernelConfig] = None):
        """y = A x (x: dense values, or an (indices, values) pair) -> (y, per-block KernelIds)."""
        y = np.empty(self.rows, self.dtype)
        ks = np.zeros(self.ngpu, np.int32)
        c = (cfg or KernelConfig())._c()
        if isinstance(x, tuple):
            xi = np.ascontiguousarray(x[0], dtype=np.int64)
            xv = np.ascontiguousarray(x[1], dtype=self.dtype)
            nnz = len(xi)
        else:
            xi, xv, nnz = None, np.ascontiguousarray(x, dtype=self.dtype), -1
        _check(_lib.adaspmv_multi_run(self.h, bundle.h if bundle else None, int(force_kernel), C.byref(c), nnz,
                                      _ptr(xi), _ptr(xv), _ptr(y), _ptr(ks)))
        return y, [KernelId.from_index(int(k)) for k in ks]

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.adaspmv_multi_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dist_unique_id() -> bytes:
    """adaspmv_dist_unique_id: a fresh ncclUniqueId (128 bytes) for rank 0 to share."""
    load()
    buf = (C.c_char * 128)()
    _check(_lib.adaspmv_dist_unique_id(buf))
    return bytes(buf)


class Dist:
    """adaspmv_dist: the exchange of the row-partitioned mode with one process
    per GPU.  `Dist.nccl(ctx, rank, world, uid)` is the
    product transport (NCCL over NVLink); `Dist.host(ctx, rank, world,
    allgather)` routes the exchange through a host callable
    `allgather(bytes) -> list[bytes]` (every rank's contribution, rank order),
    e.g. torch.distributed over gloo -- tests, and ranks sharing one GPU."""

    def __init__(self, ctx: Context, rank: int, world: int, h, keep=None):
        self.ctx, self.rank, self.world, self.h, self._keep = ctx, int(rank), int(world), h, keep

    @classmethod
    def nccl(cls, ctx: Context, rank: int, world: int, uid: bytes) -> "Dist":
        if len(uid) != 128:
            raise InvalidArgument("dist: the NCCL unique id is 128 bytes")
        buf = (C.c_char * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(_lib.adaspmv_dist_create_nccl(ctx.h, int(rank), int(world), buf, C.byref(h)))
        return cls(ctx, rank, world, h)

    @classmethod
    def host(cls, ctx: Context, rank: int, world: int, allgather) -> "Dist":
        def cb(_user, send, nbytes, recv):
            try:
                mine = C.string_at(send, nbytes) if nbytes > 0 else b""
                parts = allgather(mine)
                blob = b"".join(parts)
                if len(blob) != nbytes * world:
                    return 1
                if nbytes > 0:
                    C.memmove(recv, blob, len(blob))
                return 0
            except Exception:  # noqa: BLE001 -- reported to the library as a failed exchange
                return 1
        fn = _ALLGATHER_FN(cb)
        h = C.c_void_p()
        _check(_lib.adaspmv_dist_create_host(ctx.h, int(rank), int(world), fn, None, C.byref(h)))
        return cls(ctx, rank, world, h, keep=fn)

    def bcast_vector(self, x: "DeviceVector", root: int = 0):
        _check(_lib.adaspmv_dist_bcast_vector(self.h, x.h, int(root)))
        return x

    def alloc_peer_output(self, nbytes: int) -> int:
        """Collective: a full-y device buffer shared with every rank (CUDA
        IPC); allgather_output into it uses peer stores over NVLink."""
        p = C.c_void_p()
        _check(_lib.adaspmv_dist_alloc_peer_output(self.h, int(nbytes), C.byref(p)))
        return int(p.value)

    def run_allgather(self, block: DualMatrix, kid: int, x: "DeviceVector", y_full_ptr: int,
                      cfg: Optional[KernelConfig] = None, out: Optional["MultiplyOutput"] = None):
        """Collective: kernel `kid` on this rank's block with the y all-gather
        into the peer output fused into its store epilogue (row-bin K0/K2) or
        following it.  Returns (total rows, fused)."""
        out = out or MultiplyOutput(self.ctx)
        c = (cfg or KernelConfig())._c()
        tot, fused = C.c_int64(), C.c_int()
        _check(_lib.adaspmv_dist_run_allgather(self.h, block.h, x.h, int(kid), C.byref(c), out.h,
                                               C.c_void_p(y_full_ptr), C.byref(tot), C.byref(fused)))
        return tot.value, bool(fused.value)

    def allgather_output(self, y: "MultiplyOutput", y_full_ptr: int) -> int:
        """Every rank's dense y block into the device buffer at y_full_ptr."""
        tot = C.c_int64()
        _check(_lib.adaspmv_dist_allgather_output(self.h, y.h, C.c_void_p(y_full_ptr), C.byref(tot)))
        return tot.value

    def bfs(self, block: DualMatrix, row0: int, source: int = 0, semiring: int = OR_AND,
            bundle: Optional["SelectorBundle"] = None, force_kernel: int = -1, max_reports: int = 4096,
            download_levels: bool = True):
        """-> (levels of this rank's rows or None, this rank's per-level reports)."""
        levels = np.empty(block.rows(), np.int64) if download_levels else None
        nl = C.c_int64()
        reps = _report_buffer(max_reports)
        _check(_lib.adaspmv_dist_bfs(self.h, block.h, int(row0), int(source), int(semiring),
                                     bundle.h if bundle else None, int(force_kernel), _ptr(levels),
                                     C.byref(nl), C.cast(reps, C.c_void_p), max_reports))
        return levels, _reports(reps, nl.value, max_reports)

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.adaspmv_dist_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def execute_iteration(m: DualMatrix, x, bundle: Optional[SelectorBundle] = None, force_kernel: int = -1,
                      cfg: Optional[KernelConfig] = None, out: Optional[MultiplyOutput] = None):
    """execute_iteration -> (MultiplyOutput, IterationReport
    dict: kernel, feature_s, predict_s, convert_s (device), kernel_s (device))."""
    v = _as_device_vector(m, x)
    out = out or MultiplyOutput(m.ctx)
    c = (cfg or KernelConfig())._c()
    rep = _IterReport()
    _check(_lib.adaspmv_execute_iteration(m.ctx.h, m.h, v.h, bundle.h if bundle else None, int(force_kernel),
                                          C.byref(c), out.h, C.byref(rep)))
    out._operand = v
    return out, dict(kernel=KernelId.from_index(rep.kernel), nnz_x=rep.nnz_x, feature_s=rep.feature_s,
                     predict_s=rep.predict_s, convert_s=rep.convert_s, kernel_s=rep.kernel_s)


def run_trace(m: DualMatrix, xs, bundle: Optional[SelectorBundle] = None, force_kernel: int = -1,
              cfg: Optional[KernelConfig] = None, oracle_times=None) -> dict:
    """run_trace: execute_iteration over a sequence of
    vectors -> TraceStats: per-iteration reports, overhead fraction
    (feature + predict + convert over total), kernel-switch
    count, and regret = sum(chosen kernel time) / sum(best time) when
    `oracle_times[i][k]` (seconds of kernel k on vector i) is supplied."""
    out = MultiplyOutput(m.ctx)
    reports = []
    for x in xs:
        _, rep = execute_iteration(m, x, bundle, force_kernel, cfg, out)
        reports.append(rep)
    over = sum(r["feature_s"] + r["predict_s"] + r["convert_s"] for r in reports)
    total = over + sum(r["kernel_s"] for r in reports)
    ks = [r["kernel"].index() for r in reports]
    stats = {"iterations": reports, "overhead_fraction": (over / total) if total > 0 else 0.0,
             "kernel_switches": sum(1 for a, b in zip(ks, ks[1:]) if a != b)}
    if oracle_times is not None and len(reports):
        ot = np.asarray(oracle_times, np.float64)
        stats["regret"] = float(ot[np.arange(len(ks)), ks].sum() / ot.min(axis=1).sum())
    return stats


def effective_nnz(m: DualMatrix, x) -> int:
    v = _as_device_vector(m, x)
    k = C.c_int64()
    _check(_lib.adaspmv_effective_nnz(m.ctx.h, m.h, v.h, C.byref(k)))
    return k.value


def make_partition(offsets, total_items: int, workers: int) -> np.ndarray:
    """make_partition (partition.hpp:37-56) -> array [W,4] of
    (item_begin, item_end, span_begin, span_end)."""
    load()
    o = np.ascontiguousarray(offsets, dtype=np.int64)
    out = np.zeros(4 * max(int(workers), 1), np.int64)
    _check(_lib.adaspmv_make_partition(_ptr(o), len(o), int(total_items), int(workers), _ptr(out)))
    return out.reshape(-1, 4)


def sort_reduce_pairs(rows, values, nrows: int, ctx: Optional[Context] = None) -> SparseVector:
    """sort_reduce_pairs (kernels.hpp:341-345) on the device."""
    ctx = ctx or default_context()
    r = np.ascontiguousarray(rows, dtype=np.int64)
    v = np.ascontiguousarray(values)
    code = _dtype_code(v.dtype)
    oi = np.zeros(max(len(r), 1), np.int64)
    ov = np.zeros(max(len(r), 1), v.dtype)
    k = C.c_int64()
    _check(_lib.adaspmv_sort_reduce_pairs(ctx.h, len(r), _ptr(r), _ptr(v), code, int(nrows), _ptr(oi), _ptr(ov),
                                          C.byref(k)))
    return SparseVector(nrows, oi[:k.value], ov[:k.value])


def shard_rows(row_offsets, nshards: int) -> np.ndarray:
    load()
    ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
    cuts = np.zeros(int(nshards) + 1, np.int64)
    _check(_lib.adaspmv_shard_rows(_ptr(ro), len(ro) - 1, int(nshards), _ptr(cuts)))
    return cuts


def bfs(m: DualMatrix, source: int = 0, semiring: int = OR_AND, bundle: Optional[SelectorBundle] = None,
        force_kernel: int = -1, max_reports: int = 4096, download_levels: bool = True):
    """Level-synchronous BFS -> (levels int64[n] or None, reports list)."""
    levels = np.empty(m.rows(), np.int64) if download_levels else None
    nl = C.c_int64()
    reps = _report_buffer(max_reports)
    _check(_lib.adaspmv_bfs(m.ctx.h, m.h, int(source), int(semiring), bundle.h if bundle else None,
                            int(force_kernel), _ptr(levels), C.byref(nl), C.cast(reps, C.c_void_p), max_reports))
    out = []
    for i in range(min(nl.value, max_reports)):
        r = reps[i]
        out.append(dict(iteration=r.iteration, nnz_x=r.nnz_x, kernel=r.kernel, exec_mode=r.exec_mode,
                        feature_s=r.feature_s, predict_s=r.predict_s, convert_s=r.convert_s,
                        kernel_s=r.kernel_s))
    return levels, out


_report_tls = threading.local()


def _report_buffer(n: int):
    """A per-thread reusable IterationReport array of >= n entries (a fresh
    zeroed ctypes array of the default 4096 reports costs ~80 us per call)."""
    buf = getattr(_report_tls, "buf", None)
    if buf is None or len(buf) < n:
        buf = (_IterReport * max(int(n), 1))()
        _report_tls.buf = buf
    return buf


def _reports(reps, n, max_reports):
    out = []
    for i in range(min(n, max_reports)):
        r = reps[i]
        out.append(dict(iteration=r.iteration, nnz_x=r.nnz_x, kernel=r.kernel, exec_mode=r.exec_mode,
                        feature_s=r.feature_s, predict_s=r.predict_s, convert_s=r.convert_s,
                        kernel_s=r.kernel_s))
    return out


def pagerank_incremental(m: DualMatrix, damping: float = 0.85, prune: float = 1e-6, max_iters: int = 300,
                         bundle: Optional[SelectorBundle] = None, force_kernel: int = -1,
                         max_reports: int = 4096, download_rank: bool = True):
    """Incremental delta-propagation PageRank -> (rank float64[n] or None, reports)."""
    rank = np.empty(m.rows(), np.float64) if download_rank else None
    nit = C.c_int64()
    reps = _report_buffer(max_reports)
    _check(_lib.adaspmv_pagerank(m.ctx.h, m.h, float(damping), float(prune), int(max_iters),
                                 bundle.h if bundle else None, int(force_kernel), _ptr(rank), C.byref(nit),
                                 C.cast(reps, C.c_void_p), max_reports))
    return rank, _reports(reps, nit.value, max_reports)
