"""CPU: the C-ABI library loads, exports every symbol include/adaspmv_cuda.h
declares, and its host-only entry points (partition, row sharding, model
files, error mapping) behave like the reference.  No kernel is launched."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2006_16767_b200 import adaspmv as A
from paper_2006_16767_b200 import selector as S

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "adaspmv_cuda.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(adaspmv_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    A.load()
    out = subprocess.run(["nm", "-D", "--defined-only", str(A.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (adaspmv_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert len(declared_symbols()) >= 45


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(A.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_kernel_id_mirror():
    # kernels.hpp:52-92: index, names, parse, equality ignoring write-back unless Col
    names = ["spmv_direct", "spmv_lb", "row_direct", "row_lb", "col_direct_atomic",
             "col_direct_sort", "col_lb_atomic", "col_lb_sort"]
    for i, n in enumerate(names):
        k = A.KernelId.from_index(i)
        assert k.index() == i and k.name() == n and A.KernelId.parse(n) == k
    assert A.KernelId.parse("nope") is None
    assert A.KernelId(A.Pattern.SpMV, A.Workload.Direct, A.Writeback.Sort) == A.KernelId.from_index(0)
    assert A.KernelId(A.Pattern.ColSpMSpV, A.Workload.Direct, A.Writeback.Sort) != A.KernelId.from_index(4)
    with pytest.raises(A.InvalidArgument):
        A.KernelId.from_index(8)
    assert len(A.all_kernels()) == 8


def test_make_partition_matches_oracle(port):
    rng = np.random.default_rng(0)
    for _ in range(300):
        n = int(rng.integers(1, 60))
        off = np.concatenate([[0], np.cumsum(rng.integers(0, 5, size=n))])
        w = int(rng.integers(1, 40))
        got = A.make_partition(off, int(off[-1]), w)
        assert np.array_equal(got, port.make_partition(off, int(off[-1]), w))
        sizes = got[:, 1] - got[:, 0]
        assert sizes.max() - sizes.min() <= 1
    with pytest.raises(A.InvalidArgument):
        A.make_partition([0, 3], 3, 0)
    with pytest.raises(A.InvalidArgument):
        A.make_partition([0, 3], 4, 2)


def test_shard_rows_balanced_and_whole_rows():
    rng = np.random.default_rng(1)
    for _ in range(100):
        deg = rng.integers(0, 50, size=int(rng.integers(1, 400)))
        ro = np.concatenate([[0], np.cumsum(deg)])
        g = int(rng.integers(1, 9))
        cuts = A.shard_rows(ro, g)
        assert cuts[0] == 0 and cuts[-1] == len(deg) and np.all(np.diff(cuts) >= 0)
        nnz = ro[-1]
        for i in range(1, g):  # cut = first row starting at/after i*nnz/g
            assert ro[cuts[i]] >= nnz * i // g or cuts[i] == len(deg)


def test_bundle_files(tmp_path):
    # the shipped (trained) bundle loads and predicts valid kernels
    b = A.SelectorBundle.load(S.DEFAULT_PATH)
    assert b.h
    shipped = S.read_bundle(S.DEFAULT_PATH)
    rng = np.random.default_rng(0)
    for _ in range(100):
        assert 0 <= S.predict(shipped, rng.random(13) * 1e6) <= 7
    # hand-set cascade: host mirror agrees with the node arrays
    p0 = tmp_path / "default.txt"
    S.write_bundle(p0, S.default_trees())
    trees = S.read_bundle(p0)
    f = np.zeros(13)
    f[12] = 0.01
    f[11] = 100
    assert S.predict(trees, f) == 5  # Col, Direct (gc 0), Sort
    f[12] = 1.0
    assert S.predict(trees, f) == 0
    # round trip
    p = tmp_path / "b.txt"
    S.write_bundle(p, trees)
    assert S.read_bundle(p) == trees
    A.SelectorBundle.load(p)
    # malformed files -> FormatError, no partial bundle
    text = p.read_text()
    for bad in (text[: len(text) // 2], text.replace("adaspmv-bundle 1", "adaspmv-bundle 2"),
                text.replace(S.feature_order_hash(), "0" * 16), "garbage"):
        q = tmp_path / "bad.txt"
        q.write_text(bad)
        with pytest.raises(A.FormatError):
            A.SelectorBundle.load(q)
    with pytest.raises(A.FormatError):
        A.SelectorBundle.load(tmp_path / "missing.txt")
    # a node reading a feature outside its tree's mask is rejected
    bad = dict(trees)
    bad["workload"] = {"feature": [11, -1, -1], "threshold": [1.0, 0, 0], "left": [1, -1, -1],
                       "right": [2, -1, -1], "leaf": [-1, 0, 1]}
    S.write_bundle(p, bad)
    with pytest.raises(A.FormatError):
        A.SelectorBundle.load(p)
    with pytest.raises(A.InvalidArgument):
        A.SelectorBundle.from_trees([bad["pattern"], bad["workload"], bad["writeback"]])
    # schema 2 (a workload tree for the ColSpMSpV family) round-trips and loads;
    # the shipped v2 bundle too
    v2 = dict(trees)
    v2["workload_col"] = {"feature": [11, -1, -1], "threshold": [5000.0, 0, 0], "left": [1, -1, -1],
                          "right": [2, -1, -1], "leaf": [-1, 0, 1]}
    S.write_bundle(p, v2)
    assert p.read_text().startswith("adaspmv-bundle 2") and S.read_bundle(p) == v2
    A.SelectorBundle.load(p)
    f = np.zeros(13)
    f[12], f[11] = 0.01, 100.0  # Col; workload_col: nnz_s <= 5000 -> Direct; Sort
    assert S.predict(v2, f) == 5
    f[11] = 9000.0  # -> LB; write-back tree: nnz_s > 4096 -> Atomic
    assert S.predict(v2, f) == 6
    A.SelectorBundle.load(S.DEFAULT_PATH.parent / "b200_bundle_v2.txt")


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(A.CudaError):
        A.Context(0)


def test_cpp_wrapper_compiles_and_links(tmp_path):
    """include/adaspmv_cuda.hpp (the reference-shaped C++ API) compiles
    against the C-ABI and links the library; host-only calls run."""
    src = tmp_path / "t.cpp"
    src.write_text(r'''
#include "adaspmv_cuda.hpp"
#include <cstdio>
int main() {
  using namespace adaspmv::cuda;
  KernelId k = KernelId::from_index(7);
  if (k.index() != 7 || k.name() != "col_lb_sort") return 1;
  if (!(KernelId::parse("spmv_lb") == KernelId::from_index(1))) return 2;
  std::vector<adaspmv::cuda::index_t> off = {0, 0, 0, 9, 10};
  WorkPartition p = make_partition(off, 10, 2);
  if (p.worker_ranges[1].span_begin != 2 || p.worker_ranges[1].span_end != 4) return 3;
  try { make_partition(off, 10, 0); return 4; } catch (const std::invalid_argument&) {}
  std::puts("ok");
  return 0;
}
''')
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(src), "-o", str(exe),
                    str(A.LIB_PATH), f"-Wl,-rpath,{A.LIB_PATH.parent}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.strip() == "ok", (out.returncode, out.stderr)
