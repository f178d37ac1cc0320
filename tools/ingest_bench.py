"""Ingestion at scale: time DualMatrix::from_triplets and
load_matrix (Matrix Market, parallel parser) against the reference's own
implementations (oracle/_ref, single-threaded by construction) on a
uniform-random matrix; prints one JSON line.

  python tools/ingest_bench.py --log-rows 22 --log-draws 24 --out gpurun_out/ingest.json
"""
import argparse
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_16767_b200 import adaspmv as A  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log-rows", type=int, default=22)
    ap.add_argument("--log-draws", type=int, default=24)
    ap.add_argument("--no-ref", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = cols = 1 << a.log_rows
    n = 1 << a.log_draws
    rng = np.random.default_rng(1)
    tr = rng.integers(0, rows, n, dtype=np.int64)
    tc = rng.integers(0, cols, n, dtype=np.int64)
    tv = rng.uniform(-1, 1, n).astype(np.float32)
    ctx = A.Context(0)
    A.DualMatrix.from_triplets(4, 4, [0, 1], [1, 2], np.ones(2, np.float32), dtype=np.float32, ctx=ctx)  # warm
    res = {"rows": rows, "cols": cols, "triplets": n, "host_threads": os.cpu_count()}
    t0 = time.perf_counter()
    m = A.DualMatrix.from_triplets(rows, cols, tr, tc, tv, dtype=np.float32, ctx=ctx)
    ctx.synchronize()
    res["from_triplets_s"] = round(time.perf_counter() - t0, 3)
    res["nnz"] = m.nnz()
    with tempfile.TemporaryDirectory(dir=os.environ.get("TMPDIR", "/tmp")) as d:
        p = Path(d) / "c.mtx"
        t0 = time.perf_counter()
        m.write_matrix_market(p)
        res["write_mm_s"] = round(time.perf_counter() - t0, 3)
        res["mm_bytes"] = p.stat().st_size
        t0 = time.perf_counter()
        m2 = A.load_matrix(p, dtype=np.float32, ctx=ctx)
        ctx.synchronize()
        res["load_mm_s"] = round(time.perf_counter() - t0, 3)
        pb = Path(d) / "c.bin"
        m.save_binary(pb)
        t0 = time.perf_counter()
        m3 = A.load_matrix(pb, dtype=np.float32, ctx=ctx)
        ctx.synchronize()
        res["load_binary_s"] = round(time.perf_counter() - t0, 3)
        a1, a2, a3 = m.download(), m2.download(), m3.download()
        res["mm_round_trip_exact"] = all(np.array_equal(x, y) for x, y in zip(a1[:3], a2[:3]))
        res["bin_round_trip_exact"] = all(np.array_equal(x, y) for x, y in zip(a1[:3], a3[:3]))
        if not a.no_ref:
            from oracle.oracle import Ref
            ref = Ref(np.float32)
            t0 = time.perf_counter()
            R = ref.from_triplets(rows, cols, tr, tc, tv)
            res["ref_from_triplets_s"] = round(time.perf_counter() - t0, 3)
            ro, ci, cv, *_ = R.export()
            res["from_triplets_exact_vs_ref"] = bool(np.array_equal(ro, a1[0]) and np.array_equal(ci, a1[1])
                                                     and cv.tobytes() == a1[2].tobytes())
            del R
            t0 = time.perf_counter()
            R = ref.load_matrix(p)
            res["ref_load_mm_s"] = round(time.perf_counter() - t0, 3)
            del R
            t0 = time.perf_counter()
            R = ref.load_matrix(pb)
            res["ref_load_binary_s"] = round(time.perf_counter() - t0, 3)
    line = json.dumps(res)
    print(line)
    if a.out:
        Path(a.out).write_text(line + "\n")


if __name__ == "__main__":
    main()
