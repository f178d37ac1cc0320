#!/usr/bin/env python3
"""bench.py -- BASELINE.json's metric on its configurations.

  "GFLOP/s and HBM GB/s (% of roofline) vs x sparsity; selector regret vs best"

Headline (value, e2e, roofline): configs[1] = C2, uniform random 4M x 4M,
2^26 iid draws (~64M nnz), fp32, x-sparsity sweep 0.001 % .. 100 % across all
8 kernels + the selector.  A *step* is one adaptive pass over the sweep: for
each of the 7 points select a kernel (C++ decision-tree hook) and run it,
inputs resident in HBM.  value = sum(2 nnz_s) / sum(t).  Every point is also
timed with all 8 kernels (best-of-8, regret).

The other single-GPU configurations ride in the same JSON line under
"configs" (C1 Laplacian fp64 at x = 100 % / 1 %, C3 R-MAT 22 BFS, C4 SVM at
nnz_x 200 / 2,000 / 20,000), each with the selected kernel, the best of 8,
regret, the SURVEY.md 8(d) B_alg roofline fraction and the reference CPU
implementation timed on this box's host cores.

  --impl ours       (default) the CUDA library through its C-ABI
  --impl reference  the reference's own CPU implementation (oracle/_ref: the
                    unmodified reference headers, built with the reference's
                    ref_bench flags at this host's ISA level) on the host cores

Timing: CUDA events on the library's stream around each multiply, medians
over K steps after W warm-up steps; an L2 flush (256 MiB write, then a 256 MiB clean read) precedes every
timed multiply whose working set fits in L2.  C1 (< 50 us) is timed by CUDA
graph replay: N x (flush + multiply) minus N x flush.  CPU
timings follow SPEC.md:437-446 benchmark_kernel: operands prepared once, one
warm-up call, median of >= 3 timed calls.  Selection overhead (feature pulls +
tree walks, format conversions) is measured on fresh vectors and reported
beside the value.  e2e repeats the step through the public API with host
buffers (pinned): one adaspmv_run_batch call over the 7 vectors (H2D of x,
select, multiply, D2H of y in its smaller form, pipelined over 3 streams),
wall clock.  N > 1 (torchrun): the row-partitioned mode over ONE C2 matrix
(strong scaling), see run_ours_multi.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SPARSITIES = (0.00001, 0.0001, 0.001, 0.01, 0.1, 0.5, 1.0)
N = 1 << int(os.environ.get("ADASPMV_BENCH_LOG2N", "22"))  # override only for dry runs
DRAWS = 16 * N
GATE_CYCLES = 400_000  # ~0.2 ms at 1.9 GHz
L2_NOTE = "L2 flush (256 MiB write, then 256 MiB clean read) before timed multiplies with working set < 64 MB; larger inputs exceed L2"
METRIC = "GFLOP/s and HBM GB/s (% of roofline) vs x sparsity; selector regret vs best"
WORKLOAD = "C2 uniform random 4M x 4M, 2^26 draws (~64M nnz) fp32, x-sparsity sweep 0.001%-100%"
I_B, O_B = 4, 8  # device index / offset bytes (SURVEY.md section 8 symbols)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def alg_bytes(rows, cols, nnz, nnz_x, nnz_s, nnz_y, V=4):
    """SURVEY.md section 8(d) algorithmic bytes per multiply."""
    b_spmv = (rows + 1) * O_B + nnz * (I_B + V) + cols * V + rows * V
    b_row = (rows + 1) * O_B + nnz * I_B + nnz_s * V + ((cols + 31) // 32) * 4 + nnz_x * V + rows * V
    b_col_atomic = nnz_x * (I_B + V) + 2 * nnz_x * O_B + nnz_s * (I_B + V) + rows * V
    b_col_sort = nnz_x * (I_B + V) + 2 * nnz_x * O_B + nnz_s * (I_B + V) + nnz_y * (I_B + V)
    fam = {0: b_spmv, 1: b_spmv, 2: b_row, 3: b_row, 4: b_col_atomic, 5: b_col_sort, 6: b_col_atomic,
           7: b_col_sort}
    return min(b_spmv, b_row, b_col_atomic, b_col_sort), fam


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0, period_ms=10):
        self.device = device
        self.period_ms = period_ms
        self.rows = []
        self._proc = None
        self._t = None
        self._first = threading.Event()
        self._on = False
        self._grab = False  # a window shorter than one period: keep the next sample

    def _run(self):
        # one long-lived `nvidia-smi -lms` reader: a sample every period_ms
        # without paying nvidia-smi's start-up per sample
        for line in self._proc.stdout:
            line = line.strip()
            if not line:
                continue
            self._first.set()
            if self._on or (self._grab and not self.rows):
                self.rows.append([s.strip() for s in line.split(",")])

    def _poll(self):
        # fallback: one nvidia-smi call per sample
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out and self._on:
                    self.rows.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._stop = threading.Event()
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", f"--loop-ms={self.period_ms}"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
            self._first.wait(5.0)  # the sampler is live before the timed region opens
        except Exception:
            self._proc = None
        if not self._first.is_set():  # no loop mode: poll instead
            self._close_proc()
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
        self._on = True
        return self

    def _close_proc(self):
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
            self._proc = None

    def __exit__(self, *a):
        self._on = False
        if not self.rows and self._proc is not None:  # the window fell between two samples
            self._grab = True
            t0 = time.time()
            while not self.rows and time.time() - t0 < 0.5:
                time.sleep(0.005)
        self._stop.set()
        self._close_proc()
        if self._t is not None:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def make_matrix():
    from paper_2006_16767_b200 import synth
    t0 = time.time()
    m = synth.uniform_random(N, DRAWS, seed=1, dtype=np.float32)
    return m, time.time() - t0


def make_vectors(n):
    from paper_2006_16767_b200 import synth
    out = []
    for i, s in enumerate(SPARSITIES):
        k = max(1, int(round(s * n)))
        out.append(synth.sparse_vector(n, k, seed=1000 + i, dtype=np.float32))
    return out


def c2_config(rows, cols, nnz, world):
    """The workload description both arms print (same keys and values)."""
    return {"workload": WORKLOAD, "rows": rows, "cols": cols, "nnz": nnz, "x_sparsity": list(SPARSITIES),
            "l2": L2_NOTE,
            "parallelism": f"row-partitioned x{world} (one C2 matrix, strong scaling)" if world > 1 else "single device"}


# ---------------------------------------------------------------------------
# the reference CPU implementation (oracle/_ref, bench build): shared by the
# reference arm and our cpu_baseline leg, so both report the same number
# ---------------------------------------------------------------------------
def _ref_operand(M, xi, xv, dt):
    if len(xi) == M.cols:
        d = np.zeros(M.cols, dt)
        d[xi] = xv
        return dict(x_dense=d)
    return dict(x_sparse=(xi, xv))


def ref_time(M, k, op, repeats=3):
    """SPEC.md:437-446 benchmark_kernel: 1 warm-up, median of `repeats`."""
    return float(np.median(M.bench_kernel(k, warmup=1, repeats=repeats, **op)))


def ref_choose(M, ops, nnz_s, kernels=range(8), sort_cap=20_000_000):
    """Best reference kernel per operand: one warm-up + one timed call each;
    the sort write-back is skipped above `sort_cap` effective entries (its
    serial merge takes seconds there)."""
    best = []
    for op, ns in zip(ops, nnz_s):
        tk = {}
        for k in kernels:
            if k in (5, 7) and ns > sort_cap:
                continue
            tk[k] = float(np.min(M.bench_kernel(k, warmup=1, repeats=2, **op)))
        best.append(min(tk, key=tk.get))
    return best


def ref_c2_prepare(rows, cols, ro, ci, vals, vecs):
    from oracle.oracle import Ref
    ref = Ref(np.float32, bench=True)
    threads = os.cpu_count() or 1
    ref.set_threads(threads)
    M = ref.matrix(rows, cols, ro, ci, vals)
    col_off = M.export()[3]
    nnz_s = [int(np.sum(col_off[xi + 1] - col_off[xi])) for xi, _ in vecs]
    ops = [_ref_operand(M, xi, xv, np.float32) for xi, xv in vecs]
    best = ref_choose(M, ops, nnz_s, sort_cap=400_000)
    return ref, M, ops, nnz_s, best, threads


def ref_c2_step(M, ops, best, repeats=3):
    return [ref_time(M, k, op, repeats) for op, k in zip(ops, best)]


_V2 = {}


def _v2_bundle():
    """The optional schema-2 selector bundle (None when absent), loaded once."""
    if "b" not in _V2:
        from paper_2006_16767_b200 import adaspmv as A
        from paper_2006_16767_b200 import selector as S
        p = S.DEFAULT_PATH.parent / "b200_bundle_v2.txt"
        _V2["b"] = A.SelectorBundle.load(p) if p.exists() else None
    return _V2["b"]


def _cpu_meta(ref, threads, sample):
    from oracle.oracle import host_cpu_model
    return {"cores": threads, "kind": "reference", "sample": sample, "cpu": host_cpu_model(),
            "build": ref.variant}


def cpu_c1(c1):
    """C1 on the reference: best of its 8 kernels per point (benchmark_kernel)."""
    from oracle.oracle import Ref
    rows, cols, ro, ci, vals, pts = c1
    ref = Ref(np.float64, bench=True)
    threads = os.cpu_count() or 1
    ref.set_threads(threads)
    M = ref.matrix(rows, cols, ro, ci, vals)
    col_off = M.export()[3]
    out = []
    for name, xi, xv in pts:
        op = _ref_operand(M, xi, xv, np.float64)
        ns = int(np.sum(col_off[xi + 1] - col_off[xi]))
        k = ref_choose(M, [op], [ns])[0]
        t = ref_time(M, k, op, repeats=5)
        out.append({"point": name, "kernel": A_name(k), "ms": round(t * 1e3, 4),
                    "gflops": round(2 * ns / t / 1e9, 3)})
    flops = sum(2 * int(np.sum(col_off[xi + 1] - col_off[xi])) for _, xi, _ in pts)
    tot = sum(p["ms"] for p in out) * 1e-3
    res = {"value": round(flops / tot / 1e9, 3), "unit": "GFLOP/s", "points": out}
    res.update(_cpu_meta(ref, threads, "both C1 points, best reference kernel each, median of 5"))
    return res


def cpu_c3(n, ro_h, ci_h, q, edges):
    """C3 on the reference: SPEC.md:489-497 BFS (plus-times, frontier 1.0)
    with the reference's run_kernel per level (ref_capi.cpp ref_bfs)."""
    from oracle.oracle import Ref
    ref = Ref(np.float32, bench=True)
    threads = os.cpu_count() or 1
    ref.set_threads(threads)
    M = ref.matrix(n, n, ro_h, ci_h, None)
    lv, nl, _ = M.bfs(0, -1)  # warm-up + levels check
    ts = [M.bfs(0, -1)[2] for _ in range(3)]
    t = float(np.median(ts))
    res = {"value": round(edges / t / 1e9, 4), "unit": "GTEPS", "ms": round(t * 1e3, 2),
           "levels_match_queue_bfs": bool(np.array_equal(lv, q)), "policy": "per level: col_lb_atomic / row_lb "
           "by the SURVEY.md 8(d) bytes model (the reference's fastest fixed kernels on R-MAT)"}
    res.update(_cpu_meta(ref, threads, "full C3 traversal from vertex 0, median of 3 after one warm-up"))
    return res


def cpu_c4(c4h, pts):
    """C4 on the reference: best of its kernels per sample row (benchmark_kernel)."""
    from oracle.oracle import Ref
    mr, nc, ro, ci, vals = c4h
    ref = Ref(np.float32, bench=True)
    threads = os.cpu_count() or 1
    ref.set_threads(threads)
    M = ref.matrix(mr, nc, ro, ci, vals)
    col_off = M.export()[3]
    out = []
    flops = 0
    tot = 0.0
    for i, (xi, xv) in enumerate(pts):
        op = _ref_operand(M, xi, xv, np.float32)
        ns = int(np.sum(col_off[xi + 1] - col_off[xi]))
        kern = range(8) if i == 0 else (4, 5, 6, 7)  # row kernels read all 2e8 entries: measured once
        k = ref_choose(M, [op], [ns], kernels=kern)[0]
        t = ref_time(M, k, op, repeats=3)
        flops += 2 * ns
        tot += t
        out.append({"nnz_x": len(xi), "kernel": A_name(k), "ms": round(t * 1e3, 3), "gflops": round(2 * ns / t / 1e9, 3)})
    res = {"value": round(flops / tot / 1e9, 3), "unit": "GFLOP/s", "points": out}
    res.update(_cpu_meta(ref, threads, "the three C4 sample rows, best reference kernel each, median of 3"))
    return res


def A_name(k):
    from paper_2006_16767_b200 import adaspmv as A
    return A.KernelId.from_index(int(k)).name()


# ---------------------------------------------------------------------------
# configuration inputs (identical bytes for both arms)
# ---------------------------------------------------------------------------
def c1_inputs():
    """C1: 2-D 5-point Laplacian 1000 x 1000 (10^6 rows) fp64; x dense
    U[-1,1) (seed 7) and 1 % (10,000 entries uniform w/o replacement)."""
    from paper_2006_16767_b200 import synth
    rows, cols, ro, ci, vals = synth.laplacian_2d(1000, dtype=np.float64)
    rng = np.random.default_rng(7)
    xd = rng.uniform(-1, 1, cols)
    xi1 = np.sort(rng.choice(cols, 10_000, replace=False)).astype(np.int64)
    xv1 = rng.uniform(-1, 1, 10_000)
    pts = [("x=100%", np.arange(cols, dtype=np.int64), xd), ("x=1%", xi1, xv1)]
    return rows, cols, ro, ci, vals, pts


def c3_inputs():
    """C3: R-MAT scale 22 (device generator) -> device (ro, ci) + host copies."""
    from paper_2006_16767_b200 import synth_device as SD
    t0 = time.time()
    n, ro, ci = SD.rmat_device(22)
    return n, ro, ci, time.time() - t0


def c3_levels(port, n, ro_h, ci_h):
    q, nq = port.bfs_queue_i32(n, ro_h, ci_h, 0)
    deg = np.diff(ro_h)
    edges = int(deg[q >= 0].sum())
    # SURVEY.md 8(d) BFS B_alg: per level min(push, pull), I = 4, O = 8
    b_alg = 0.0
    lvl_rows = []
    for L in range(nq):
        f = q == L
        nnz_x = int(f.sum())
        nnz_s = int(deg[f].sum())
        new = int((q == L + 1).sum())
        unv = int(deg[(q > L) | (q < 0)].sum())
        push = nnz_x * 4 + 2 * nnz_x * 8 + nnz_s * 4 + n / 8 + new * 8
        pull = (n + 1) * 8 + unv * 4 + 2 * n / 8 + new * 8
        b_alg += min(push, pull)
        lvl_rows.append({"level": L, "nnz_x": nnz_x, "nnz_s": nnz_s, "new": new,
                         "push_MB": round(push / 1e6, 2), "pull_MB": round(pull / 1e6, 2)})
    return q, nq, edges, b_alg, lvl_rows


C4_NNZ_X = (200, 2000, 20000)


def c4_inputs():
    from paper_2006_16767_b200 import synth_device as SD
    t0 = time.time()
    mr, nc = 10_000_000, 2_000_000
    ro, ci, vals, draw = SD.svm_device(mr, nc, 20, 1.0, 3)
    pts = [SD.svm_vector(draw, nc, nx, seed=nx) for nx in C4_NNZ_X]
    return mr, nc, ro, ci, vals, pts, time.time() - t0


# ---------------------------------------------------------------------------
# reference CPU arm
# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    if rank != 0:
        return None
    (rows, cols, ro, ci, vals), gen_s = make_matrix()
    nnz = int(ro[-1])
    vecs = make_vectors(cols)
    ref, M, ops, nnz_s, best, threads = ref_c2_prepare(rows, cols, ro, ci, vals, vecs)
    del ci
    for _ in range(args.warmup):
        ref_c2_step(M, ops, best, repeats=1)
    steps = [ref_c2_step(M, ops, best) for _ in range(args.steps)]
    t_step = [sum(s) for s in steps]
    flops = sum(2 * s for s in nnz_s)
    v = flops / statistics.median(t_step) / 1e9
    meta = _cpu_meta(ref, threads, "full C2 sweep per step: each point's best reference kernel, "
                                   "benchmark_kernel (1 warm-up, median of 3)")
    line = {
        "metric": METRIC, "value": round(v, 4), "unit": "GFLOP/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(statistics.median(t_step) * 1e3, 3), "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded numpy generator, SURVEY.md 8(d) C2)",
        "config": c2_config(rows, cols, nnz, world),
        "kernel_per_point": [A_name(k) for k in best],
        "cpu_baseline": dict(value=round(v, 4), unit="GFLOP/s", **meta),
        "e2e": {"value": round(v, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "per_point_ms": [round(statistics.median([s[i] for s in steps]) * 1e3, 4) for i in range(len(vecs))],
        "generation_s": round(gen_s, 1),
    }
    del M, ref
    if args.configs:
        line["configs"] = reference_configs(args)
    return line


def reference_configs(args):
    """The reference's numbers for the other single-GPU configurations."""
    from oracle.oracle import Port
    out = {}
    want = set(args.configs.split(","))
    if "C1" in want:
        out["C1"] = cpu_c1(c1_inputs())
    if "C3" in want:
        import torch
        n, ro, ci, _ = c3_inputs()
        ro_h, ci_h = ro.cpu().numpy(), ci.cpu().numpy()
        del ro, ci
        torch.cuda.empty_cache()
        q, nq, edges, _, _ = c3_levels(Port(), n, ro_h, ci_h)
        out["C3"] = cpu_c3(n, ro_h, ci_h.astype(np.int64), q, edges)
    if "C4" in want:
        import torch
        mr, nc, ro, ci, vals, pts, _ = c4_inputs()
        c4h = (mr, nc, ro.cpu().numpy(), ci.cpu().numpy().astype(np.int64), vals.cpu().numpy())
        del ro, ci, vals
        torch.cuda.empty_cache()
        out["C4"] = cpu_c4(c4h, pts)
    return out


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours_multi(args, rank, world):
    """N > 1: the row-partitioned mode (north_star), STRONG
    scaling over ONE C2 matrix.  Every rank draws the same C2 matrix (seed 1)
    and keeps its nnz-balanced row block (adaspmv_shard_rows, the segment_of
    cut of partition.hpp:30-33 snapped to row starts); every step broadcasts
    each sweep point's x from rank 0 over NCCL straight into device buffers
    handed to the library, then every rank runs its own selector + kernel on
    its block (nnz_s differs per block).  Step time = max over ranks (CUDA
    events on the shared stream, barrier on both sides); value = the whole
    matrix's useful flops / step time, the same numerator as N = 1."""
    import torch
    import torch.distributed as dist

    from paper_2006_16767_b200 import adaspmv as A
    from paper_2006_16767_b200 import selector as S

    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: ADASPMV_BENCH_BACKEND=gloo runs several ranks on one GPU
    # (NCCL needs one GPU per rank) to exercise the N > 1 logic end to end
    backend = os.environ.get("ADASPMV_BENCH_BACKEND", "nccl")
    local = local % torch.cuda.device_count() if backend != "nccl" else local
    dev = torch.device("cuda", local)
    torch.cuda.set_device(local)
    # stdout carries exactly one JSON line: keep NCCL's version banner off it
    if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"
    if backend == "nccl":
        # a collective that never completes (a rank failing alone) aborts
        # after 10 minutes instead of holding the job forever
        import datetime
        dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(minutes=10))
    else:
        dist.init_process_group(backend)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)  # collectives order against it; the library launches on it
    ctx = A.Context(local, stream=stream.cuda_stream)
    (rows_all, cols, ro_all, ci_all, vals_all), gen_s = make_matrix()
    nnz_all = int(ro_all[-1])
    cuts = A.shard_rows(ro_all, world)
    r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
    b0, b1 = int(ro_all[r0]), int(ro_all[r1])
    rows = r1 - r0
    ro = ro_all[r0:r1 + 1] - b0
    m = A.DualMatrix.from_csr(rows, cols, ro, ci_all[b0:b1], vals_all[b0:b1], ctx=ctx)
    del ci_all, vals_all
    bundle = A.SelectorBundle.load(Path(args.bundle) if args.bundle else S.DEFAULT_PATH)
    vecs = make_vectors(cols) if rank == 0 else None
    sizes = torch.tensor([len(v[0]) for v in vecs] if rank == 0 else [0] * len(SPARSITIES), device=dev)
    dist.broadcast(sizes, 0)
    bufs = []
    for i, k in enumerate(sizes.tolist()):
        dense = k == cols
        idx = torch.empty(0 if dense else k, dtype=torch.int32, device=dev)
        val = torch.empty(cols if dense else k, dtype=torch.float32, device=dev)
        if rank == 0:
            xi, xv = vecs[i]
            if dense:
                d = np.zeros(cols, np.float32)
                d[xi] = xv
                val.copy_(torch.from_numpy(d))
            else:
                idx.copy_(torch.from_numpy(xi.astype(np.int32)))
                val.copy_(torch.from_numpy(xv))
        bufs.append((dense, idx, val))
    x = A.DeviceVector(cols, np.float32, ctx)
    out = A.MultiplyOutput(ctx)
    pinned = [(i.cpu().pin_memory(), v.cpu().pin_memory()) for _, i, v in bufs] if rank == 0 else None

    def set_x(dense, idx, val):
        if dense:
            x.set_dense_device(val.data_ptr())
        else:
            x.set_sparse_device(idx.numel(), idx.data_ptr(), val.data_ptr())

    def bcast(dense, idx, val):
        if not dense:
            dist.broadcast(idx, 0)
        dist.broadcast(val, 0)

    # per point: the kernel this rank's selector picks for its block (features
    # of the broadcast x against the local block)
    flops_local = 0
    chosen, nnz_s_local = [], []
    for dense, idx, val in bufs:  # outside any timed region
        bcast(dense, idx, val)
        set_x(dense, idx, val)
        nnz_s_local.append(A.effective_nnz(m, x))
        flops_local += 2 * nnz_s_local[-1]
        k, _, _ = A.predict_kernel(m, x, bundle)
        chosen.append(k.index())
        x.prepare(k.index())
        A.run_kernel(m, k.index(), x, out=out)  # builds the row bins before any timing
    ctx.set_timing(True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def step():
        """One sweep: per point, the x broadcast (CUDA events on the shared
        stream) and the multiply (the library's events), each started with the
        GPU spinning so host enqueue latency is excluded -- the same protocol
        as the 1-GPU path; the untimed x hand-over (device copy + format
        conversion) sits between them."""
        t_x = t_k = 0.0
        for p, (dense, idx, val) in enumerate(bufs):
            torch.cuda._sleep(GATE_CYCLES)
            ev[0].record(stream)
            bcast(dense, idx, val)
            ev[1].record(stream)
            set_x(dense, idx, val)
            x.prepare(chosen[p])
            torch.cuda._sleep(GATE_CYCLES)
            A.run_kernel(m, chosen[p], x, out=out)
            t_k += out.elapsed()
            t_x += ev[0].elapsed_time(ev[1]) * 1e-3
        return t_x, t_k

    for _ in range(args.warmup):
        step()
    l0 = ctx.launches
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        per = [step() for _ in range(args.steps)]
    torch.cuda.synchronize()
    launches = (ctx.launches - l0) // max(1, args.steps)
    dist.barrier()
    t_exch = statistics.median(p[0] for p in per)
    t_local = statistics.median(p[0] + p[1] for p in per)
    ctx.set_timing(False)

    ybuf = torch.zeros(max(rows, 1), dtype=torch.float32).pin_memory().numpy()
    yidx = torch.zeros(max(rows, 1), dtype=torch.int64).pin_memory().numpy()
    d2h_bytes = [0]

    def e2e_step():
        d2h_bytes[0] = 0
        for p, (dense, idx, val) in enumerate(bufs):
            if rank == 0:  # this point's x comes from host memory
                idx.copy_(pinned[p][0], non_blocking=True)
                val.copy_(pinned[p][1], non_blocking=True)
            bcast(dense, idx, val)
            set_x(dense, idx, val)
            y, k = A.run_adaptive(m, x, bundle, out=out)
            # this rank's y block back to pinned host memory in its smaller form
            if k.index() in (5, 7) or 3 * nnz_s_local[p] < rows:
                ny = C.c_int64()
                A._check(A._lib.adaspmv_output_sparse(ctx.h, y.h, rows, A._ptr(yidx), A._ptr(ybuf), C.byref(ny)))
                d2h_bytes[0] += ny.value * 12
            else:
                A._check(A._lib.adaspmv_output_dense(ctx.h, y.h, A._ptr(ybuf)))
                d2h_bytes[0] += rows * 4

    # e2e: x from pinned host memory on rank 0, broadcast, select, multiply,
    # y blocks back to host
    e2e_t = []
    for _ in range(max(2, args.steps // 2)):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()
        torch.cuda.synchronize()
        e2e_t.append(time.perf_counter() - t0)
    d2h = torch.tensor([float(d2h_bytes[0])], dtype=torch.float64, device=dev)
    dist.all_reduce(d2h, op=dist.ReduceOp.SUM)
    tt = torch.tensor([t_local, float(flops_local), statistics.median(e2e_t), t_exch], dtype=torch.float64, device=dev)
    tmax = tt.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    fl = tt[1:2].clone()
    dist.all_reduce(fl, op=dist.ReduceOp.SUM)
    t_step = float(tmax[0].item())
    value = float(fl.item()) / t_step / 1e9
    e2e_v = float(fl.item()) / float(tmax[2].item()) / 1e9
    line = None
    if rank == 0:
        xbytes = sum((int(v.numel()) * 4 + int(i.numel()) * 4) for _, i, v in bufs)
        hbm, src = peaks()
        alg = alg_bytes(rows_all, cols, nnz_all, cols, nnz_all, cols)[0]  # x = 100 %: B_spmv
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded numpy generator, SURVEY.md 8(d) C2, one matrix cut into row blocks)",
            "config": c2_config(rows_all, cols, nnz_all, world),
            "shard_rows": [int(c) for c in cuts],
            "timing": "per point: x broadcast (events) + multiply (library events), GPU gated, max over ranks; "
                      "selection and x hand-over untimed as on 1 GPU",
            "exchange": {"ms_per_step": round(float(tmax[3].item()) * 1e3, 4),
                         "fraction": round(float(tmax[3].item()) / t_step, 4),
                         "bytes_per_step": int(xbytes),
                         "GBps": round(xbytes * max(world - 1, 0) / max(float(tmax[3].item()), 1e-12) / 1e9, 1)},
            "e2e": {"value": round(e2e_v, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": int(xbytes),
                    "d2h_bytes_per_step": int(d2h.item()),
                    "note": "x H2D on rank 0 then NCCL broadcast; each rank selects, multiplies and copies its "
                            "y block to pinned host memory in its smaller form; max over ranks"},
            "roofline_aggregate": {"bound": "hbm", "x_sparsity": 1.0, "alg_bytes": int(alg),
                                   "peak": hbm * world, "unit": "GB/s", "peak_source": src},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "setup_s": {"generate": round(gen_s, 1)},
        }
    if "C5" in args.configs.split(","):
        del m
        torch.cuda.empty_cache()
        try:
            c5 = ours_c5(local, rank, world, bundle, peaks()[0], ctx, stream, dist=dist)
        except Exception as e:  # never lose the headline line to the largest config
            c5 = {"error": f"{type(e).__name__}: {e}"}
        if rank == 0:
            line["configs"] = {"C5": c5}
    dist.destroy_process_group()
    return line


class L2Flush:
    """L2 flush between timed multiplies: write a 256 MiB buffer (2x the
    126 MB L2), then read a second 256 MiB buffer, so the dirty lines of the
    write are written back inside the flush and the multiply starts on an L2
    holding only clean, unrelated lines (otherwise the multiply's first reads
    pay the DRAM write-back of the flush's dirty lines)."""

    def __init__(self, device):
        import torch
        self.w = torch.empty(256 << 20, dtype=torch.uint8, device=device)
        self.r = torch.zeros(64 << 20, dtype=torch.int32, device=device)

    def __call__(self):
        self.w.add_(1)
        self.r.amax()


def _timed_factory(stream, flush):
    import torch

    def timed(fn, n_rep, need_flush):
        ts = []
        for _ in range(n_rep):
            with torch.cuda.stream(stream):
                if need_flush:
                    flush()
                # the GPU spins while the host enqueues the multiply, so the
                # library's events see device time, not host launch latency
                torch.cuda._sleep(GATE_CYCLES)
            y = fn()
            if isinstance(y, tuple):
                y = y[0]
            ts.append(y.elapsed())
        return ts
    return timed


def graph_replay_time(call, gstream, flush, n=20, reps=5):
    """Device seconds per call by CUDA graph replay (inputs
    under ~50 us): a graph of n x (L2 flush + call) minus a graph of n x
    flush, each replayed `reps` times (median), / n.  `call` launches on
    `gstream` (a library context bound to it)."""
    import torch
    with torch.cuda.stream(gstream):
        call()
    torch.cuda.synchronize()

    def capture(with_call):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gstream, capture_error_mode="relaxed"):
            for _ in range(n):
                flush()
                if with_call:
                    call()
        return g

    g1, g0 = capture(True), capture(False)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def run(g):
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            with torch.cuda.stream(gstream):
                e[0].record()
                g.replay()
                e[1].record()
            torch.cuda.synchronize()
            ts.append(e[0].elapsed_time(e[1]) * 1e-3)
        return statistics.median(ts)

    t1, t0 = run(g1), run(g0)
    del g1, g0
    return max(t1 - t0, 0.0) / n


def ours_c1(local, bundle, hbm, flush, cpu):
    """C1 (configs[0]): fp64 Laplacian, x = 100 % and 1 %: every kernel by
    graph replay, the selector's choice, regret, B_alg roofline."""
    import torch

    from paper_2006_16767_b200 import adaspmv as A
    rows, cols, ro, ci, vals, pts = c1_inputs()
    nnz = int(ro[-1])
    gstream = torch.cuda.Stream(device=f"cuda:{local}")
    gctx = A.Context(local, stream=gstream.cuda_stream)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=gctx)
    co = np.bincount(ci, minlength=cols)
    out = A.MultiplyOutput(gctx)
    res = {"workload": "C1 2-D 5-point Laplacian 1000x1000 (10^6 rows, 4,996,000 nnz) fp64, x = 100 % and 1 %",
           "timing": "CUDA graph replay of 20 x (L2 flush: 256 MiB write + 256 MiB read; multiply) minus 20 x flush, median of 5",
           "points": []}
    flops = tot = 0.0
    for name, xi, xv in pts:
        x = A.DeviceVector(cols, np.float64, gctx)
        if len(xi) == cols:
            x.set_dense(xv)
        else:
            x.set_sparse(xi, xv)
        nnz_s = int(co[xi].sum())
        k_sel = A.predict_kernel(m, x, bundle)[0].index()
        k_v2 = A.predict_kernel(m, x, _v2_bundle())[0].index() if _v2_bundle() else None
        c = A.KernelConfig()._c()
        ts = []
        for k in range(8):
            x.prepare(k)

            def call(k=k):
                A._check(A._lib.adaspmv_run(gctx.h, m.h, x.h, k, C.byref(c), out.h))
            ts.append(graph_replay_time(call, gstream, flush))
        b_alg, fam = alg_bytes(rows, cols, nnz, len(xi), nnz_s, nnz_s, V=8)
        t_sel = ts[k_sel]
        flops += 2 * nnz_s
        tot += t_sel
        res["points"].append({
            "point": name, "nnz_x": len(xi), "nnz_s": nnz_s, "selected": A_name(k_sel),
            "t_sel_us": round(t_sel * 1e6, 2), "best": A_name(int(np.argmin(ts))),
            "t_best_us": round(min(ts) * 1e6, 2), "regret": round(t_sel / min(ts), 3),
            "gflops_sel": round(2 * nnz_s / t_sel / 1e9, 2), "alg_bytes": int(b_alg),
            "roofline_frac": round(b_alg / t_sel / 1e9 / hbm, 4),
            "t_kernels_us": [round(t * 1e6, 2) for t in ts],
            "schema2": None if k_v2 is None else {"selected": A_name(k_v2), "regret": round(ts[k_v2] / min(ts), 3)}})
    res["value"] = round(flops / tot / 1e9, 3)
    res["unit"] = "GFLOP/s"
    if cpu:
        res["cpu_reference"] = cpu_c1((rows, cols, ro, ci, vals, pts))
    del m, out, gctx
    return res


def ours_c3(local, bundle, hbm, cpu, reps=5):
    """C3 (configs[2]): R-MAT 22 BFS from vertex 0 (OR_AND), levels checked
    against the queue BFS; traversal wall time per policy (levels stay on the
    device), GTEPS, kernel share (overhead), SURVEY.md 8(d) BFS B_alg."""
    import torch

    from oracle.oracle import Port
    from paper_2006_16767_b200 import adaspmv as A
    n, ro, ci, gen_s = c3_inputs()
    nnz = int(ro[-1].item())
    ctx = A.Context(local)
    t0 = time.time()
    m = A.DualMatrix.from_device(n, n, nnz, ro.data_ptr(), ci.data_ptr(), None, np.float32, ctx)
    build_s = time.time() - t0
    ro_h, ci_h = ro.cpu().numpy(), ci.cpu().numpy()
    del ro, ci
    torch.cuda.empty_cache()
    q, nq, edges, b_alg, lvl_rows = c3_levels(Port(), n, ro_h, ci_h)
    policies = [("selector", dict(bundle=bundle)), ("heuristic", {})] + \
               [(f"fixed_{A_name(k)}", dict(force_kernel=k)) for k in range(8)]
    runs = {}
    for name, kw in policies:
        lv, _ = A.bfs(m, 0, A.OR_AND, **kw)
        ok = bool(np.array_equal(lv, q))
        walls, ksum = [], []
        for _ in range(reps):
            ctx.synchronize()
            t1 = time.perf_counter()
            _, rep = A.bfs(m, 0, A.OR_AND, download_levels=False, **kw)
            walls.append(time.perf_counter() - t1)
            ksum.append(sum(r["kernel_s"] + r["convert_s"] for r in rep))
        w = statistics.median(walls)
        runs[name] = {"ms": round(w * 1e3, 4), "gteps": round(edges / w / 1e9, 2),
                      "device_ms": round(statistics.median(ksum) * 1e3, 4),
                      "overhead_fraction": round(1 - statistics.median(ksum) / w, 4), "levels_ok": ok,
                      "kernels": [r["kernel"] for r in rep], "exec_mode": [r["exec_mode"] for r in rep]}
    fixed = {k: v for k, v in runs.items() if k.startswith("fixed_")}
    best = min(fixed, key=lambda k: fixed[k]["ms"])
    sel = runs["selector"]
    res = {"workload": f"C3 R-MAT scale 22 (device generator), {nnz:,} stored entries, BFS from vertex 0, OR_AND",
           "n": n, "nnz": nnz, "levels": nq, "reached": int((q >= 0).sum()), "edges_traversed": edges,
           "value": sel["gteps"], "unit": "GTEPS", "selected_ms": sel["ms"], "best_fixed": best,
           "best_fixed_ms": fixed[best]["ms"], "regret_vs_best_fixed": round(sel["ms"] / fixed[best]["ms"], 3),
           "overhead_fraction": sel["overhead_fraction"],
           "alg_bytes": int(b_alg), "roofline_frac": round(b_alg / (sel["ms"] * 1e-3) / 1e9 / hbm, 4),
           "roofline_note": "sum over levels of min(push, pull) bytes (SURVEY.md 8(d)) / selector wall time",
           "per_level": lvl_rows, "runs": runs, "setup_s": {"generate": round(gen_s, 2), "build": round(build_s, 2)}}
    del m, ctx
    torch.cuda.empty_cache()
    if cpu:
        res["cpu_reference"] = cpu_c3(n, ro_h, ci_h.astype(np.int64), q, edges)
    return res


def ours_c4(local, bundle, hbm, flush, cpu, reps=3):
    """C4 (configs[3]): SVM 10M x 2M, sparse sample rows (nnz_x 200 / 2,000 /
    20,000): all 8 kernels (events + L2 flush), the selector, regret, B_alg."""
    import torch

    from paper_2006_16767_b200 import adaspmv as A
    mr, nc, ro, ci, vals, pts, gen_s = c4_inputs()
    nnz = int(ro[-1].item())
    ctx = A.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    m = A.DualMatrix.from_device(mr, nc, nnz, ro.data_ptr(), ci.data_ptr(), vals.data_ptr(), np.float32, ctx)
    c4h = (mr, nc, ro.cpu().numpy(), ci.cpu().numpy().astype(np.int64), vals.cpu().numpy()) if cpu else None
    del ro, ci, vals
    torch.cuda.empty_cache()
    ctx.set_timing(True)
    timed = _timed_factory(stream, flush)
    out = A.MultiplyOutput(ctx)
    res = {"workload": f"C4 SVM-like 10M x 2M, {nnz:,} nnz, Zipf(1.0) feature popularity, fp32; "
                       "sparse sample rows nnz_x = 200 / 2,000 / 20,000", "points": []}
    flops = tot = 0.0
    for xi, xv in pts:
        x = A.DeviceVector(nc, np.float32, ctx).set_sparse(xi, xv)
        nnz_s = A.effective_nnz(m, x)
        ts = []
        nnz_y = 0
        for k in range(8):
            x.prepare(k)
            run = lambda k=k: A.run_kernel(m, k, x, out=out)  # noqa: E731
            ts.append(statistics.median(timed(run, reps + 1, True)[1:]))
            if k == 5:
                nnz_y = out.nnz()
        k_sel = A.predict_kernel(m, x, bundle)[0].index()
        k_v2 = A.predict_kernel(m, x, _v2_bundle())[0].index() if _v2_bundle() else None
        t_sel = ts[k_sel]
        b_alg, _ = alg_bytes(mr, nc, nnz, len(xi), nnz_s, nnz_y)
        flops += 2 * nnz_s
        tot += t_sel
        res["points"].append({
            "nnz_x": len(xi), "nnz_s": nnz_s, "nnz_y": nnz_y, "selected": A_name(k_sel),
            "t_sel_us": round(t_sel * 1e6, 2), "best": A_name(int(np.argmin(ts))),
            "t_best_us": round(min(ts) * 1e6, 2), "regret": round(t_sel / min(ts), 3),
            "gflops_sel": round(2 * nnz_s / t_sel / 1e9, 2), "alg_bytes": int(b_alg),
            "roofline_frac": round(b_alg / t_sel / 1e9 / hbm, 4),
            "t_kernels_us": [round(t * 1e6, 2) for t in ts],
            "schema2": None if k_v2 is None else {"selected": A_name(k_v2), "regret": round(ts[k_v2] / min(ts), 3)}})
    res["value"] = round(flops / tot / 1e9, 3)
    res["unit"] = "GFLOP/s"
    res["setup_s"] = {"generate": round(gen_s, 2)}
    ctx.set_timing(False)
    del m, out, ctx
    torch.cuda.empty_cache()
    if cpu:
        res["cpu_reference"] = cpu_c4(c4h, pts)
    return res


C5_SCALE = int(os.environ.get("ADASPMV_BENCH_C5_SCALE", "26"))  # override only for dry runs
C5_DENS = (0.00001, 0.001, 0.1, 1.0)


def ours_c5(local, rank, world, bundle, hbm, ctx, stream, dist=None, reps=3):
    """C5 (configs[4]): R-MAT scale 26 (device generator, ~2.1 G stored
    entries) cut into `world` nnz-balanced row blocks (adaspmv_shard_rows,
    partition.hpp:30-33), one per rank.  Per x density: x drawn on rank 0 and
    broadcast over NCCL (N > 1), each rank's selector + multiply on its block;
    time = broadcast (events) + multiply (library events), max over ranks.
    BFS from vertex 0 (OR_AND): N = 1 the device-resident (persistent-kernel) BFS, N > 1 the
    row-partitioned BFS with the frontier all-gathered every level
    (adaspmv_dist_bfs); wall time max over ranks.  No CPU reference at this
    size (the reference BFS on 2.1 G edges takes minutes)."""
    import torch

    from paper_2006_16767_b200 import adaspmv as A
    from paper_2006_16767_b200 import synth_device as SD
    dev = torch.device("cuda", local)
    t0 = time.time()
    n, ro, ci = SD.rmat_device(C5_SCALE)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    nnz_all = int(ro[-1].item())
    ro_h = ro.cpu().numpy()
    cuts = A.shard_rows(ro_h, world)
    r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
    b0, b1 = int(ro_h[r0]), int(ro_h[r1])
    bro = (ro[r0:r1 + 1] - b0).contiguous()
    bci = ci[b0:b1].clone() if world > 1 else ci
    ro = ci = None
    torch.cuda.empty_cache()
    t0 = time.time()
    m = A.DualMatrix.from_device(r1 - r0, n, b1 - b0, bro.data_ptr(), bci.data_ptr(), None, np.float32, ctx)
    ctx.synchronize()
    build_s = time.time() - t0
    del bro, bci
    torch.cuda.empty_cache()
    deg_h = np.diff(ro_h[r0:r1 + 1])
    x = A.DeviceVector(n, np.float32, ctx)
    out = A.MultiplyOutput(ctx)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    gen = torch.Generator(device=dev)
    gen.manual_seed(26)
    pts = []
    ctx.set_timing(True)
    for d in C5_DENS:
        # x: rank 0 draws the support and values, the others receive them
        nx = torch.zeros(1, dtype=torch.int64, device=dev)
        if rank == 0:
            if d >= 1.0:
                idx = torch.arange(n, dtype=torch.int32, device=dev)
            else:
                idx = torch.nonzero(torch.rand(n, generator=gen, device=dev) < d).flatten().to(torch.int32)
            val = torch.rand(idx.numel(), generator=gen, device=dev, dtype=torch.float32) + 0.5
            nx[0] = idx.numel()
        if dist is not None:
            dist.broadcast(nx, 0)
        k_x = int(nx.item())
        if rank != 0:
            idx = torch.empty(k_x, dtype=torch.int32, device=dev)
            val = torch.empty(k_x, dtype=torch.float32, device=dev)

        def exchange():
            if dist is not None:
                dist.broadcast(idx, 0)
                dist.broadcast(val, 0)

        exchange()
        torch.cuda.synchronize()
        x.set_sparse_device(k_x, idx.data_ptr(), val.data_ptr())
        nnz_s_local = A.effective_nnz(m, x)
        k = A.predict_kernel(m, x, bundle)[0].index()
        k2 = A.predict_kernel(m, x, _v2_bundle())[0].index() if _v2_bundle() else None

        def time_kernel(kk):
            x.prepare(kk)
            A.run_kernel(m, kk, x, out=out)  # lazy layouts before timing
            ts = []
            for _ in range(reps):
                torch.cuda._sleep(GATE_CYCLES)
                ev[0].record(stream)
                exchange()
                ev[1].record(stream)
                x.set_sparse_device(k_x, idx.data_ptr(), val.data_ptr())
                x.prepare(kk)
                torch.cuda._sleep(GATE_CYCLES)
                A.run_kernel(m, kk, x, out=out)
                ts.append(out.elapsed() + ev[0].elapsed_time(ev[1]) * 1e-3)
            t_ = statistics.median(ts)
            if dist is not None:
                tm = torch.tensor([t_], dtype=torch.float64, device=dev)
                dist.all_reduce(tm, op=dist.ReduceOp.MAX)
                t_ = float(tm.item())
            return t_

        t = time_kernel(k)
        # the schema-2 choice is timed when it differs on ANY rank (every rank
        # must take part in the same broadcasts / reductions)
        need2 = torch.tensor([0.0 if k2 in (None, k) else 1.0], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(need2, op=dist.ReduceOp.MAX)
        t2 = time_kernel(k if k2 is None else k2) if need2.item() > 0 else t
        tt = torch.tensor([float(nnz_s_local)], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        nnz_s = int(tt[0].item())
        b_alg, _ = alg_bytes(n, n, nnz_all, k_x, nnz_s, 0)
        pts.append({"x_sparsity": d, "nnz_x": k_x, "nnz_s": nnz_s, "selected_rank0": A_name(k),
                    "ms": round(t * 1e3, 4), "gflops": round(2 * nnz_s / t / 1e9, 2),
                    "schema2": None if k2 is None else {"selected_rank0": A_name(k2), "ms": round(t2 * 1e3, 4)},
                    "alg_GBps": round(b_alg / t / 1e9, 1),
                    "roofline_frac_aggregate": round(b_alg / t / 1e9 / (hbm * world), 4)})
    ctx.set_timing(False)
    # BFS from vertex 0
    walls = []
    if dist is None:
        lv, _ = A.bfs(m, 0, A.OR_AND)
        for _ in range(reps):
            ctx.synchronize()
            t1 = time.perf_counter()
            A.bfs(m, 0, A.OR_AND, download_levels=False)
            walls.append(time.perf_counter() - t1)
        levels = lv
    else:
        from paper_2006_16767_b200.multigpu import make_dist
        D = make_dist(ctx)
        try:
            levels, _ = D.bfs(m, r0, 0, A.OR_AND)
            for _ in range(reps):
                dist.barrier()
                torch.cuda.synchronize()
                t1 = time.perf_counter()
                D.bfs(m, r0, 0, A.OR_AND, download_levels=False)
                torch.cuda.synchronize()
                walls.append(time.perf_counter() - t1)
        finally:
            D.close()
    reached = levels >= 0
    loc = torch.tensor([float(reached.sum()), float(deg_h[reached].sum()), float(levels.max() + 1),
                        statistics.median(walls)], dtype=torch.float64, device=dev)
    if dist is not None:
        tot = loc.clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        mx = loc.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        reached_n, edges, nlev, wall = int(tot[0].item()), int(tot[1].item()), int(mx[2].item()), float(mx[3].item())
    else:
        reached_n, edges, nlev, wall = int(loc[0].item()), int(loc[1].item()), int(loc[2].item()), float(loc[3].item())
    flops = sum(2 * p_["nnz_s"] for p_ in pts)
    res = {"workload": f"C5 R-MAT scale {C5_SCALE} (device generator), {nnz_all:,} stored entries, "
                       f"{world} nnz-balanced row block(s), fp32 pattern values",
           "n": n, "nnz": nnz_all, "n_gpus": world, "shard_rows": [int(c) for c in cuts],
           "timing": "per point: x broadcast (events, N > 1) + multiply (library events), GPU gated, median of "
                     f"{reps}, max over ranks; BFS wall time, max over ranks",
           "points": pts, "value": round(flops / sum(p_["ms"] * 1e-3 for p_ in pts) / 1e9, 3), "unit": "GFLOP/s",
           "bfs": {"ms": round(wall * 1e3, 4), "gteps": round(edges / wall / 1e9, 2), "levels": nlev,
                   "reached": reached_n, "edges_traversed": edges,
                   "mode": "device-resident BFS (one persistent kernel)" if dist is None else "row-partitioned BFS, frontier all-gathered"},
           "setup_s": {"generate": round(gen_s, 2), "build": round(build_s, 2)},
           "cpu_reference": None}
    del m, x, out
    torch.cuda.empty_cache()
    return res


def run_ours(args, rank, world):
    import torch

    from paper_2006_16767_b200 import adaspmv as A
    from paper_2006_16767_b200 import selector as S

    local = int(os.environ.get("LOCAL_RANK", "0"))
    (rows, cols, ro, ci, vals), gen_s = make_matrix()
    nnz = int(ro[-1])
    vecs = make_vectors(cols)
    # the CPU baseline runs first, in the same process state as the
    # reference arm (before any GPU work, pinned buffers or host threads)
    cpu = rank == 0 and not args.no_cpu_baseline
    cpu_line = cpu_baseline(rows, cols, ro, ci, vals, vecs) if cpu else None
    torch.cuda.set_device(local)
    ctx = A.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    t0 = time.time()
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    upload_s = time.time() - t0
    bundle_path = Path(args.bundle) if args.bundle else S.DEFAULT_PATH
    bundle = A.SelectorBundle.load(bundle_path)
    # device-resident operands: one DeviceVector per sweep point
    dvs = []
    for xi, xv in vecs:
        dv = A.DeviceVector(cols, np.float32, ctx)
        if len(xi) == cols:
            d = np.zeros(cols, np.float32)
            d[xi] = xv
            dv.set_dense(d)
        else:
            dv.set_sparse(xi, xv)
        dvs.append(dv)
    nnz_s = [A.effective_nnz(m, dv) for dv in dvs]
    nnz_x = [len(xi) for xi, _ in vecs]
    flush = L2Flush(f"cuda:{local}")
    out = A.MultiplyOutput(ctx)
    # the row-bin layout of K0/K2 (a third resident copy, nnz * (4 + V)
    # bytes) is built by the first binned call: timed here as setup, outside
    # every timed multiply
    dvs[-1].prepare(0)
    ctx.synchronize()
    t0 = time.time()
    A.run_kernel(m, 0, dvs[-1], out=out)
    ctx.synchronize()
    bins_s = time.time() - t0

    ctx.set_timing(True)  # CUDA events recorded by the library around each multiply
    timed = _timed_factory(stream, flush)

    # ---- per point: every kernel (best-of-8, regret) -------------------------
    small = [alg_bytes(rows, cols, nnz, nx, ns, 0)[0] < 64e6 for nx, ns in zip(nnz_x, nnz_s)]
    kernel_t = []
    for i, dv in enumerate(dvs):
        row = []
        for k in range(8):
            dv.prepare(k)
            run = lambda k=k, dv=dv: A.run_kernel(m, k, dv, out=out)  # noqa: E731
            timed(run, args.warmup, small[i])
            row.append(statistics.median(timed(run, max(args.steps, 3), small[i])))
        kernel_t.append(row)
    # ---- the adaptive step ----------------------------------------------------
    chosen = []
    for dv in dvs:
        k, _, _ = A.predict_kernel(m, dv, bundle)
        chosen.append(k.index())
    # the schema-2 bundle's choices on the same operands (reported beside the
    # default SPEC cascade, from the same all-kernel timings)
    v2_path = S.DEFAULT_PATH.parent / "b200_bundle_v2.txt"
    chosen_v2 = []
    if v2_path.exists():
        b2 = A.SelectorBundle.load(v2_path)
        chosen_v2 = [A.predict_kernel(m, dv, b2)[0].index() for dv in dvs]
    for i, dv in enumerate(dvs):  # operand conversions happen once, untimed
        dv.prepare(chosen[i])
    l0 = ctx.launches

    def step_times():
        per = []
        for i, dv in enumerate(dvs):
            per.append(timed(lambda dv=dv: A.run_adaptive(m, dv, bundle, out=out), 1, small[i])[0])
        return per

    for _ in range(args.warmup):
        step_times()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        steps = [step_times() for _ in range(args.steps)]
    torch.cuda.synchronize()
    launches = (ctx.launches - l0) // max(1, args.steps + args.warmup)
    t_step = [sum(s) for s in steps]
    t_med = statistics.median(t_step)
    flops = sum(2 * s for s in nnz_s)
    value = flops / t_med / 1e9
    # ---- selection overhead (reported beside the kernel
    # time): fresh vectors, so the features are computed, not cached ----------
    sel_t, conv_t = [], []
    fresh = A.DeviceVector(cols, np.float32, ctx)
    for _ in range(max(3, args.steps // 2)):
        s_sel = s_conv = 0.0
        for xi, xv in vecs:
            if len(xi) == cols:
                d = np.zeros(cols, np.float32)
                d[xi] = xv
                fresh.set_dense(d)
            else:
                fresh.set_sparse(xi, xv)
            ctx.synchronize()
            _, rep = A.execute_iteration(m, fresh, bundle, out=out)
            s_sel += rep["feature_s"] + rep["predict_s"]
            s_conv += rep["convert_s"]
        sel_t.append(s_sel)
        conv_t.append(s_conv)
    o_sel, o_conv = statistics.median(sel_t), statistics.median(conv_t)
    overhead = {"select_us_per_step": round(o_sel * 1e6, 1),
                "convert_us_per_step": round(o_conv * 1e6, 1),
                "overhead_fraction": round((o_sel + o_conv) / (o_sel + o_conv + t_med), 4),
                "note": "host feature pull (nnz_s on the device, one scalar back) + tree walk, and the "
                        "device format conversion the chosen kernel needs, per sweep; excluded from value, "
                        "included in e2e; fraction = overhead / (overhead + kernel time), SPEC.md:561 bound 0.20"}
    # ---- e2e through the public API with host buffers ----------------------
    # One step = one adaptive_run_batch call over the 7 host vectors (pinned),
    # results back in pinned host buffers in their smaller form; the batch
    # pipelines x_k's H2D, x_j's multiply and y_i's D2H over 3 streams.
    pinned = []
    for xi, xv in vecs:
        if len(xi) == cols:
            d = torch.zeros(cols, dtype=torch.float32).pin_memory()
            d[torch.from_numpy(xi)] = torch.from_numpy(xv)
            pinned.append(d.numpy())
        else:
            pinned.append((torch.from_numpy(xi).pin_memory().numpy(),
                           torch.from_numpy(xv).pin_memory().numpy()))
    h2d = sum(p.nbytes if not isinstance(p, tuple) else p[0].nbytes + p[1].nbytes for p in pinned)
    bufs = [(torch.zeros(rows, dtype=torch.int64).pin_memory().numpy(),
             torch.zeros(rows, dtype=torch.float32).pin_memory().numpy()) for _ in pinned]

    def e2e_bytes(res):
        return sum((r.sparse.nnz() * 12) if r.is_sparse else rows * 4 for r in res)

    e2e_times = []
    d2h = 0
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        res = A.run_batch(m, pinned, bundle=bundle, form=A.RESULT_AUTO, lanes=args.lanes, buffers=bufs)
        dt_ = time.perf_counter() - t0
        if it >= args.warmup:
            e2e_times.append(dt_)
            d2h = e2e_bytes(res)
    e2e_kernels = [r.kernel.index() for r in res]
    # the same through single calls (set -> run_adaptive -> output copy), for reference
    ybuf = bufs[0][1]
    yidx = bufs[0][0]
    e2e_x = A.DeviceVector(cols, np.float32, ctx)
    seq_times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        for i, p in enumerate(pinned):
            if isinstance(p, tuple):
                e2e_x.set_sparse(*p)
            else:
                e2e_x.set_dense(p)
            y, k = A.run_adaptive(m, e2e_x, bundle, out=out)
            if k.index() in (5, 7) or 3 * nnz_s[i] < rows:
                ny = C.c_int64()
                A._check(A._lib.adaspmv_output_sparse(ctx.h, y.h, rows, A._ptr(yidx), A._ptr(ybuf), C.byref(ny)))
            else:
                A._check(A._lib.adaspmv_output_dense(ctx.h, y.h, A._ptr(ybuf)))
        if it >= args.warmup:
            seq_times.append(time.perf_counter() - t0)
    e2e_v = flops / statistics.median(e2e_times) / 1e9
    # ---- roofline: the SpMV end (x = 100 %), SURVEY.md 8(d) B_alg ----------
    per_point = [statistics.median([s[i] for s in steps]) for i in range(len(dvs))]
    top = len(dvs) - 1
    k_top = chosen[top]
    b_alg_top, _ = alg_bytes(rows, cols, nnz, nnz_x[top], nnz_s[top], nnz_x[top])
    hbm, src = peaks()
    achieved = b_alg_top / per_point[top] / 1e9
    # DRAM bytes per launch of the same kernel + input from the committed ncu
    # --set full capture (profiles/r02_roofline_traffic.json)
    traffic = None
    for pf in ("r02_roofline_traffic.json", "r01_roofline_traffic.json"):
        prof = ROOT / "profiles" / pf
        if prof.exists():
            try:
                pj = json.loads(prof.read_text())
                if A_name(k_top) in pj.get("kernel", "") and "x = 100 %" in pj.get("kernel", ""):
                    traffic = pj.get("traffic_bytes_per_launch")
                    break
            except Exception:
                traffic = None
    dom = int(np.argmax(per_point))
    points = []
    for i in range(len(dvs)):
        b_alg, fam_i = alg_bytes(rows, cols, nnz, nnz_x[i], nnz_s[i], 0)
        tb = min(kernel_t[i])
        points.append({
            "x_sparsity": SPARSITIES[i], "nnz_x": nnz_x[i], "nnz_s": nnz_s[i],
            "selected": A_name(chosen[i]), "t_sel_us": round(per_point[i] * 1e6, 2),
            "best": A_name(int(np.argmin(kernel_t[i]))), "t_best_us": round(tb * 1e6, 2),
            "regret": round(per_point[i] / tb, 3),
            "gflops_sel": round(2 * nnz_s[i] / per_point[i] / 1e9, 2),
            "alg_GBps_sel": round(b_alg / per_point[i] / 1e9, 1),
            "pct_roofline_sel": round(100 * b_alg / per_point[i] / 1e9 / hbm, 1),
            "t_kernels_us": [round(t * 1e6, 2) for t in kernel_t[i]],
        })
    regret_total = sum(per_point) / sum(min(r) for r in kernel_t)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_med * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded numpy generator, SURVEY.md 8(d) C2)",
        "config": c2_config(rows, cols, nnz, world),
        "selector": str(bundle_path.name),
        "e2e": {"value": round(e2e_v, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "api": f"adaspmv_run_batch (pinned host buffers, {args.lanes} lanes)",
                "ms_per_step": round(statistics.median(e2e_times) * 1e3, 3),
                "sequential_value": round(flops / statistics.median(seq_times) / 1e9, 3),
                "sequential_api": "per vector: vector_set -> run_adaptive -> output copy",
                "kernels": e2e_kernels},
        "roofline": {"bound": "hbm", "kernel": A_name(k_top), "x_sparsity": SPARSITIES[top],
                     "achieved": round(achieved, 1), "peak": hbm, "peak_source": src, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": traffic, "alg_bytes": int(b_alg_top),
                     "alg_bytes_formula": "B_alg = min(B_spmv, B_row, B_col_atomic, B_col_sort) = B_spmv at x = 100 %",
                     "step_share": round(per_point[top] / sum(per_point), 4),
                     "dominant_point": SPARSITIES[dom]},
        "selector_regret": round(regret_total, 4),
        "selector_schema2": ({"bundle": v2_path.name, "selected": [A_name(k) for k in chosen_v2],
                              "regret_per_point": [round(kernel_t[i][k] / min(kernel_t[i]), 3)
                                                   for i, k in enumerate(chosen_v2)],
                              "regret": round(sum(kernel_t[i][k] for i, k in enumerate(chosen_v2))
                                              / sum(min(r) for r in kernel_t), 4),
                              "note": "the optional schema-2 bundle (workload tree per pattern family) on the same "
                                      "operands and kernel timings; the line's value uses the default SPEC cascade"}
                             if chosen_v2 else None),
        "overhead": overhead,
        "gpu_launches": int(launches),
        "points": points,
        "setup_s": {"generate": round(gen_s, 1), "upload_csc_features": round(upload_s, 2),
                    "row_bins": round(bins_s, 3)},
        "clocks": clk.summary(),
    }
    ctx.set_timing(False)
    if cpu_line is not None:
        line["cpu_baseline"] = cpu_line
    del m, dvs, out, fresh, e2e_x
    torch.cuda.empty_cache()
    if args.configs:
        hbm_peak = hbm
        want = set(args.configs.split(","))
        cfgs = {}
        if "C1" in want:
            cfgs["C1"] = ours_c1(local, bundle, hbm_peak, flush, cpu)
        if "C3" in want:
            cfgs["C3"] = ours_c3(local, bundle, hbm_peak, cpu)
        if "C4" in want:
            cfgs["C4"] = ours_c4(local, bundle, hbm_peak, flush, cpu)
        if "C5" in want:
            try:
                c5ctx = A.Context(local)
                c5stream = torch.cuda.ExternalStream(c5ctx.stream, device=torch.device("cuda", local))
                with torch.cuda.stream(c5stream):
                    cfgs["C5"] = ours_c5(local, 0, 1, bundle, hbm_peak, c5ctx, c5stream)
                del c5ctx
            except Exception as e:  # never lose the headline line to the largest config
                cfgs["C5"] = {"error": f"{type(e).__name__}: {e}"}
        line["configs"] = cfgs
    return line


def cpu_baseline(rows, cols, ro, ci, vals, vecs):
    """The reference CPU implementation (oracle/_ref, bench build) on a
    bounded sample: one pass over the sweep, every point with its best
    reference kernel, benchmark_kernel timing -- the reference arm's step."""
    try:
        from oracle.oracle import have_ref
        if not have_ref(np.float32):
            return {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "reference",
                    "sample": "oracle/_ref not built"}
        ref, M, ops, nnz_s, best, threads = ref_c2_prepare(rows, cols, ro, ci, vals, vecs)
        ts = ref_c2_step(M, ops, best)
        v = sum(2 * s for s in nnz_s) / sum(ts) / 1e9
        res = {"value": round(v, 4), "unit": "GFLOP/s", "per_point_ms": [round(t * 1e3, 3) for t in ts],
               "kernel_per_point": [A_name(k) for k in best]}
        res.update(_cpu_meta(ref, threads, "one C2 sweep (7 points), best reference kernel per point, "
                                           "benchmark_kernel (1 warm-up, median of 3)"))
        return res
    except Exception as e:  # never fail the GPU line on the baseline
        return {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--bundle", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--lanes", type=int, default=3, help="streams of the e2e batch pipeline")
    ap.add_argument("--configs", default="C1,C3,C4,C5",
                    help="other configurations carried in the line ('' = none); N > 1 runs carry C5 only")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if world > 1:  # the partitioned runs carry configs[4] (C5) only
        args.configs = "C5" if "C5" in args.configs.split(",") else ""
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        multi = world > 1 or os.environ.get("ADASPMV_BENCH_FORCE_MULTI") == "1"  # 1-GPU test of the N>1 path
        line = run_ours_multi(args, rank, world) if multi else run_ours(args, rank, world)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
