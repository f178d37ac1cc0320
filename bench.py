#!/usr/bin/env python3
"""bench.py -- BASELINE.json metric on its 1-GPU configuration (configs[1]):

  "GFLOP/s and HBM GB/s (% of roofline) vs x sparsity; selector regret vs best"
  workload C2: uniform random 4M x 4M, 2^26 iid draws (~64M nnz), fp32,
  x-sparsity sweep 0.001 % .. 100 % across all 8 kernels + the selector.

A *step* is one adaptive pass over the sweep: for each of the 7 x-sparsity
points, select a kernel (C++ decision-tree hook) and run it, inputs resident
in HBM.  value = total useful GFLOP/s of the step = sum(2 nnz_s) / sum(t).
Every point is also timed with all 8 kernels (best-of-8, regret).

  --impl ours       (default) the CUDA library through its C-ABI
  --impl reference  the reference's own CPU implementation (oracle/_ref: the
                    unmodified reference headers) on the host cores

Timing: CUDA events on the library's stream around each multiply, medians
over K steps after W warm-up steps; an L2 flush (256 MiB write) precedes every
timed multiply whose working set fits in L2.  Selection overhead (feature
pulls + tree walks, format conversions) is measured on fresh vectors and
reported beside the value ("overhead").  e2e repeats the step through the
public API with host buffers (pinned): one adaspmv_run_batch call over the 7
vectors (H2D of x, select, multiply, D2H of y in its smaller form, pipelined
over 3 streams), wall clock; "sequential_value" is the same through single
calls.  N > 1 (torchrun): the row-partitioned mode, see run_ours_multi.
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

    def __init__(self, device=0):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
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


# ---------------------------------------------------------------------------
# reference CPU arm
# ---------------------------------------------------------------------------
def ref_sweep_times(ref_m, vecs, kernels_per_point, repeats=1, warmup=0):
    """Times the given kernel per point with the reference's run_kernel."""
    ts = []
    for (xi, xv), k in zip(vecs, kernels_per_point):
        dense = None
        if len(xi) == ref_m.cols:
            dense = np.zeros(ref_m.cols, np.float32)
            dense[xi] = xv
        t = ref_m.bench_kernel(k, x_dense=dense, x_sparse=None if dense is not None else (xi, xv),
                               warmup=warmup, repeats=repeats)
        ts.append(float(np.median(t)))
    return ts


def cpu_choose(ref_m, vecs):
    """Best reference kernel per point (1 warm-up + 1 run each); the sort
    write-back is skipped where nnz_x >= 1 % (seconds per call on CPU)."""
    best = []
    for (xi, xv) in vecs:
        dense = None
        if len(xi) == ref_m.cols:
            dense = np.zeros(ref_m.cols, np.float32)
            dense[xi] = xv
        cand = range(8) if len(xi) < 0.01 * ref_m.cols else (0, 1, 2, 3, 4, 6)
        tk = {}
        for k in cand:
            t = ref_m.bench_kernel(k, x_dense=dense, x_sparse=None if dense is not None else (xi, xv),
                                   warmup=1, repeats=1)
            tk[k] = float(t[0])
        best.append(min(tk, key=tk.get))
    return best


def run_reference(args, rank, world):
    from oracle.oracle import Ref

    if rank != 0:
        return None
    (rows, cols, ro, ci, vals), gen_s = make_matrix()
    nnz = int(ro[-1])
    vecs = make_vectors(cols)
    ref = Ref(np.float32)
    threads = os.cpu_count() or 1
    ref.set_threads(threads)
    M = ref.matrix(rows, cols, ro, ci, vals)
    del ci
    col_off = M.export()[3]
    nnz_s = [int(np.sum(col_off[xi + 1] - col_off[xi])) for xi, _ in vecs]
    best = cpu_choose(M, vecs)
    for _ in range(args.warmup):
        ref_sweep_times(M, vecs, best)
    steps = [ref_sweep_times(M, vecs, best) for _ in range(args.steps)]
    t_step = [sum(s) for s in steps]
    flops = sum(2 * s for s in nnz_s)
    v = flops / statistics.median(t_step) / 1e9
    line = {
        "metric": METRIC, "value": round(v, 4), "unit": "GFLOP/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(statistics.median(t_step) * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "rows": rows, "cols": cols, "nnz": nnz,
                   "x_sparsity": list(SPARSITIES), "kernel_per_point": best},
        "cpu_baseline": {"value": round(v, 4), "unit": "GFLOP/s", "cores": threads, "kind": "reference",
                         "sample": "full C2 sweep, best reference kernel per point (chosen by one timed "
                                   "pass; sort write-back skipped at >=1 % density)"},
        "e2e": {"value": round(v, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "per_point_ms": [round(statistics.median([s[i] for s in steps]) * 1e3, 4) for i in range(len(vecs))],
        "generation_s": round(gen_s, 1),
    }
    return line


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours_multi(args, rank, world):
    """N > 1: the row-partitioned mode (north_star), weak
    scaling.  Rank g owns a C2-sized row block (4M rows x 4M columns, 2^26
    draws, seed 1+g) of a (N*4M) x 4M matrix; every step broadcasts each sweep
    point's x from rank 0 over NCCL straight into device buffers handed to the
    library, then every rank runs its own selector + kernel on its block.
    Step time = max over ranks (CUDA events on the shared stream, barrier on
    both sides); value = all ranks' useful flops / step time."""
    import torch
    import torch.distributed as dist

    from paper_2006_16767_b200 import adaspmv as A
    from paper_2006_16767_b200 import selector as S
    from paper_2006_16767_b200 import synth

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
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)  # collectives order against it; the library launches on it
    ctx = A.Context(local, stream=stream.cuda_stream)
    rows, cols, ro, ci, vals = synth.uniform_random(N, DRAWS, seed=1 + rank, dtype=np.float32)
    m = A.DualMatrix.from_csr(rows, cols, ro, ci, vals, ctx=ctx)
    del ci
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

    ybuf = torch.zeros(rows, dtype=torch.float32).pin_memory().numpy()
    yidx = torch.zeros(rows, dtype=torch.int64).pin_memory().numpy()
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
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded numpy generator, SURVEY.md 8(d) C2 per rank)",
            "config": {"workload": WORKLOAD + ", row-partitioned: one C2-sized row block per GPU",
                       "rows_per_gpu": rows, "cols": cols, "x_sparsity": list(SPARSITIES),
                       "parallelism": f"row-partitioned x{world} (NCCL broadcast of x per point)",
                       "exchange_bytes_per_step": xbytes, "l2": "inputs larger than L2 at the dense points",
                       "timing": "per point: x broadcast (events) + multiply (library events), GPU gated, "
                                 "max over ranks; selection and x hand-over untimed as on 1 GPU"},
            "exchange": {"ms_per_step": round(float(tmax[3].item()) * 1e3, 4),
                         "fraction": round(float(tmax[3].item()) / t_step, 4),
                         "GBps": round(xbytes * max(world - 1, 0) / max(float(tmax[3].item()), 1e-12) / 1e9, 1)},
            "e2e": {"value": round(e2e_v, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": int(xbytes),
                    "d2h_bytes_per_step": int(d2h_bytes[0]),
                    "note": "x H2D on rank 0 then NCCL broadcast; each rank selects, multiplies and copies its "
                            "y block to pinned host memory in its smaller form; max over ranks"},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
    dist.destroy_process_group()
    return line


def run_ours(args, rank, world):
    import torch

    from paper_2006_16767_b200 import adaspmv as A
    from paper_2006_16767_b200 import selector as S

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = A.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    (rows, cols, ro, ci, vals), gen_s = make_matrix()
    nnz = int(ro[-1])
    vecs = make_vectors(cols)
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
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    out = A.MultiplyOutput(ctx)

    ctx.set_timing(True)  # CUDA events recorded by the library around each multiply

    def timed(fn, n_rep, need_flush):
        ts = []
        for _ in range(n_rep):
            with torch.cuda.stream(stream):
                if need_flush:
                    flush.add_(1)
                # the GPU spins while the host enqueues the multiply, so the
                # library's events see device time, not host launch latency
                torch.cuda._sleep(GATE_CYCLES)
            y = fn()
            if isinstance(y, tuple):
                y = y[0]
            ts.append(y.elapsed())
        return ts

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
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        steps = [step_times() for _ in range(args.steps)]
    torch.cuda.synchronize()
    launches = (ctx.launches - l0) // max(1, args.steps + args.warmup)
    t_step = [sum(s) for s in steps]
    t_med = statistics.median(t_step)
    if dist:
        tt = torch.tensor([t_med], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_med = float(tt.item())
    flops = sum(2 * s for s in nnz_s)
    value = world * flops / t_med / 1e9
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
    overhead = {"select_us_per_step": round(statistics.median(sel_t) * 1e6, 1),
                "convert_us_per_step": round(statistics.median(conv_t) * 1e6, 1),
                "note": "host feature pull (nnz_s on the device, one scalar back) + tree walk, and the "
                        "device format conversion the chosen kernel needs; excluded from value, "
                        "included in e2e"}
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
    e2e_v = world * flops / statistics.median(e2e_times) / 1e9
    # ---- roofline of the dominant kernel (the largest share of the step) ----
    per_point = [statistics.median([s[i] for s in steps]) for i in range(len(dvs))]
    dom = int(np.argmax(per_point))
    k_dom = chosen[dom]
    out_nnz = nnz_x[dom]
    _, fam = alg_bytes(rows, cols, nnz, nnz_x[dom], nnz_s[dom], out_nnz)
    hbm, src = peaks()
    achieved = fam[k_dom] / per_point[dom] / 1e9
    # DRAM bytes of the same kernel + input from the committed ncu --set full
    # capture (only when it is the kernel that dominates this run)
    prof = ROOT / "profiles" / "r01_roofline_traffic.json"
    traffic = None
    if prof.exists():
        try:
            pj = json.loads(prof.read_text())
            # spmv_direct reads the whole matrix whatever x holds: its DRAM
            # traffic per launch does not depend on the x sparsity
            if A.KernelId.from_index(k_dom).name() in pj.get("kernel", "") and \
                    (k_dom == 0 or f"x = {int(SPARSITIES[dom] * 100)} %" in pj.get("kernel", "")):
                traffic = pj.get("traffic_bytes_per_launch")
        except Exception:
            traffic = None
    points = []
    for i in range(len(dvs)):
        b_alg, fam_i = alg_bytes(rows, cols, nnz, nnz_x[i], nnz_s[i], 0)
        tb = min(kernel_t[i])
        points.append({
            "x_sparsity": SPARSITIES[i], "nnz_x": nnz_x[i], "nnz_s": nnz_s[i],
            "selected": A.KernelId.from_index(chosen[i]).name(), "t_sel_us": round(per_point[i] * 1e6, 2),
            "best": A.KernelId.from_index(int(np.argmin(kernel_t[i]))).name(), "t_best_us": round(tb * 1e6, 2),
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
        "config": {"workload": WORKLOAD, "rows": rows, "cols": cols, "nnz": nnz,
                   "x_sparsity": list(SPARSITIES), "l2": "256 MiB flush before timed multiplies with "
                   "working set < 64 MB; larger inputs exceed L2", "selector": str(bundle_path.name),
                   "parallelism": f"row-replicated x{world}" if world > 1 else "1 GPU"},
        "e2e": {"value": round(e2e_v, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "api": f"adaspmv_run_batch (pinned host buffers, {args.lanes} lanes)",
                "ms_per_step": round(statistics.median(e2e_times) * 1e3, 3),
                "sequential_value": round(world * flops / statistics.median(seq_times) / 1e9, 3),
                "sequential_api": "per vector: vector_set -> run_adaptive -> output copy",
                "kernels": e2e_kernels},
        "roofline": {"bound": "hbm", "kernel": A.KernelId.from_index(k_dom).name(),
                     "x_sparsity": SPARSITIES[dom], "achieved": round(achieved, 1), "peak": hbm,
                     "peak_source": src, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                     "traffic": traffic, "alg_bytes": int(fam[k_dom])},
        "selector_regret": round(regret_total, 4),
        "overhead": overhead,
        "gpu_launches": int(launches),
        "points": points,
        "setup_s": {"generate": round(gen_s, 1), "upload_csc_features": round(upload_s, 2)},
    }
    line["clocks"] = clk.summary()
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(rows, cols, ro, ci, vals, vecs)
    if dist:
        dist.destroy_process_group()
    return line if rank == 0 else None


def cpu_baseline(rows, cols, ro, ci, vals, vecs):
    """The reference CPU implementation (oracle/_ref) on a bounded sample:
    one pass over the sweep, every point with its best reference kernel."""
    try:
        from oracle.oracle import Ref, have_ref
        if not have_ref(np.float32):
            return {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "reference",
                    "sample": "oracle/_ref not built"}
        ref = Ref(np.float32)
        threads = os.cpu_count() or 1
        ref.set_threads(threads)
        M = ref.matrix(rows, cols, ro, ci, vals)
        col_off = M.export()[3]
        nnz_s = [int(np.sum(col_off[xi + 1] - col_off[xi])) for xi, _ in vecs]
        best = cpu_choose(M, vecs)
        ts = ref_sweep_times(M, vecs, best, repeats=3, warmup=1)
        v = sum(2 * s for s in nnz_s) / sum(ts) / 1e9
        return {"value": round(v, 4), "unit": "GFLOP/s", "cores": threads, "kind": "reference",
                "sample": "one C2 sweep (7 points), best reference kernel per point, median of 3",
                "per_point_ms": [round(t * 1e3, 3) for t in ts],
                "kernel_per_point": best}
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
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        multi = world > 1 or os.environ.get("ADASPMV_BENCH_FORCE_MULTI") == "1"  # 1-GPU test of the N>1 path
        line = run_ours_multi(args, rank, world) if multi else run_ours(args, rank, world)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
