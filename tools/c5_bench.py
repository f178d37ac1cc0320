"""C5-scale run on one B200 (BASELINE.json configs[4] at N = 1): an R-MAT
scale-26 graph (Graph500 parameters, ~2.1 G stored entries after
symmetrisation) generated ON THE DEVICE with torch (measurement input only),
handed to the library as device CSR (adaspmv_matrix_create_csr_device: the
CSC is built on the device), then

  * SpMV / SpMSpV over an x-sparsity sweep with every kernel that finishes
    (device time, CUDA events), GFLOP/s and % of the HBM roofline;
  * BFS from vertex 0 (OR_AND), traversal time and GTEPS.

No CPU oracle at this size; correctness is covered by the parity tests and,
here, by checking the BFS level counts against a second BFS run with a
different kernel policy and y sums against spmv_lb.

  python tools/c5_bench.py --scale 26 --out gpurun_out/c5.json
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_16767_b200 import adaspmv as A  # noqa: E402
from paper_2006_16767_b200 import selector as S  # noqa: E402


def rmat_device(scale, edge_factor=16, abcd=(0.57, 0.19, 0.19, 0.05), seed=2, chunk=1 << 26):
    """Symmetrised, deduplicated, self-loop-free R-MAT on the GPU -> (row_offsets
    int64, col_indices int32) device tensors."""
    n = 1 << scale
    m = edge_factor * n
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    a, b, c, _ = abcd
    keys = []
    for s0 in range(0, m, chunk):
        k = min(chunk, m - s0)
        rs = torch.zeros(k, dtype=torch.int64, device="cuda")
        cs = torch.zeros(k, dtype=torch.int64, device="cuda")
        for _ in range(scale):
            u = torch.rand(k, generator=g, device="cuda")
            rbit = (u >= a + b).long()
            cbit = (((u >= a) & (u < a + b)) | (u >= a + b + c)).long()
            rs = (rs << 1) | rbit
            cs = (cs << 1) | cbit
        keep = rs != cs
        rs, cs = rs[keep], cs[keep]
        keys.append(rs * n + cs)
        keys.append(cs * n + rs)
        del rs, cs, keep
    keys = torch.cat(keys)
    keys = torch.unique(keys)  # sorted, deduplicated
    rows = keys >> scale
    cols = (keys & (n - 1)).to(torch.int32)
    del keys
    ro = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    ro[1:] = torch.cumsum(torch.bincount(rows, minlength=n), 0)
    del rows
    return n, ro, cols


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--kernels", default="0,1,2,3,4,6")
    ap.add_argument("--densities", default="0.00001,0.001,0.1,1.0")
    ap.add_argument("--panels", default="", help="x KiB per column panel to time spmv_direct with (dense x)")
    a = ap.parse_args()
    t0 = time.time()
    n, ro, ci = rmat_device(a.scale)
    nnz = int(ro[-1].item())
    gen_s = time.time() - t0
    vals = torch.rand(nnz, dtype=torch.float32, device="cuda") * 2 - 1
    torch.cuda.empty_cache()  # return the generator's sort buffers before the CSC build
    ctx = A.Context(0)
    t0 = time.time()
    m = A.DualMatrix.from_device(n, n, nnz, ro.data_ptr(), ci.data_ptr(), vals.data_ptr(), np.float32, ctx)
    build_s = time.time() - t0
    free, total = torch.cuda.mem_get_info()
    del ci, vals
    torch.cuda.empty_cache()
    res = {"scale": a.scale, "n": n, "nnz": nnz, "generate_s": round(gen_s, 1),
           "device_csr_to_dual_s": round(build_s, 2), "gpu_mem_used_gb_at_build": round((total - free) / 1e9, 1),
           "features": m.features().tolist(), "spmv": [], "bfs": {}}
    print(json.dumps({k: res[k] for k in ("scale", "n", "nnz", "generate_s", "device_csr_to_dual_s",
                                          "gpu_mem_used_gb_at_build")}), flush=True)
    ctx.set_timing(True)
    stream = torch.cuda.ExternalStream(ctx.stream)
    out = A.MultiplyOutput(ctx)
    bundle = A.SelectorBundle.load(S.DEFAULT_PATH)
    ro_h = ro.cpu().numpy()
    del ro
    hbm = 6532.9e9
    for dens in [float(s) for s in a.densities.split(",")]:
        nx = max(1, int(round(dens * n)))
        rng = np.random.default_rng(7)
        xi = np.sort(rng.choice(n, size=nx, replace=False)) if nx < n else np.arange(n)
        xv = rng.uniform(-1, 1, nx).astype(np.float32)
        x = A.DeviceVector(n, np.float32, ctx)
        if nx == n:
            d = np.zeros(n, np.float32)
            d[xi] = xv
            x.set_dense(d)
        else:
            x.set_sparse(xi, xv)
        nnz_s = A.effective_nnz(m, x)
        b_spmv = (n + 1) * 8 + nnz * 8 + n * 4 + n * 4
        row = {"x_sparsity": dens, "nnz_x": nx, "nnz_s": nnz_s, "kernels": {}}
        ref_sum = None
        for k in [int(s) for s in a.kernels.split(",")] + ["adaptive"]:
            ts = []
            for r in range(a.reps + 1):
                with torch.cuda.stream(stream):
                    torch.cuda._sleep(400_000)
                if k == "adaptive":
                    y, kk = A.run_adaptive(m, x, bundle, out=out)
                else:
                    x.prepare(k)
                    y = A.run_kernel(m, k, x, out=out)
                if r:
                    ts.append(y.elapsed())
            t = float(np.median(ts))
            ent = {"t_us": round(t * 1e6, 2), "gflops": round(2 * nnz_s / t / 1e9, 2)}
            if k == "adaptive":
                ent["selected"] = kk.name()
            if dens == 1.0:
                ent["pct_hbm_spmv_bytes"] = round(100 * b_spmv / t / hbm, 1)
            s = float(np.sum(y.dense().values, dtype=np.float64))
            ref_sum = s if ref_sum is None else ref_sum
            ent["y_sum_rel_diff"] = abs(s - ref_sum) / max(abs(ref_sum), 1e-30)
            row["kernels"][str(k)] = ent
            print(dens, k, ent, flush=True)
        res["spmv"].append(row)
    if a.panels:  # spmv_direct (row bins) vs the column-panel width, dense x
        xd = np.random.default_rng(7).uniform(-1, 1, n).astype(np.float32)
        x = A.DeviceVector(n, np.float32, ctx).set_dense(xd)
        ref = None
        res["panels"] = []
        for pk in [int(v) for v in a.panels.split(",")]:
            cfg = A.KernelConfig(row_layout=2, bin_panel_kib=pk)
            y = A.run_kernel(m, 0, x, cfg, out=out)
            s_ = float(np.sum(y.dense().values, dtype=np.float64))
            ref = s_ if ref is None else ref
            ts = []
            for _ in range(a.reps):
                with torch.cuda.stream(stream):
                    torch.cuda._sleep(400_000)
                ts.append(A.run_kernel(m, 0, x, cfg, out=out).elapsed())
            t = float(np.median(ts))
            b_spmv = (n + 1) * 8 + nnz * 8 + n * 4 + n * 4
            ent = {"panel_kib": pk, "t_us": round(t * 1e6, 1), "pct_hbm_spmv_bytes": round(100 * b_spmv / t / hbm, 1),
                   "y_sum_rel_diff": abs(s_ - ref) / max(abs(ref), 1e-30)}
            res["panels"].append(ent)
            print("panel", ent, flush=True)
    del out
    lv_ref = None
    for name, forced in (("heuristic", -1), ("row_lb_masked_pull", 3), ("col_lb_atomic", 6)):
        ts = []
        for r in range(a.reps):
            ctx.synchronize()
            t1 = time.perf_counter()
            _, reps = A.bfs(m, 0, A.OR_AND, force_kernel=forced, download_levels=False)
            ts.append(time.perf_counter() - t1)
        lv, _ = A.bfs(m, 0, A.OR_AND, force_kernel=forced)
        lv_ref = lv if lv_ref is None else lv_ref
        reached = lv >= 0
        edges = int(np.sum(np.diff(ro_h)[reached]))
        t = float(np.median(ts))
        res["bfs"][name] = {"seconds": round(t, 5), "levels": len(reps), "reached": int(reached.sum()),
                            "gteps": round(edges / t / 1e9, 2), "levels_equal_heuristic": bool(np.array_equal(lv, lv_ref)),
                            "per_level": [{"nnz_x": r_["nnz_x"], "kernel": A.KernelId.from_index(r_["kernel"]).name(),
                                           "kernel_ms": round(r_["kernel_s"] * 1e3, 3)} for r_ in reps]}
        print(name, res["bfs"][name]["seconds"], res["bfs"][name]["gteps"], flush=True)
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
