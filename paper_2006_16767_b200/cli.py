"""Command-line surface of SPEC.md:516-531 (module cli-apps) over the CUDA
library: corpus tools, the selector training pipeline, benchmarks and the two
driver applications (BFS, incremental PageRank).

    python -m paper_2006_16767_b200.cli <subcommand> [flags]

  convert        --input <mtx> --output <bin>
  features       --matrix <path> [--vector <path> | --density <r>] [--seed s]
  bench          --matrix <path> --kernels <all|id,...> --densities <uniform:k|geometric:k> --repeats <n>
  gen-train      --corpus <dir> --densities <spec> --repeats <n> --split 7:3 --seed <s> --out <dir>
  train          --samples <dir> --out <model file> --folds 5 [--cost-lambda <l>]
  rank-features  --samples <dir>
  run            --app <bfs|pagerank> --matrix <path> --model <file|none> [--source v]
                 [--damping d --prune p] [--force-kernel <id>] [--threads w] --stats <csv>

Flags are the SPEC's.  Exit code 0 on success, 1 with a
one-line diagnostic on failure (unknown flag, missing file, schema mismatch).
CSV outputs carry a versioned header row; the stats CSV columns
are iter, nnz_x, kernel, feature_s, predict_s, convert_s, kernel_s, followed
by a `# summary` line.  Randomness is seeded by `--seed`.  `--threads` is
accepted for compatibility and ignored: the kernels run on the GPU (the
reference's worker count has no device meaning).

Matrix files: Matrix Market (.mtx) or the reference's ASPMVBIN cache (.bin),
through the library's loader (matrix_market.hpp:38-238 semantics).  Vector
files (--vector): Matrix Market "matrix coordinate" n x 1, or lines of
"index value" (0-based) with a first line "n <length>".
"""
from __future__ import annotations

import argparse
import csv
import json
import sys
import time
from pathlib import Path

import numpy as np

from . import adaspmv as A
from . import selector as S

SCHEMA = "adaspmv-csv-v1"
STATS_COLUMNS = ["iter", "nnz_x", "kernel", "feature_s", "predict_s", "convert_s", "kernel_s"]
SAMPLE_COLUMNS = ["matrix", "dtype", "nnz_x"] + [f"f{i}" for i in range(13)] + [f"t{k}" for k in range(8)]


class CliError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # one-line diagnostic, nonzero exit
        raise CliError(message)


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------
def density_points(spec: str, n: int) -> list[int]:
    """SPEC.md:456 / :434: "uniform:k" = k points linearly interpolated from 1
    to n (uniform:4 on n=100 -> 1, 34, 67, 100); "geometric:k" = k points
    geometrically spaced from 1 to n.  Comma-separated specs are merged."""
    pts: set[int] = set()
    for part in spec.split(","):
        kind, _, k = part.partition(":")
        try:
            k = int(k)
        except ValueError:
            raise CliError(f"bad density spec '{part}' (want uniform:k or geometric:k)") from None
        if k < 1 or n < 1:
            raise CliError(f"bad density spec '{part}'")
        if kind == "uniform":
            vals = [1 + (n - 1) * i / (k - 1) for i in range(k)] if k > 1 else [n]
        elif kind == "geometric":
            vals = np.geomspace(1, n, k).tolist() if k > 1 else [n]
        else:
            raise CliError(f"bad density spec '{part}' (want uniform:k or geometric:k)")
        pts.update(min(n, max(1, int(np.floor(v + 0.5)))) for v in vals)
    return sorted(pts)


def _load_matrix(path, ctx, dtype=np.float64):
    p = Path(path)
    if not p.is_file():
        raise CliError(f"missing file: {path}")
    return A.load_matrix(p, dtype=dtype, ctx=ctx)


def _load_vector(path, n):
    p = Path(path)
    if not p.is_file():
        raise CliError(f"missing file: {path}")
    lines = [ln.split() for ln in p.read_text().splitlines() if ln.strip() and not ln.startswith("%")]
    if not lines:
        raise CliError(f"empty vector file: {path}")
    if lines[0][0] == "n":
        length = int(lines[0][1])
        body = [(int(a), float(b)) for a, b in lines[1:]]
    else:  # Matrix Market coordinate n x 1 (1-based)
        length = int(lines[0][0])
        body = [(int(a) - 1, float(c)) for a, _, c in lines[1:]]
    if length != n:
        raise CliError(f"vector length {length} != matrix columns {n}")
    body.sort()
    idx = np.array([i for i, _ in body], np.int64)
    val = np.array([v for _, v in body], np.float64)
    return idx, val


def _random_sparse(n, nnz, seed, dtype):
    """distinct uniform indices, values U[-1,1], fixed seed."""
    rng = np.random.default_rng(seed)
    nnz = min(max(int(nnz), 0), n)
    idx = np.sort(rng.choice(n, size=nnz, replace=False)).astype(np.int64) if nnz < n else np.arange(n)
    return idx, rng.uniform(-1.0, 1.0, nnz).astype(dtype)


def _time_kernels(m, x, kernels, repeats, out):
    """benchmark_kernel: 1 warm-up, median of `repeats`,
    kernel only (device time from the library's CUDA events)."""
    ts = {}
    for k in kernels:
        x.prepare(k)
        A.run_kernel(m, k, x, out=out)
        rep = []
        for _ in range(max(1, repeats)):
            A.run_kernel(m, k, x, out=out)
            rep.append(out.elapsed())
        ts[k] = float(np.median(rep))
    return ts


def _write_csv(path, header, rows):
    with open(path, "w", newline="") as fh:
        fh.write(f"# {SCHEMA}\n")
        w = csv.writer(fh)
        w.writerow(header)
        w.writerows(rows)


def _read_samples(d):
    d = Path(d)
    files = [d] if d.is_file() else sorted(d.glob("*.csv"))
    if not files:
        raise CliError(f"no sample CSVs under {d}")
    out = {}
    for f in files:
        with open(f) as fh:
            lines = [ln for ln in fh if not ln.startswith("#")]
        rd = csv.DictReader(lines)
        if rd.fieldnames is None or list(rd.fieldnames) != SAMPLE_COLUMNS:
            raise CliError(f"schema mismatch in {f}")
        rows = list(rd)
        F = np.array([[float(r[f"f{i}"]) for i in range(13)] for r in rows]).reshape(-1, 13)
        T = np.array([[float(r[f"t{k}"]) for k in range(8)] for r in rows]).reshape(-1, 8)
        out[f.stem] = (F, T, [r["matrix"] for r in rows])
    return out


# ---------------------------------------------------------------------------
# subcommands
# ---------------------------------------------------------------------------
def _need(path):
    if not Path(path).is_file():
        raise CliError(f"missing file: {path}")


def cmd_convert(a):
    _need(a.input)
    ctx = A.Context(0)
    m = _load_matrix(a.input, ctx)
    m.save_binary(a.output)
    print(json.dumps({"rows": m.rows(), "cols": m.cols(), "nnz": m.nnz(), "output": a.output}))


def cmd_features(a):
    _need(a.matrix)
    if a.vector:
        _need(a.vector)
    ctx = A.Context(0)
    m = _load_matrix(a.matrix, ctx)
    if a.vector:
        idx, val = _load_vector(a.vector, m.cols())
    else:
        idx, val = _random_sparse(m.cols(), round(a.density * m.cols()), a.seed, np.float64)
    x = A.DeviceVector(m.cols(), np.float64, ctx).set_sparse(idx, val)
    f = A.features(m, x)
    w = csv.writer(sys.stdout)
    sys.stdout.write(f"# {SCHEMA}\n")
    w.writerow(S.FEATURES)
    w.writerow([repr(float(v)) for v in f])


def _kernel_list(spec):
    if spec == "all":
        return list(range(8))
    try:
        ks = [int(s) for s in spec.split(",")]
    except ValueError:
        ks = []
        for s in spec.split(","):
            kid = A.KernelId.parse(s)
            if kid is None:
                raise CliError(f"unknown kernel '{s}'") from None
            ks.append(kid.index())
    if any(k < 0 or k > 7 for k in ks):
        raise CliError("kernel ids are 0..7")
    return ks


def cmd_bench(a):
    _need(a.matrix)
    ks = _kernel_list(a.kernels)
    ctx = A.Context(0)
    ctx.set_timing(True)
    m = _load_matrix(a.matrix, ctx, np.float32 if a.dtype == "f32" else np.float64)
    dt = np.float32 if a.dtype == "f32" else np.float64
    out = A.MultiplyOutput(ctx)
    rows = []
    for i, nx in enumerate(density_points(a.densities, m.cols())):
        idx, val = _random_sparse(m.cols(), nx, a.seed + i, dt)
        x = A.DeviceVector(m.cols(), dt, ctx)
        if nx == m.cols():
            d = np.zeros(m.cols(), dt)
            d[idx] = val
            x.set_dense(d)
        else:
            x.set_sparse(idx, val)
        ts = _time_kernels(m, x, ks, a.repeats, out)
        rows.append([nx, nx / m.cols()] + [repr(ts.get(k, float("nan"))) for k in range(8)])
    out_f = open(a.out, "w", newline="") if a.out else sys.stdout
    out_f.write(f"# {SCHEMA}\n")
    w = csv.writer(out_f)
    w.writerow(["nnz_x", "density"] + [A.KernelId.from_index(k).name() for k in range(8)])
    w.writerows(rows)
    if a.out:
        out_f.close()


def cmd_gen_train(a):
    """generate_training_data."""
    corpus = sorted(p for p in Path(a.corpus).glob("*") if p.suffix in (".mtx", ".bin"))
    if not corpus:
        raise CliError(f"empty corpus: {a.corpus}")
    try:
        tr_w, te_w = (int(v) for v in a.split.split(":"))
    except ValueError:
        raise CliError(f"bad --split '{a.split}'") from None
    ctx = A.Context(0)
    ctx.set_timing(True)
    out = A.MultiplyOutput(ctx)
    rng = np.random.default_rng(a.seed)
    rows = []
    for mi, path in enumerate(corpus):
        m = _load_matrix(path, ctx)
        for i, nx in enumerate(density_points(a.densities, m.cols())):
            idx, val = _random_sparse(m.cols(), nx, a.seed * 1_000_003 + mi * 1009 + i, np.float64)
            x = A.DeviceVector(m.cols(), np.float64, ctx)
            if nx == m.cols():
                d = np.zeros(m.cols())
                d[idx] = val
                x.set_dense(d)
            else:
                x.set_sparse(idx, val)
            f = A.features(m, x)
            ts = _time_kernels(m, x, range(8), a.repeats, out)
            rows.append([path.name, "float64", nx] + [repr(float(v)) for v in f] +
                        [repr(ts[k]) for k in range(8)])
    perm = rng.permutation(len(rows))
    ntr = int(round(len(rows) * tr_w / max(tr_w + te_w, 1)))
    od = Path(a.out)
    od.mkdir(parents=True, exist_ok=True)
    _write_csv(od / "train.csv", SAMPLE_COLUMNS, [rows[i] for i in perm[:ntr]])
    _write_csv(od / "test.csv", SAMPLE_COLUMNS, [rows[i] for i in perm[ntr:]])
    print(json.dumps({"samples": len(rows), "train": ntr, "test": len(rows) - ntr, "out": str(od)}))


def cmd_train(a):
    sets = _read_samples(a.samples)
    F, T, _ = sets.get("train", next(iter(sets.values())))
    lab = np.array([S.labels_from_times(t) for t in T])
    cst = np.array([S.costs_from_times(t) for t in T]) if a.cost_lambda > 0 else None
    trees, scores = {}, {}
    for j, t in enumerate(S.TARGETS):
        c = None if cst is None else 1.0 + a.cost_lambda * cst[:, j]
        trees[t], scores[t] = S.train_tree(F, lab[:, j], S.MASKS[t], folds=a.folds, seed=a.seed, cost=c)
    S.write_bundle(a.out, trees, hardware_tag="B200-cli")
    rep = {"cv": scores, "out": a.out}
    if "test" in sets:
        Ft, Tt, _ = sets["test"]
        sel = np.array([S.predict(trees, f) for f in Ft])
        chosen = Tt[np.arange(len(Tt)), sel]
        rep["test_regret_total"] = float(chosen.sum() / Tt.min(axis=1).sum())
    print(json.dumps(rep))


def cmd_rank_features(a):
    """chi^2 ordering of the 13 features per target."""
    from sklearn.feature_selection import chi2
    sets = _read_samples(a.samples)
    F = np.concatenate([v[0] for v in sets.values()])
    T = np.concatenate([v[1] for v in sets.values()])
    lab = np.array([S.labels_from_times(t) for t in T])
    out = {}
    for j, t in enumerate(S.TARGETS):
        cols = [i for i in range(13) if S.MASKS[t] & (1 << i)]
        if len(np.unique(lab[:, j])) < 2:
            out[t] = [S.FEATURES[i] for i in cols]
            continue
        Fn = F[:, cols] - F[:, cols].min(axis=0)
        chi, _ = chi2(Fn, lab[:, j])
        chi = np.nan_to_num(chi)
        out[t] = [S.FEATURES[cols[i]] for i in np.argsort(-chi, kind="stable")]
    print(json.dumps(out))


def cmd_run(a):
    _need(a.matrix)
    if a.model and a.model != "none":
        _need(a.model)
    ctx = A.Context(0)
    m = _load_matrix(a.matrix, ctx, np.float32 if a.dtype == "f32" else np.float64)
    bundle = None
    if a.model and a.model != "none":
        if not Path(a.model).is_file():
            raise CliError(f"missing file: {a.model}")
        bundle = A.SelectorBundle.load(a.model)
    if a.force_kernel is not None:
        bundle = None
    forced = -1 if a.force_kernel is None else int(a.force_kernel)
    t0 = time.perf_counter()
    if a.app == "bfs":
        res, reps = A.bfs(m, a.source, A.PLUS_TIMES if a.semiring == "plus_times" else
                          (A.MIN_PLUS if a.semiring == "min_plus" else A.OR_AND), bundle=bundle,
                          force_kernel=forced)
    else:
        res, reps = A.pagerank_incremental(m, a.damping, a.prune, a.max_iters, bundle=bundle,
                                           force_kernel=forced)
    wall = time.perf_counter() - t0
    rows = [[r["iteration"], r["nnz_x"], A.KernelId.from_index(r["kernel"]).name(), repr(r["feature_s"]),
             repr(r["predict_s"]), repr(r["convert_s"]), repr(r["kernel_s"])] for r in reps]
    overhead = sum(r["feature_s"] + r["predict_s"] + r["convert_s"] for r in reps)
    total = overhead + sum(r["kernel_s"] for r in reps)
    switches = sum(1 for i in range(1, len(reps)) if reps[i]["kernel"] != reps[i - 1]["kernel"])
    summary = {"app": a.app, "iterations": len(reps), "kernel_switches": switches, "wall_s": wall,
               "overhead_fraction": overhead / total if total > 0 else 0.0}
    if a.stats:
        _write_csv(a.stats, STATS_COLUMNS, rows)
        with open(a.stats, "a") as fh:
            fh.write("# summary " + json.dumps(summary) + "\n")
    if a.output:
        np.savetxt(a.output, res, fmt="%d" if a.app == "bfs" else "%.17g")
    print(json.dumps(summary))


def build_parser():
    p = _Parser(prog="adaspmv", description=__doc__.split("\n\n")[0])
    sub = p.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    c = sub.add_parser("convert")
    c.add_argument("--input", required=True)
    c.add_argument("--output", required=True)
    c.set_defaults(fn=cmd_convert)
    c = sub.add_parser("features")
    c.add_argument("--matrix", required=True)
    g = c.add_mutually_exclusive_group()
    g.add_argument("--vector")
    g.add_argument("--density", type=float, default=0.01)
    c.add_argument("--seed", type=int, default=0)
    c.set_defaults(fn=cmd_features)
    c = sub.add_parser("bench")
    c.add_argument("--matrix", required=True)
    c.add_argument("--kernels", default="all")
    c.add_argument("--densities", default="geometric:8")
    c.add_argument("--repeats", type=int, default=10)
    c.add_argument("--dtype", choices=("f32", "f64"), default="f64")
    c.add_argument("--seed", type=int, default=0)
    c.add_argument("--out")
    c.set_defaults(fn=cmd_bench)
    c = sub.add_parser("gen-train")
    c.add_argument("--corpus", required=True)
    c.add_argument("--densities", default="geometric:16,uniform:8")
    c.add_argument("--repeats", type=int, default=10)
    c.add_argument("--split", default="7:3")
    c.add_argument("--seed", type=int, default=0)
    c.add_argument("--out", required=True)
    c.set_defaults(fn=cmd_gen_train)
    c = sub.add_parser("train")
    c.add_argument("--samples", required=True)
    c.add_argument("--out", required=True)
    c.add_argument("--folds", type=int, default=5)
    c.add_argument("--cost-lambda", type=float, default=0.0)
    c.add_argument("--seed", type=int, default=0)
    c.set_defaults(fn=cmd_train)
    c = sub.add_parser("rank-features")
    c.add_argument("--samples", required=True)
    c.set_defaults(fn=cmd_rank_features)
    c = sub.add_parser("run")
    c.add_argument("--app", choices=("bfs", "pagerank"), required=True)
    c.add_argument("--matrix", required=True)
    c.add_argument("--model", default="none")
    c.add_argument("--source", type=int, default=0)
    c.add_argument("--semiring", choices=("plus_times", "or_and", "min_plus"), default="plus_times")
    c.add_argument("--damping", type=float, default=0.85)
    c.add_argument("--prune", type=float, default=1e-6)
    c.add_argument("--max-iters", type=int, default=300)
    c.add_argument("--force-kernel", type=int)
    c.add_argument("--threads", type=int)
    c.add_argument("--dtype", choices=("f32", "f64"), default="f64")
    c.add_argument("--stats")
    c.add_argument("--output")
    c.add_argument("--seed", type=int, default=0)
    c.set_defaults(fn=cmd_run)
    return p


def main(argv=None) -> int:
    try:
        a = build_parser().parse_args(argv)
        a.fn(a)
        return 0
    except CliError as e:
        print(f"adaspmv: error: {e}", file=sys.stderr)
        return 1
    except (A.AdaspmvError, A.LibraryMissing, OSError, ValueError) as e:
        print(f"adaspmv: error: {type(e).__name__}: {str(e).splitlines()[0] if str(e) else ''}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
