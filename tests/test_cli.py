"""CLI surface: flag parsing, density specs, diagnostics
and exit codes on CPU; the `run`, `bench`, `features`, `convert` and
`gen-train -> train -> run` paths on the GPU."""
import csv
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2006_16767_b200 import cli

ROOT = Path(__file__).resolve().parents[1]


def test_density_points_spec_examples():
    assert cli.density_points("uniform:4", 100) == [1, 34, 67, 100]
    g = cli.density_points("geometric:5", 10000)
    assert g[0] == 1 and g[-1] == 10000 and len(g) == 5
    assert cli.density_points("uniform:4,geometric:3", 100) == [1, 10, 34, 67, 100]
    with pytest.raises(cli.CliError):
        cli.density_points("linear:3", 10)


def test_errors_exit_nonzero_with_one_line(tmp_path, capsys):
    assert cli.main(["run", "--app", "bfs", "--matrix", str(tmp_path / "nope.mtx")]) == 1
    err = capsys.readouterr().err.strip().splitlines()
    assert len(err) == 1 and "missing file" in err[0]
    assert cli.main(["bench", "--matrix", "x.mtx", "--bogus"]) == 1
    assert cli.main(["frobnicate"]) == 1
    bad = tmp_path / "s.csv"
    bad.write_text("a,b\n1,2\n")
    assert cli.main(["train", "--samples", str(bad), "--out", str(tmp_path / "m.txt")]) == 1
    assert "schema mismatch" in capsys.readouterr().err


def test_train_and_rank_features_on_samples(tmp_path):
    # a synthetic sample set in the gen-train schema: SpMV wins when x is dense
    rng = np.random.default_rng(0)
    rows = []
    for i in range(80):
        f = rng.random(13)
        dense = f[10] > 0.5
        t = rng.random(8) + 1.0
        t[0 if dense else 4] = 0.1
        rows.append(["m%d" % (i % 5), "float64", i] + [repr(float(v)) for v in f] + [repr(float(v)) for v in t])
    d = tmp_path / "samples"
    d.mkdir()
    cli._write_csv(d / "train.csv", cli.SAMPLE_COLUMNS, rows[:56])
    cli._write_csv(d / "test.csv", cli.SAMPLE_COLUMNS, rows[56:])
    out = tmp_path / "model.txt"
    r = subprocess.run([sys.executable, "-m", "paper_2006_16767_b200.cli", "train", "--samples", str(d),
                        "--out", str(out), "--folds", "3"], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "test_regret_total" in r.stdout and out.read_text().startswith("adaspmv-bundle 1")
    r = subprocess.run([sys.executable, "-m", "paper_2006_16767_b200.cli", "rank-features", "--samples", str(d)],
                       cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert '"pattern": ["x_sparsity"' in r.stdout


def _path_graph(tmp_path):
    p = tmp_path / "path.mtx"
    p.write_text("%%MatrixMarket matrix coordinate pattern symmetric\n4 4 3\n2 1\n3 2\n4 3\n")
    return p


@pytest.mark.gpu
def test_run_bfs_path_graph_stats(tmp_path):
    p = _path_graph(tmp_path)
    stats, lv = tmp_path / "stats.csv", tmp_path / "levels.txt"
    assert cli.main(["run", "--app", "bfs", "--matrix", str(p), "--stats", str(stats), "--output", str(lv)]) == 0
    lines = [ln for ln in stats.read_text().splitlines() if not ln.startswith("#")]
    rows = list(csv.reader(lines))
    assert rows[0] == cli.STATS_COLUMNS and len(rows) == 5  # 4 stat rows
    assert np.loadtxt(lv, dtype=np.int64).tolist() == [0, 1, 2, 3]
    assert stats.read_text().splitlines()[-1].startswith("# summary")


@pytest.mark.gpu
def test_bench_features_convert_pagerank(tmp_path, capsys):
    p = _path_graph(tmp_path)
    out = tmp_path / "b.csv"
    assert cli.main(["bench", "--matrix", str(p), "--kernels", "all", "--densities", "uniform:4",
                     "--repeats", "2", "--out", str(out)]) == 0
    rows = list(csv.reader(ln for ln in out.read_text().splitlines() if not ln.startswith("#")))
    assert len(rows) == 1 + 4 and all(len(r) == 2 + 8 for r in rows)  # 8 timing columns per density row
    capsys.readouterr()
    assert cli.main(["features", "--matrix", str(p), "--density", "0.5"]) == 0
    feat = [ln for ln in capsys.readouterr().out.splitlines() if not ln.startswith("#")]
    assert len(feat[0].split(",")) == 13 and len(feat[1].split(",")) == 13
    b = tmp_path / "p.bin"
    assert cli.main(["convert", "--input", str(p), "--output", str(b)]) == 0 and b.stat().st_size > 0
    rk = tmp_path / "rank.txt"
    assert cli.main(["run", "--app", "pagerank", "--matrix", str(b), "--prune", "0", "--max-iters", "2000",
                     "--output", str(rk)]) == 0
    r = np.loadtxt(rk)
    assert r[1] > r[0] and abs(r[1] - r[2]) < 1e-12 and abs(r[0] - r[3]) < 1e-12


@pytest.mark.gpu
def test_gen_train_train_run_round_trip(tmp_path):
    from paper_2006_16767_b200 import adaspmv as A
    from paper_2006_16767_b200 import synth
    corpus = tmp_path / "corpus"
    corpus.mkdir()
    ctx = A.Context(0)
    for i, (r, c, ro, ci, v) in enumerate([synth.random_csr(400, 400, 0.02, seed=1),
                                           synth.random_csr(900, 900, 0.005, seed=2)]):
        A.DualMatrix.from_csr(r, c, ro, ci, v, ctx=ctx).write_matrix_market(corpus / f"m{i}.mtx")
    samples = tmp_path / "samples"
    assert cli.main(["gen-train", "--corpus", str(corpus), "--densities", "uniform:4,geometric:4", "--repeats", "2",
                     "--split", "7:3", "--seed", "3", "--out", str(samples)]) == 0
    model = tmp_path / "model.txt"
    assert cli.main(["train", "--samples", str(samples), "--out", str(model), "--folds", "3"]) == 0
    stats = tmp_path / "s.csv"
    assert cli.main(["run", "--app", "bfs", "--matrix", str(corpus / "m0.mtx"), "--model", str(model),
                     "--stats", str(stats)]) == 0
