"""train: fits the three-tree selector
bundle on samples from tools/gen_train.py and writes the model file the C++
runtime loads (paper_2006_16767_b200/selector/b200_bundle.txt).

  7:3 train/test split by seeded shuffle, CART grid search over
  depth [1,10] x class_weight {balanced, uniform} with 5-fold CV per tree.
  Four variants are fitted: all features vs a cheap-feature set that never
  reads nnz_s / m_sparsity (no device round trip per call),
  each with plain labels or cost-sensitive sample weights (the relative time
  lost by a wrong label, selector.costs_from_times).  The variant with the
  lowest held-out per-input regret (chosen / best-of-8) is written; a cheap
  variant within 2 % of it is preferred.  Per-tree held-out accuracies are
  reported for comparison with PAPER.md:582-593.
"""
from __future__ import annotations

import argparse
import csv
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_16767_b200 import selector as S  # noqa: E402


def load(paths):
    F, T, names = [], [], []
    for p in paths:
        with open(p) as fh:
            for row in csv.DictReader(fh):
                F.append([float(row[f"f{i}"]) for i in range(13)])
                T.append([float(row[f"t{k}"]) for k in range(8)])
                names.append(row["matrix"])
    return np.array(F), np.array(T), names


def regret(trees, F, T):
    sel = np.array([S.predict(trees, f) for f in F])
    chosen = T[np.arange(len(T)), sel]
    best = T.min(axis=1)
    return float(chosen.sum() / best.sum()), float(np.mean(chosen / best)), float(np.max(chosen / best)), sel


def accuracy(trees, F, T):
    lab = np.array([S.labels_from_times(t) for t in T])
    out = {}
    for j, t in enumerate(S.TARGETS):
        pred = []
        for f in F:
            nd = trees[t]
            i = 0
            while nd["feature"][i] >= 0:
                i = nd["left"][i] if f[nd["feature"][i]] <= nd["threshold"][i] else nd["right"][i]
            pred.append(nd["leaf"][i])
        pred = np.array(pred)
        mask = lab[:, 0] == 0 if t == "writeback" else np.ones(len(lab), bool)
        out[t] = float(np.mean(pred[mask] == lab[mask, j])) if mask.any() else 1.0
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("samples", nargs="+")
    ap.add_argument("--out", default=str(S.DEFAULT_PATH))
    ap.add_argument("--report", default="profiles/selector_r01.json")
    ap.add_argument("--seed", type=int, default=7)
    a = ap.parse_args()
    F, T, names = load(a.samples)
    rng = np.random.default_rng(a.seed)
    perm = rng.permutation(len(F))
    ntr = int(round(0.7 * len(F)))
    tr, te = perm[:ntr], perm[ntr:]
    results = {}
    for variant, hide, cs in (("full", 0, False), ("cheap", (1 << 11) | (1 << 12), False),
                              ("full_cost", 0, True), ("cheap_cost", (1 << 11) | (1 << 12), True)):
        saved = dict(S.MASKS)
        try:
            for t in S.TARGETS:
                S.MASKS[t] = saved[t] & ~hide
            trees, cv = S.train_bundle(F[tr], T[tr], seed=a.seed, cost_sensitive=cs)
        finally:
            S.MASKS.update(saved)
        rg_tot, rg_mean, rg_max, _ = regret(trees, F[te], T[te])
        results[variant] = {"trees": trees, "cv": cv, "test_accuracy": accuracy(trees, F[te], T[te]),
                            "test_regret_total": rg_tot, "test_regret_mean": rg_mean,
                            "test_regret_max": rg_max,
                            "train_regret_total": regret(trees, F[tr], T[tr])[0],
                            "nodes": {t: len(trees[t]["feature"]) for t in S.TARGETS}}
    # per-input regret (north_star: "within 10 % of the best of the eight per
    # input"); a cheap-feature variant wins ties within 2 % (no device round trip)
    order = sorted(results, key=lambda v: results[v]["test_regret_mean"])
    best_v = order[0]
    for v in order:
        if v.startswith("cheap") and results[v]["test_regret_mean"] <= 1.02 * results[best_v]["test_regret_mean"]:
            best_v = v
            break
    pick = best_v
    S.write_bundle(a.out, results[pick]["trees"], hardware_tag=f"B200-trained-{pick}")
    oracle_best = T.min(axis=1)
    fixed = {k: float(T[:, k].sum() / oracle_best.sum()) for k in range(8)}
    rep = {"samples": len(F), "matrices": sorted(set(names)), "train": int(ntr), "test": int(len(te)),
           "picked": pick, "fixed_kernel_regret_total": fixed,
           "variants": {v: {k: r[k] for k in r if k != "trees"} for v, r in results.items()}}
    Path(a.report).parent.mkdir(parents=True, exist_ok=True)
    Path(a.report).write_text(json.dumps(rep, indent=1))
    print(json.dumps({v: {k: rep["variants"][v][k] for k in ("test_accuracy", "test_regret_total",
                                                               "test_regret_mean", "test_regret_max", "nodes")}
                      for v in rep["variants"]}, indent=1))
    print("picked", pick, "-> wrote", a.out)


if __name__ == "__main__":
    main()
