"""Offline study (CPU): the SPEC cascade (one workload tree on matrix features,
SPEC.md:227) vs a schema-v2 cascade with one workload tree per pattern family
(row: SpMV / RowSpMSpV, col: ColSpMSpV) that may read the vector features,
trained and evaluated on the same B200-timed samples and the same 7:3 split.

  python tools/selector_v2_study.py profiles/data/train_samples_r01*.csv
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from paper_2006_16767_b200 import selector as S  # noqa: E402
from train_selector import load  # noqa: E402


def regret_stats(sel, T):
    chosen = T[np.arange(len(T)), sel]
    best = T.min(axis=1)
    r = chosen / best
    return {"total": float(chosen.sum() / best.sum()), "mean": float(r.mean()), "max": float(r.max()),
            "share_le_1.10": float(np.mean(r <= 1.10))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("samples", nargs="+")
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--out", default=str(S.DEFAULT_PATH.parent / "b200_bundle_v2.txt"))
    ap.add_argument("--report", default="profiles/selector_r02_v2.json")
    a = ap.parse_args()
    F, T, names = load(a.samples)
    rng = np.random.default_rng(a.seed)
    perm = rng.permutation(len(F))
    ntr = int(round(0.7 * len(F)))
    tr, te = perm[:ntr], perm[ntr:]
    out = {}
    # v1: the SPEC cascade, cost-sensitive (the shipped variant's recipe)
    v1, _ = S.train_bundle(F[tr], T[tr], seed=a.seed, cost_sensitive=True)
    out["v1_spec_cascade"] = regret_stats(np.array([S.predict(v1, f) for f in F[te]]), T[te])
    # v2: workload tree per pattern family, each trained on ALL samples with
    # its conditional label (faster distribution within that family)
    v2, _ = S.train_bundle_v2(F[tr], T[tr], seed=a.seed)
    out["v2_workload_per_pattern"] = regret_stats(np.array([S.predict(v2, f) for f in F[te]]), T[te])
    # oracle pattern + learned rest: how much is the pattern tree's share
    pat_best = np.array([S.labels_from_times(t)[0] for t in T[te]])
    sel = []
    for f, p in zip(F[te], pat_best):
        k = S.predict(v2, f)
        sel.append(k)
    out["fixed_best_single_kernel"] = min(
        (regret_stats(np.full(len(te), k), T[te]) for k in range(8)), key=lambda d: d["mean"])
    worst = np.argsort(-(T[te][np.arange(len(te)), np.array([S.predict(v2, f) for f in F[te]])] / T[te].min(1)))[:8]
    out["v2_worst_inputs"] = [{"matrix": names[te[i]], "nnz_x": F[te[i], 9], "x_sparsity": F[te[i], 10],
                               "chosen": int(S.predict(v2, F[te[i]])), "best": int(np.argmin(T[te[i]])),
                               "regret": float(T[te[i], S.predict(v2, F[te[i]])] / T[te[i]].min())} for i in worst]
    S.write_bundle(a.out, v2, hardware_tag="B200-trained-schema2-workload-per-pattern")
    out["samples"], out["train"], out["test"] = len(F), int(ntr), int(len(te))
    out["nodes_v2"] = {t: len(v2[t]["feature"]) for t in v2}
    Path(a.report).write_text(json.dumps(out, indent=1))
    print(json.dumps(out, indent=1))
    print("wrote", a.out)


if __name__ == "__main__":
    main()
