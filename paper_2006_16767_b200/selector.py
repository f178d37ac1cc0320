"""Selector model files: writing / training the three-tree
SelectorBundle that the C++ runtime evaluates (csrc/selector.cpp).

Model file (text form of SPEC.md:383's schema):

    adaspmv-bundle 1
    hardware_tag <tag>
    feature_order_hash <hex>                      # FNV-1a of the frozen order
    tree <pattern|workload|writeback> mask <u32> nodes <N>
    <feature> <threshold %.17g> <left> <right> <leaf>    # N lines, leaf: feature -1
    ... (3 trees) ...
    end

Classes: pattern {0 ColSpMSpV, 1 RowSpMSpV, 2 SpMV} (kernels.hpp:34),
workload {0 Direct, 1 LoadBalanced}, write-back {0 Atomic, 1 Sort}.
Feature masks: pattern all 13, workload ids 0-8, write-back
{0,1,2,9,10,11,12}.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np

FEATURES = ("m", "n", "nnz", "max_row", "min_row", "avg_row", "relative_range", "var_nnz_row",
            "gc", "nnz_x", "x_sparsity", "nnz_s", "m_sparsity")
MASKS = {"pattern": 0x1FFF, "workload": 0x1FF,
         "writeback": (1 << 0) | (1 << 1) | (1 << 2) | (1 << 9) | (1 << 10) | (1 << 11) | (1 << 12)}
TARGETS = ("pattern", "workload", "writeback")
DEFAULT_PATH = Path(__file__).resolve().parent / "selector" / "b200_bundle.txt"


def feature_order_hash() -> str:
    h = 1469598103934665603
    for ch in ",".join(FEATURES).encode():
        h ^= ch
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def leaf(c: int) -> dict:
    return {"feature": [-1], "threshold": [0.0], "left": [-1], "right": [-1], "leaf": [int(c)]}


def write_bundle(path, trees: dict, hardware_tag: str = "B200") -> None:
    """trees: {"pattern": nodes, "workload": nodes, "writeback": nodes}; with a
    "workload_col" tree the file is schema 2 (selector.cpp)."""
    v2 = "workload_col" in trees
    lines = [f"adaspmv-bundle {2 if v2 else 1}", f"hardware_tag {hardware_tag}",
             f"feature_order_hash {feature_order_hash()}"]
    for t in TARGETS + (("workload_col",) if v2 else ()):
        nd = trees[t]
        n = len(nd["feature"])
        lines.append(f"tree {t} mask {(MASKS_V2 if v2 else MASKS)[t]} nodes {n}")
        for i in range(n):
            lines.append(f"{int(nd['feature'][i])} {float(nd['threshold'][i]):.17g} {int(nd['left'][i])} "
                         f"{int(nd['right'][i])} {int(nd['leaf'][i])}")
    lines.append("end")
    Path(path).write_text("\n".join(lines) + "\n")


def read_bundle(path) -> dict:
    toks = Path(path).read_text().split()
    assert toks[0] == "adaspmv-bundle"
    i = 6
    trees = {}
    for _ in range(4 if toks[1] == "2" else 3):
        _, target, _, mask, _, n = toks[i:i + 6]
        i += 6
        n = int(n)
        nd = {"feature": [], "threshold": [], "left": [], "right": [], "leaf": []}
        for _ in range(n):
            f, th, lft, rgt, lf = toks[i:i + 5]
            i += 5
            nd["feature"].append(int(f))
            nd["threshold"].append(float(th))
            nd["left"].append(int(lft))
            nd["right"].append(int(rgt))
            nd["leaf"].append(int(lf))
        trees[target] = nd
    return trees


def predict(trees: dict, f13) -> int:
    """Host mirror of the cascade -> KernelId::index().
    Schema v2 (optional "workload_col" tree): the ColSpMSpV pattern reads its
    own workload tree, the row patterns the "workload" one."""
    def walk(nd):
        i = 0
        while nd["feature"][i] >= 0:
            i = nd["left"][i] if f13[nd["feature"][i]] <= nd["threshold"][i] else nd["right"][i]
        return nd["leaf"][i]
    p = walk(trees["pattern"])
    lb = walk(trees["workload_col"] if p == 0 and "workload_col" in trees else trees["workload"])
    if p == 2:
        return lb
    if p == 1:
        return 2 + lb
    return 4 + 2 * lb + walk(trees["writeback"])


def default_trees() -> dict:
    """Hand-set cascade used until a B200-trained bundle exists: cheap
    features first."""
    pattern = {  # m_sparsity (12) <= 0.02 -> Col; <= 0.35 -> Row; else SpMV
        "feature": [12, -1, 12, -1, -1], "threshold": [0.02, 0, 0.35, 0, 0],
        "left": [1, -1, 3, -1, -1], "right": [2, -1, 4, -1, -1], "leaf": [-1, 0, -1, 1, 2]}
    workload = {  # Gini of row degrees (8) <= 0.5 -> Direct
        "feature": [8, -1, -1], "threshold": [0.5, 0, 0], "left": [1, -1, -1],
        "right": [2, -1, -1], "leaf": [-1, 0, 1]}
    writeback = {  # nnz_s (11) <= 4096 -> Sort (single-CTA path) else Atomic
        "feature": [11, -1, -1], "threshold": [4096.0, 0, 0], "left": [1, -1, -1],
        "right": [2, -1, -1], "leaf": [-1, 1, 0]}
    return {"pattern": pattern, "workload": workload, "writeback": writeback}


# --------------------------------------------------------------------------
# training: labels from measured kernel times
# --------------------------------------------------------------------------
def labels_from_times(times8) -> tuple[int, int, int]:
    """pattern of the argmin kernel; workload = faster
    distribution within that pattern; write-back = faster write-back among the
    four ColSpMSpV kernels (best over both workloads)."""
    t = np.asarray(times8, np.float64)
    k = int(np.argmin(t))
    pat = 2 if k <= 1 else (1 if k <= 3 else 0)
    if pat == 2:
        wl = int(t[1] < t[0])
    elif pat == 1:
        wl = int(t[3] < t[2])
    else:
        wl = int(min(t[6], t[7]) < min(t[4], t[5]))
    wb = int(min(t[5], t[7]) < min(t[4], t[6]))
    return pat, wl, wb


def _export_sklearn(clf, mask: int) -> dict:
    tr = clf.tree_
    n = tr.node_count
    nd = {"feature": [], "threshold": [], "left": [], "right": [], "leaf": []}
    cls = clf.classes_
    for i in range(n):
        if tr.children_left[i] < 0:
            nd["feature"].append(-1)
            nd["threshold"].append(0.0)
            nd["left"].append(-1)
            nd["right"].append(-1)
            nd["leaf"].append(int(cls[int(np.argmax(tr.value[i][0]))]))
        else:
            f = int(tr.feature[i])
            assert mask & (1 << f)
            nd["feature"].append(f)
            nd["threshold"].append(float(tr.threshold[i]))
            nd["left"].append(int(tr.children_left[i]))
            nd["right"].append(int(tr.children_right[i]))
            nd["leaf"].append(-1)
    return nd


def costs_from_times(times8) -> tuple[float, float, float]:
    """Relative cost of getting each tree's label wrong for one sample:
    (time of the alternative / time of the label) - 1, averaged over the
    alternatives for the 3-class pattern tree.  Used as CART sample weights
    (cost-sensitive training), so that the trees spend their splits where a
    wrong choice is expensive rather than where classes merely alternate."""
    t = np.asarray(times8, np.float64)
    per_pat = {2: min(t[0], t[1]), 1: min(t[2], t[3]), 0: min(t[4:8])}
    pat, wl, wb = labels_from_times(t)
    best = per_pat[pat]
    c_pat = float(np.mean([per_pat[p] / best - 1.0 for p in per_pat if p != pat]))
    if pat == 2:
        pair = (t[0], t[1])
    elif pat == 1:
        pair = (t[2], t[3])
    else:
        pair = (min(t[4], t[5]), min(t[6], t[7]))
    c_wl = float(pair[1 - wl] / pair[wl] - 1.0)
    atomic, sort = min(t[4], t[6]), min(t[5], t[7])
    c_wb = float((atomic / sort if wb else sort / atomic) - 1.0)
    return c_pat, c_wl, c_wb


def train_tree(X, y, mask: int, max_depths=range(1, 11), folds: int = 5, seed: int = 0,
               cost=None):
    """CART with grid search over depth [1,10] x class_weight {balanced,
    uniform} and k-fold CV.  Features
    outside `mask` are hidden from the tree.  With `cost` (per-sample
    misclassification cost), samples are weighted by it and the CV score is
    the cost-weighted accuracy; ties go to the smaller depth."""
    from sklearn.model_selection import StratifiedKFold
    from sklearn.tree import DecisionTreeClassifier

    X = np.asarray(X, np.float64).copy()
    y = np.asarray(y).astype(int)
    cols = [i for i in range(13) if mask & (1 << i)]
    Xm = np.zeros_like(X)
    Xm[:, cols] = X[:, cols]  # constant (zeroed) features are never split on
    if len(np.unique(y)) == 1:
        return leaf(int(y[0])), 1.0
    w = np.ones(len(y)) if cost is None else np.clip(np.asarray(cost, np.float64), 1e-3, 10.0)
    counts = np.bincount(y)
    k = max(2, min(folds, int(np.min(counts[counts > 0]))))
    cv = StratifiedKFold(n_splits=k, shuffle=True, random_state=seed)
    splits = list(cv.split(Xm, y))
    best = None
    for depth in max_depths:
        for cw in ("balanced", None):
            score = 0.0
            for tr, te in splits:
                clf = DecisionTreeClassifier(max_depth=depth, class_weight=cw, random_state=seed)
                clf.fit(Xm[tr], y[tr], sample_weight=w[tr])
                score += float(np.sum(w[te] * (clf.predict(Xm[te]) == y[te])) / np.sum(w[te]))
            score /= len(splits)
            if best is None or score > best[0] + 1e-12:
                best = (score, depth, cw)
    clf = DecisionTreeClassifier(max_depth=best[1], class_weight=best[2], random_state=seed)
    clf.fit(Xm, y, sample_weight=w)
    return _export_sklearn(clf, mask), float(best[0])


def train_bundle(features, times, seed: int = 0, cost_sensitive: bool = True) -> tuple[dict, dict]:
    """features: [S,13]; times: [S,8] seconds -> (trees, cv scores)."""
    F = np.asarray(features, np.float64)
    lab = np.array([labels_from_times(t) for t in times])
    cst = np.array([costs_from_times(t) for t in times]) if cost_sensitive else None
    trees, scores = {}, {}
    for j, t in enumerate(TARGETS):
        trees[t], scores[t] = train_tree(F, lab[:, j], MASKS[t], seed=seed,
                                         cost=None if cst is None else cst[:, j])
    return trees, scores


# Schema v2: feature masks of the per-family workload trees (vector features
# allowed: the column distribution depends on the frontier's degrees)
MASKS_V2 = {"pattern": 0x1FFF, "workload": 0x1FFF, "workload_col": 0x1FFF, "writeback": MASKS["writeback"]}


def train_bundle_v2(features, times, seed: int = 0) -> tuple[dict, dict]:
    """Schema v2: pattern + write-back as train_bundle (cost-sensitive); the
    workload decision split by pattern family, each tree trained on every
    sample with its CONDITIONAL label (faster distribution within the family,
    so a pattern mistake still gets a good distribution) and cost."""
    F = np.asarray(features, np.float64)
    t = np.asarray(times, np.float64)
    lab = np.array([labels_from_times(x) for x in t])
    cst = np.array([costs_from_times(x) for x in t])
    trees, scores = {}, {}
    trees["pattern"], scores["pattern"] = train_tree(F, lab[:, 0], MASKS_V2["pattern"], seed=seed, cost=cst[:, 0])
    trees["writeback"], scores["writeback"] = train_tree(F, lab[:, 2], MASKS_V2["writeback"], seed=seed,
                                                         cost=cst[:, 2])
    # row family: direct vs LB of the better row pattern of the sample
    rd = np.minimum(t[:, 0], t[:, 2])
    rl = np.minimum(t[:, 1], t[:, 3])
    y_row = (rl < rd).astype(int)
    c_row = np.maximum(rd, rl) / np.minimum(rd, rl) - 1.0
    trees["workload"], scores["workload"] = train_tree(F, y_row, MASKS_V2["workload"], seed=seed, cost=c_row)
    cd = np.minimum(t[:, 4], t[:, 5])
    cl = np.minimum(t[:, 6], t[:, 7])
    y_col = (cl < cd).astype(int)
    c_col = np.maximum(cd, cl) / np.minimum(cd, cl) - 1.0
    trees["workload_col"], scores["workload_col"] = train_tree(F, y_col, MASKS_V2["workload_col"], seed=seed,
                                                               cost=c_col)
    return trees, scores


if __name__ == "__main__":
    DEFAULT_PATH.parent.mkdir(parents=True, exist_ok=True)
    if not DEFAULT_PATH.exists():
        write_bundle(DEFAULT_PATH, default_trees(), "B200-default")
        print("wrote", DEFAULT_PATH)
