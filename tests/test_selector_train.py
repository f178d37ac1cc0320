"""CPU: selector training pipeline: labels from timings,
CART grid search, cost-sensitive weights, model file round trip, cascade."""
import numpy as np

from paper_2006_16767_b200 import selector as S


def test_labels_from_times_spec_309():
    # argmin kernel 1 (spmv_lb) -> pattern SpMV, workload LB; write-back from col kernels
    t = [5, 1, 6, 7, 9, 8, 10, 11]
    assert S.labels_from_times(t) == (2, 1, 1)
    t = [9, 9, 9, 9, 1, 2, 3, 0.5]  # col_lb_sort best
    assert S.labels_from_times(t) == (0, 1, 1)
    t = [9, 9, 2, 3, 4, 5, 6, 7]    # row_direct
    assert S.labels_from_times(t) == (1, 0, 0)


def test_separable_single_class_and_xor():
    rng = np.random.default_rng(0)
    X = np.zeros((200, 13))
    X[:, 10] = rng.random(200)
    y = (X[:, 10] > 0.3).astype(int)
    tree, _ = S.train_tree(X, y, S.MASKS["pattern"])
    assert tree["feature"][0] == 10 and len(tree["feature"]) == 3  # depth-1
    assert X[y == 0, 10].max() <= tree["threshold"][0] < X[y == 1, 10].min()
    tree, _ = S.train_tree(X, np.ones(200, int), S.MASKS["pattern"])
    assert tree["feature"] == [-1] and tree["leaf"] == [1]  # single class -> leaf
    X2 = np.zeros((400, 13))
    X2[:, 9] = rng.random(400)
    X2[:, 10] = rng.random(400)
    yx = ((X2[:, 9] > 0.5) ^ (X2[:, 10] > 0.5)).astype(int)
    tree, score = S.train_tree(X2, yx, S.MASKS["pattern"])
    pred = np.array([S.predict({"pattern": tree, "workload": S.leaf(0), "writeback": S.leaf(0)}, f) for f in X2])
    # pattern class 0 -> col kernels (index 4), class 1 -> row kernels (index 2)
    acc = np.mean((pred == 2) == (yx == 1))
    assert acc > 0.95 and score > 0.9  # XOR needs depth >= 2


def test_cost_sensitive_weights_follow_expensive_mistakes():
    # the label alternates with density, but one class is cheap to get wrong:
    # cost-weighted CART must prefer the class whose misses are expensive
    X = np.zeros((100, 13))
    X[:, 8] = 0.9  # same matrix (workload tree sees matrix features only)
    T = []
    for i in range(100):
        if i % 2:  # LB wins big
            T.append([10.0, 1.0, 20, 20, 20, 20, 20, 20])
        else:      # direct wins by a hair
            T.append([1.0, 1.05, 20, 20, 20, 20, 20, 20])
    T = np.array(T)
    lab = np.array([S.labels_from_times(t) for t in T])
    cost = np.array([S.costs_from_times(t) for t in T])
    tree, _ = S.train_tree(X, lab[:, 1], S.MASKS["workload"], cost=cost[:, 1])
    assert tree["feature"] == [-1] and tree["leaf"] == [1]


def test_bundle_round_trip_and_cascade(tmp_path):
    trees = S.default_trees()
    p = tmp_path / "b.txt"
    S.write_bundle(p, trees, "test")
    assert S.read_bundle(p) == trees
    rng = np.random.default_rng(1)
    for _ in range(1000):  # SPEC.md:365 prediction replay
        f = rng.random(13) * 10
        assert S.predict(S.read_bundle(p), f) == S.predict(trees, f)
