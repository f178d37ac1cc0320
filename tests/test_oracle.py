"""CPU: pins the C oracle (oracle/adaspmv_oracle.c) against the reference.

1. Golden fixtures made by the reference itself (tests/golden/make_golden.py,
   oracle/_ref) -- always run; they travel with the repo.
2. Live comparison with oracle/_ref when it is built (property test over
   random inputs).
3. SPEC.md known-answer examples for the SPEC-only functions (features,
   Gini, tree routing, BFS), which have no reference code.
"""
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2006_16767_b200 import synth

GOLD = Path(__file__).resolve().parent / "golden"


def _cases(dt):
    z = np.load(GOLD / f"kernels_{np.dtype(dt).name}.npz")
    for c in range(int(z["ncases"][0])):
        p = f"c{c}_"
        yield c, {k[len(p):]: z[k] for k in z.files if k.startswith(p)}, p, z


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
def test_port_matches_reference_golden(port, dt):
    tol = 1e-12 if dt == np.float64 else 1e-5
    n = 0
    for c, g, p, z in _cases(dt):
        rows, cols = (int(v) for v in g["dims"])
        ro, ci, vals = g["ro"], g["ci"], g["vals"]
        # structure: csr_to_csc (sparse.hpp:157-178) bit-exact
        co, ri, cv = port.csr_to_csc(rows, cols, ro, ci, vals)
        assert np.array_equal(co, g["co"]) and np.array_equal(ri, g["ri"]) and cv.tobytes() == g["cv"].tobytes()
        xi, xv = g["xi"], g["xv"]
        xd = port.sparse_to_dense(cols, xi, xv)
        # oracle (kernels.hpp:197-209) bit-exact
        assert port.reference_multiply(rows, ro, ci, vals, xd).tobytes() == g["y_oracle"].tobytes()
        assert port.effective_nnz(co, xi) == int(g["eff"][0])
        bound = port.reference_multiply(rows, ro, ci, np.abs(vals).astype(np.float64), np.abs(xd).astype(np.float64))
        for w in (1, 3):
            for k in range(8):
                q = f"k{k}_w{w}_"
                kind, y = port.run_kernel(k, rows, cols, ro, ci, vals, (co, ri, cv), x_sparse=(xi, xv), workers=w)
                yd_ref, yi_ref, yv_ref = g[q + "yd"], g[q + "yi"], g[q + "yv"]
                if kind == "dense":
                    # deterministic paths (single simulated order) are bit-exact
                    # with the reference built with -ffp-contract=off
                    if k <= 3 or w == 1:
                        assert y.tobytes() == yd_ref.tobytes(), (c, k, w)
                    else:
                        assert np.all(np.abs(y - yd_ref) <= tol * bound + 1e-300)
                    yi_p, yv_p = port.dense_to_sparse(y)
                else:
                    yi_p, yv_p = y
                assert np.array_equal(yi_p, yi_ref), (c, k, w)
                assert np.all(np.abs(yv_p - yv_ref) <= tol * bound[yi_ref] + 1e-300), (c, k, w)
                # counters (kernels.hpp:107-111): values_read == nnz_s on Row/Col paths
                cnt = g[q + "cnt"]
                if k >= 2:
                    assert int(cnt[0]) == int(g["eff"][0]), (c, k, w)
                if k in (5, 7):
                    assert int(cnt[1]) == int(g["eff"][0])
                n += 1
    assert n >= 300


def test_prims_golden(port):
    z = np.load(GOLD / "prims.npz")
    for i in range(int(z["npart"][0])):
        t, w = (int(v) for v in z[f"part{i}_meta"])
        assert np.array_equal(port.make_partition(z[f"part{i}_off"], t, w), z[f"part{i}_out"])
    for p, e in zip(z["seg_pos"], z["seg_out"]):
        assert port.segment_of(z["seg_off"], p) == e
    idx, val = port.dense_to_sparse(z["d2s_in"])
    assert np.array_equal(idx, z["d2s_idx"]) and val.tobytes() == z["d2s_val"].tobytes()
    assert np.array_equal(port.build_bitmask_dense(z["d2s_in"]), z["mask_dense"])
    assert np.array_equal(port.build_bitmask_sparse(201, z["mask_sparse_idx"]), z["mask_sparse"])
    si, sv = port.sort_reduce_pairs(z["srp_rows"], z["srp_vals"])
    assert np.array_equal(si, z["srp_idx"]) and np.array_equal(sv, z["srp_val"])


def test_spec_known_answers(port):
    # partition examples
    p = port.make_partition([0, 0, 0, 9, 10], 10, 2)
    assert p.tolist() == [[0, 5, 2, 3], [5, 10, 2, 4]]
    p = port.make_partition(list(range(8)), 7, 3)
    assert [(a, b) for a, b, _, _ in p.tolist()] == [(0, 2), (2, 4), (4, 7)]
    # 3x3 rows {(0:2),(1:3),(0:1,2:4)} x ones -> [2,3,5]
    y = port.reference_multiply(3, [0, 1, 2, 4], [0, 1, 0, 2], np.array([2., 3., 1., 4.]), np.ones(3))
    assert y.tolist() == [2.0, 3.0, 5.0]
    # sort_reduce_pairs [(2,1),(0,2),(2,3)] -> {0:2, 2:4}
    i, v = port.sort_reduce_pairs([2, 0, 2], np.array([1., 2., 3.]))
    assert i.tolist() == [0, 2] and v.tolist() == [2.0, 4.0]
    # Gini
    assert port.gini([3, 3, 3, 3]) == 0.0
    assert port.gini([0, 0, 0, 4]) == 0.75
    rng = np.random.default_rng(0)
    for _ in range(200):
        d = rng.integers(0, 50, size=int(rng.integers(1, 200)))
        assert abs(port.gini(d) - port.gini_pairwise(d)) <= 1e-12
        assert abs(port.gini(d * 7) - port.gini(d)) <= 1e-12          # scale invariant
        assert port.gini(rng.permutation(d)) == port.gini(d)         # permutation invariant
        assert -1e-15 <= port.gini(d) <= (len(d) - 1) / len(d) + 1e-15
    # matrix features 4x8 degrees [1,5,2,2]
    f = port.matrix_features(4, 8, [0, 1, 6, 8, 10])
    assert f[3] == 5 and f[4] == 1 and f[5] == 2.5 and f[6] == 0.5
    f = port.matrix_features(5, 5, list(range(6)))  # identity: var 0, gc 0
    assert f[7] == 0.0 and f[8] == 0.0
    # path graph BFS 0-1-2-3 -> [0,1,2,3], 4 iterations
    co = np.array([0, 1, 3, 5, 6])
    ri = np.array([1, 0, 2, 1, 3, 2])
    lv, nl = port.bfs_queue(4, co, ri, 0)
    assert lv.tolist() == [0, 1, 2, 3] and nl == 4
    # tree routing: value <= threshold -> left
    f13 = np.zeros(13)
    f13[10] = 0.3
    k = port.tree_predict([10, -1, -1], [0.3, 0, 0], [1, -1, -1], [2, -1, -1], [-1, 7, 9], f13)
    assert k == 7
    f13[10] = 0.31
    assert port.tree_predict([10, -1, -1], [0.3, 0, 0], [1, -1, -1], [2, -1, -1], [-1, 7, 9], f13) == 9


needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (reference not mounted)")


@needs_ref
@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
def test_port_vs_reference_live_property(port, dt):
    """SPEC.md:189 oracle equivalence over random shapes <= 500, all densities."""
    ref = O.Ref(dt)
    ref.set_threads(3)
    tol = 1e-12 if dt == np.float64 else 1e-5
    rng = np.random.default_rng(42 if dt == np.float64 else 43)
    cases = 0
    for t in range(130):
        r = int(rng.integers(1, 200))
        c = int(rng.integers(1, 200))
        d = float(rng.choice([0.0, 0.01, 0.05, 0.3, 1.0]))
        rows, cols, ro, ci, vals = synth.random_csr(r, c, d, seed=t, dtype=dt)
        M = ref.matrix(rows, cols, ro, ci, vals)
        _, _, _, co, ri, cv = M.export()
        nx = int(rng.integers(0, cols + 1))
        xi, xv = synth.sparse_vector(cols, nx, seed=t, dtype=dt)
        xd = port.sparse_to_dense(cols, xi, xv)
        bound = port.reference_multiply(rows, ro, ci, np.abs(vals).astype(np.float64), np.abs(xd).astype(np.float64))
        w = int(rng.integers(1, 9))
        for k in range(8):
            yd, (yi, yv), _ = M.run_kernel(k, x_sparse=(xi, xv), workers=w)
            kind, y = port.run_kernel(k, rows, cols, ro, ci, vals, (co, ri, cv), x_sparse=(xi, xv), workers=w)
            if kind == "dense":
                assert np.all(np.abs(y.astype(np.float64) - yd) <= tol * bound + 1e-300), (t, k)
            else:
                assert np.array_equal(y[0], yi), (t, k)
                assert np.all(np.abs(y[1] - yv) <= tol * bound[yi] + 1e-300), (t, k)
            cases += 1
    assert cases >= 1000


@needs_ref
def test_reference_loader_matches_golden(tmp_path):
    z = np.load(GOLD / "mm_cases.npz")
    ref = O.Ref(np.float64)
    for i in range(int(z["nmm"][0])):
        p = tmp_path / f"m{i}.mtx"
        p.write_text(str(z[f"mm{i}_text"]))
        M = ref.load_matrix(p)
        ro, ci, cv, *_ = M.export()
        assert np.array_equal(ro, z[f"mm{i}_ro"]) and np.array_equal(ci, z[f"mm{i}_ci"])
        assert cv.tobytes() == z[f"mm{i}_v"].tobytes()
