"""Pins the numpy oracle (oracle/figaro_np.py) to the reference's own known
answers (restated numbers from proj/tests/*.cpp) and to the golden fixtures
written by the compiled reference (tests/golden, make_golden.py).  CPU only."""
import math

import numpy as np
import pytest

from oracle import figaro_np as fo
from paper_2204_00525_b200 import fgdb
from tests.helpers import golden_stems, r_distance, rel_fro
from tests.conftest import golden

S2 = math.sqrt(2.0)


def test_givens_coeffs_pins():
    # test_givens.cpp:27-42
    c, s, r = fo.givens_coeffs(3.0, 4.0)
    assert c == pytest.approx(0.6, rel=1e-14) and s == pytest.approx(-0.8, rel=1e-14)
    assert r == pytest.approx(5.0, rel=1e-14)
    assert fo.givens_coeffs(-2.5, 0.0) == (1.0, 0.0, -2.5)
    assert fo.givens_coeffs(0.0, 1.0) == (0.0, -1.0, 1.0)


def test_head_tail_small():
    # test_givens.cpp:89-136
    a = np.array([[3.0, 1.0], [1.0, 7.0]])
    h = fo.head(a)
    assert h[0] == pytest.approx(4 / S2, rel=1e-14) and h[1] == pytest.approx(8 / S2, rel=1e-14)
    t = fo.tail(a)
    assert t.shape == (1, 2)
    assert t[0, 0] == pytest.approx(-2 / S2, rel=1e-14) and t[0, 1] == pytest.approx(6 / S2, rel=1e-14)
    stack = np.vstack([h, t])
    np.testing.assert_allclose(stack.T @ stack, [[10, 10], [10, 50]], rtol=1e-12)
    assert np.array_equal(fo.head(np.array([[2.0, -1.0, 0.5]])), [2.0, -1.0, 0.5])
    assert fo.tail(np.array([[1.0, 2.0]])).shape[0] == 0
    with pytest.raises(fo.error):
        fo.head(np.zeros((0, 2)))


def test_head_repeated_value():
    # test_givens.cpp:104-113
    for q in (2, 5, 9):
        assert fo.head(np.full((q, 1), 1.5))[0] == pytest.approx(1.5 * math.sqrt(q), rel=1e-14)


def test_streaming_tail_equals_naive():
    # test_givens.cpp:150-155 (oracle support.hpp:74-88)
    rng = np.random.default_rng(1)
    a = rng.uniform(-3, 3, (12, 3))
    naive = np.zeros((11, 3))
    for j in range(1, 12):
        for c in range(3):
            pre = 0.0
            for i in range(j):
                pre += a[i, c]
            sj = math.sqrt(j)
            naive[j - 1, c] = (sj * a[j, c] - pre / sj) / math.sqrt(j + 1)
    assert np.array_equal(fo.tail(a), naive)


def test_generalized_pins():
    # test_givens.cpp:157-174
    assert fo.generalized_head(np.array([[1.0], [1.0]]), [3.0, 4.0])[0] == pytest.approx(1.4, rel=1e-14)
    rng = np.random.default_rng(31)
    a = rng.uniform(-3, 3, (8, 3))
    ones = [1.0] * 8
    assert np.array_equal(fo.generalized_head(a, ones), fo.head(a))
    assert np.array_equal(fo.generalized_tail(a, ones), fo.tail(a))
    with pytest.raises(fo.error):
        fo.generalized_head(np.array([[1.0], [1.0]]), [1.0])
    with pytest.raises(fo.error):
        fo.generalized_head(np.array([[1.0], [1.0]]), [1.0, -2.0])


def test_generalized_homogeneity_and_gram():
    # test_givens.cpp:176-220
    rng = np.random.default_rng(37)
    a = rng.uniform(-3, 3, (6, 2))
    v = rng.uniform(0.1, 4.0, 6)
    h, t = fo.generalized_head(a, v), fo.generalized_tail(a, v)
    np.testing.assert_allclose(fo.generalized_head(a * 2.0, v), 2 * h, rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(fo.generalized_tail(a * -3.0, v * 2.0), -3 * t, rtol=1e-14, atol=1e-14)
    # The generalized transform is orthogonal with first row v/||v||.
    stack = np.vstack([h, t])
    assert rel_fro(stack.T @ stack, a.T @ a) <= 1e-12


def _counts_for(stem):
    db = fgdb.read_fgdb(golden(stem + ".fgdb"))
    rels, root, parent = fo.from_fgdb(db)
    rels = [fo.canonicalize(r) for r in rels]
    tree = fo.build_join_tree(rels, root, parent)
    return fo.compute_counts(rels, tree), rels, tree


def test_counts_by_hand():
    # test_counts.cpp:35-60
    c, _, _ = _counts_for("hand_st")
    assert list(c[0].phi_circ.values()) == [3, 2]
    assert list(c[1].phi_circ.values()) == [2, 1]
    assert list(c[0].full_join_size.values()) == [6, 2]
    assert sum(c[0].full_join_size.values()) == 8


def test_counts_single_and_chain():
    # test_counts.cpp:62-75, 107-138
    c, _, _ = _counts_for("hand_single")
    assert list(c[0].phi_circ.values()) == [1, 1]
    assert c[0].full_join_size == c[0].rows_per_key
    c, _, _ = _counts_for("hand_chain")
    assert c[1].phi_up == {(1,): 2, (2,): 1}


def test_counts_four_relation():
    # test_counts.cpp:77-105
    c, rels, tree = _counts_for("hand_four")
    assert c[3].phi_circ[(1,)] == 13
    assert c[2].phi_circ[(1,)] == 19
    assert c[0].full_join_size == c[0].theta_down
    for leaf in (2, 3):
        for key, n in c[leaf].rows_per_key.items():
            xp = fo.project_key(key, rels[leaf].key_attrs, tree.parent_attrs[leaf])
            assert c[leaf].phi_down[xp] == n
            assert c[leaf].phi_circ[key] == c[leaf].phi_up[xp]


def test_counts_errors():
    # test_counts.cpp:150-194
    mk = fo.Relation
    s = mk("S", ["X"], ["a"], [[1], [2]], [[1.0], [2.0]])
    t = mk("T", ["X"], ["b"], [[1]], [[1.0]])
    with pytest.raises(fo.integrity_error):
        fo.compute_counts([s, t], fo.build_join_tree([s, t], 0, [-1, 0]))
    s = mk("S", ["X"], ["a"], [[1]], [[1.0]])
    t = mk("T", ["X"], ["b"], [[1], [2]], [[1.0], [2.0]])
    with pytest.raises(fo.integrity_error):
        fo.compute_counts([s, t], fo.build_join_tree([s, t], 0, [-1, 0]))
    rels = [mk(f"S{i}", ["X"], [f"y{i}"], np.ones((300, 1), dtype=np.int64),
               np.arange(300.0).reshape(300, 1)) for i in range(8)]
    with pytest.raises(fo.size_error):
        fo.compute_counts(rels, fo.build_join_tree(rels, 0, [-1] + [0] * 7))


def test_cartesian_and_child_pins():
    # test_figaro.cpp:55-74 and 98-138
    db = fgdb.read_fgdb(golden("hand_cartesian.fgdb"))
    res = fo.run_pipeline(*fo.from_fgdb(db))
    g = fo.dense_r0(res.r0, 2)
    np.testing.assert_allclose(g.T @ g, [[10, 12], [12, 20]], rtol=1e-12)
    assert res.r0_rows <= 4
    db = fgdb.read_fgdb(golden("hand_child.fgdb"))
    rels, root, parent = fo.from_fgdb(db)
    rels = [fo.canonicalize(r) for r in rels]
    tree = fo.build_join_tree(rels, root, parent)
    lay = fo.Layout(rels, tree)
    counts = fo.compute_counts(rels, tree)
    assert counts[1].phi_circ[(1,)] == 4
    out, keys, data, scales = fo.figaro_node(rels, tree, lay, counts, 1)
    assert scales[0] == pytest.approx(S2, rel=1e-14)
    assert data[0, 0] == pytest.approx(4 / S2, rel=1e-14)
    assert out[0].rows[0, 0] == pytest.approx(2 * 2 / S2, rel=1e-12)


def test_householder_pin():
    # test_postprocess.cpp:133-140
    a = np.array([[1.0, 1.0], [1.0, 3.0], [2.0, 1.0], [2.0, 3.0]])
    r = fo.normalize_signs(fo.householder_r(a))
    np.testing.assert_allclose(r, [[math.sqrt(10), 12 / math.sqrt(10)], [0, math.sqrt(5.6)]],
                               rtol=1e-14)


@pytest.mark.parametrize("stem", golden_stems("rnd_") + golden_stems("hand_") + golden_stems("big_"))
def test_oracle_matches_reference_golden(stem):
    """Counts and key groups bit-exact, R0 blocks bit-exact, R within 1e-12."""
    db = fgdb.read_fgdb(golden(stem + ".fgdb"))
    ref = fgdb.read_fgrs(golden(stem + ".fgrs"))
    res = fo.run_pipeline(*fo.from_fgdb(db))
    assert res.r0_rows == ref.r0_rows
    assert r_distance(res.R, ref.R) <= 1e-12
    for i, nc in enumerate(res.counts):
        rn = ref.nodes[i]
        for name in ("rows_per_key", "theta_down", "full_join_size", "phi_circ"):
            assert list(getattr(nc, name).values()) == getattr(rn, name).tolist(), name
        assert [list(k) for k in nc.rows_per_key] == rn.keys.tolist()
        assert list(nc.phi_down.values()) == rn.phi_down.tolist()
        assert list(nc.phi_up.values()) == rn.phi_up.tolist()
        assert [list(k) for k in nc.phi_down] == rn.pkeys.tolist()
    assert len(res.r0) == len(ref.r0)
    for a, b in zip(res.r0, ref.r0):
        assert (a.node, a.col_begin) == (b.node, b.col_begin)
        assert np.array_equal(a.rows, b.rows)
    import os
    fgrm = golden(stem + ".fgrm")
    if os.path.exists(fgrm):
        assert r_distance(res.R, fgdb.read_fgrm(fgrm)) <= 1e-10


def test_ground_truth_accuracy():
    # acceptance criterion 6 (acceptance_main.cpp:265-287): <= 5e-14 at 512x16
    for stem, bound in (("gt_512x16", 5e-14), ("gt_64x8", 5e-14)):
        db = fgdb.read_fgdb(golden(stem + ".fgdb"))
        rfix = fgdb.read_fgrm(golden(stem + ".rfix.fgrm"))
        res = fo.run_pipeline(*fo.from_fgdb(db))
        n = rfix.shape[0]
        assert rel_fro(fo.normalize_signs(res.R[:n, :n]), fo.normalize_signs(rfix)) <= bound


def test_c1_golden_checksum_and_oracle():
    """The seeded C1 generator still produces the bytes the golden R came from."""
    from paper_2204_00525_b200 import workloads
    from tests.golden.make_golden import db_digest
    db = workloads.config_c1(seed=7)
    with open(golden("c1_seed7.sha256")) as f:
        assert db_digest(db) == f.read().strip()
    ref = fgdb.read_fgrs(golden("c1_seed7.fgrs"))
    assert [n.rows_per_key.tolist() for n in ref.nodes] == [[10] * 1000] * 2
    assert [n.phi_circ.tolist() for n in ref.nodes] == [[10] * 1000] * 2


# ---------------------------------------------------------------- join rows / Q


def _mk(name, ka, da, rows):
    keys = np.array([r[0] for r in rows], dtype=np.int64).reshape(len(rows), len(ka))
    data = np.array([r[1] for r in rows], dtype=np.float64).reshape(len(rows), len(da))
    return fo.Relation(name, ka, da, keys, data)


def test_materialize_join_pins():
    # test_relational.cpp:189-235
    s = _mk("S", [], ["y1"], [([], [1.0]), ([], [2.0]), ([], [3.0])])
    t = _mk("T", [], ["y2"], [([], [4.0]), ([], [5.0])])
    a = fo.join_rows([s, t], fo.build_join_tree([s, t], 0, [-1, 0]))
    assert a.shape == (6, 2)
    np.testing.assert_array_equal(a[:, 0], [1, 1, 2, 2, 3, 3])  # depth-first order
    s = _mk("S", ["X"], ["y", "z"], [([1], [1.0, 2.0]), ([2], [3.0, 4.0])])
    a = fo.join_rows([s], fo.build_join_tree([s], 0, [-1]))
    assert a.shape == (2, 2) and a[0, 0] == 1.0 and a[1, 1] == 4.0
    s = _mk("S", ["X"], ["y"], [([1], [1.0]), ([1], [2.0])])
    t = _mk("T", ["X"], ["z"], [([1], [3.0]), ([1], [4.0]), ([1], [5.0])])
    assert fo.join_rows([s, t], fo.build_join_tree([s, t], 0, [-1, 0])).shape[0] == 6
    s = _mk("S", [], ["y"], [([], [1.0]), ([], [2.0])])
    t = _mk("T", [], ["z"], [([], [3.0]), ([], [4.0])])
    with pytest.raises(fo.size_error):
        fo.join_rows([s, t], fo.build_join_tree([s, t], 0, [-1, 0]), cap=3)


def test_recover_q_pins():
    # test_postprocess.cpp:185-247
    s = _mk("S", [], ["y"], [([], [2.0])])
    a, q = fo.recover_q([s], fo.build_join_tree([s], 0, [-1]), np.array([[2.0]]))
    assert q.shape == (1, 1) and q[0, 0] == pytest.approx(1.0)
    s = _mk("S", [], ["y1"], [([], [1.0]), ([], [2.0])])
    t = _mk("T", [], ["y2"], [([], [1.0]), ([], [3.0])])
    rels = [s, t]
    tree = fo.build_join_tree(rels, 0, [-1, 0])
    R = fo.run_pipeline(rels, 0, [-1, 0]).R
    a, q = fo.recover_q(rels, tree, R)
    assert q.shape[0] == 4
    np.testing.assert_allclose(q.T @ q, np.eye(2), atol=1e-10)
    assert rel_fro(q @ R, a) <= 1e-10
    s = _mk("S", [], ["y", "z"], [([], [1.0, 1.0])])
    with pytest.raises(fo.rank_error):
        fo.recover_q([s], fo.build_join_tree([s], 0, [-1]), np.array([[1.0, 1.0], [0.0, 0.0]]))


@pytest.mark.parametrize("stem", [s for s in golden_stems("hand_") + golden_stems("rnd_")
                                  if __import__("os").path.exists(golden(s + ".fgrq"))])
def test_oracle_recover_q_matches_reference(stem):
    """The restated join order and forward substitution reproduce the
    reference's streamed (a_row, q_row) pairs bit for bit."""
    db = fgdb.read_fgdb(golden(stem + ".fgdb"))
    R = fgdb.read_fgrs(golden(stem + ".fgrs")).R
    A_ref, Q_ref = fgdb.read_fgrq(golden(stem + ".fgrq"))
    rels, root, parent = fo.from_fgdb(db)
    A, Q = fo.recover_q(rels, fo.build_join_tree(rels, root, parent), R, cap=5000)
    np.testing.assert_array_equal(A, A_ref)
    np.testing.assert_array_equal(Q, Q_ref)


@pytest.mark.parametrize("stem,err", [("rnd_15", "rank"), ("rnd_19", "rank"),
                                      ("rnd_10", "size"), ("rnd_4", "size")])
def test_oracle_recover_q_errors(stem, err):
    """The reference raised rank_error / size_error (cap 5000) on these."""
    db = fgdb.read_fgdb(golden(stem + ".fgdb"))
    R = fgdb.read_fgrs(golden(stem + ".fgrs")).R
    rels, root, parent = fo.from_fgdb(db)
    with pytest.raises(fo.rank_error if err == "rank" else fo.size_error):
        fo.recover_q(rels, fo.build_join_tree(rels, root, parent), R, cap=5000)
