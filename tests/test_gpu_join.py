"""Join enumeration and Q = A R^-1 on the GPU (fg_join_size /
fg_materialize_join / fg_recover_q) against the compiled reference's
recover_q output (tests/golden/*.fgrq) and the numpy oracle.

Bars: join rows (A) bit-exact and in the reference's order; Q bit-exact for
the same R (the device uses the reference's unfused operation order); error
taxonomy as the reference (rank_error, size_error at the cap)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import figaro_np as fo  # noqa: E402
from paper_2204_00525_b200 import fgdb, workloads  # noqa: E402
from paper_2204_00525_b200 import figaro as F  # noqa: E402
from tests.conftest import golden  # noqa: E402
from tests.helpers import golden_stems, rel_fro  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def to_rels(db, device):
    out = []
    for r in db.relations:
        keys, data = np.ascontiguousarray(r.keys), np.ascontiguousarray(r.data)
        if device:
            keys, data = torch.from_numpy(keys).cuda(), torch.from_numpy(data).cuda()
        out.append(F.Relation(r.name, r.key_attrs, r.data_attrs, keys, data))
    return out


Q_STEMS = [s for s in golden_stems("hand_") + golden_stems("rnd_")
           if os.path.exists(golden(s + ".fgrq"))]


@pytest.mark.parametrize("device", [True, False])
@pytest.mark.parametrize("stem", Q_STEMS)
def test_recover_q_matches_reference(stem, device):
    db = fgdb.read_fgdb(golden(stem + ".fgdb"))
    R = fgdb.read_fgrs(golden(stem + ".fgrs")).R
    A_ref, Q_ref = fgdb.read_fgrq(golden(stem + ".fgrq"))
    rels = to_rels(db, device)
    tree = F.build_join_tree(rels, db.root, db.parent)
    assert F.join_size(rels, tree, cap=5000) == A_ref.shape[0]
    Rin = torch.from_numpy(R).cuda() if device else R
    A, Q = F.recover_q(rels, tree, Rin, cap=5000)
    if device:
        A, Q = A.cpu().numpy(), Q.cpu().numpy()
    np.testing.assert_array_equal(A, A_ref)
    np.testing.assert_array_equal(Q, Q_ref)
    M = F.materialize_join(rels, tree, cap=5000)
    np.testing.assert_array_equal(M.cpu().numpy() if device else M, A_ref)


@pytest.mark.parametrize("stem,err", [("rnd_15", F.rank_error), ("rnd_19", F.rank_error),
                                      ("rnd_22", F.rank_error), ("rnd_10", F.size_error),
                                      ("rnd_4", F.size_error)])
def test_recover_q_errors_match_reference(stem, err):
    db = fgdb.read_fgdb(golden(stem + ".fgdb"))
    R = fgdb.read_fgrs(golden(stem + ".fgrs")).R
    rels = to_rels(db, False)
    tree = F.build_join_tree(rels, db.root, db.parent)
    with pytest.raises(err):
        F.recover_q(rels, tree, R, cap=5000)


def test_reference_unit_cases():
    """test_relational.cpp:189-235 and test_postprocess.cpp:185-247."""
    def rel(name, ka, da, rows):
        keys = np.array([r[0] for r in rows], dtype=np.int64).reshape(len(rows), len(ka))
        data = np.array([r[1] for r in rows], dtype=np.float64).reshape(len(rows), len(da))
        return F.Relation(name, ka, da, keys, data)

    s = rel("S", [], ["y1"], [([], [1.0]), ([], [2.0]), ([], [3.0])])
    t = rel("T", [], ["y2"], [([], [4.0]), ([], [5.0])])
    tree = F.build_join_tree([s, t], 0, [-1, 0])
    a = F.materialize_join([s, t], tree)
    np.testing.assert_array_equal(a, [[1, 4], [1, 5], [2, 4], [2, 5], [3, 4], [3, 5]])
    with pytest.raises(F.size_error):
        F.materialize_join([s, t], tree, cap=5)
    s = rel("S", ["X"], ["y"], [([1], [1.0]), ([1], [2.0])])
    t = rel("T", ["X"], ["z"], [([1], [3.0]), ([1], [4.0]), ([1], [5.0])])
    assert F.join_size([s, t], F.build_join_tree([s, t], 0, [-1, 0])) == 6
    s = rel("S", [], ["y"], [([], [2.0])])
    _, q = F.recover_q([s], F.build_join_tree([s], 0, [-1]), np.array([[2.0]]))
    assert q.shape == (1, 1) and q[0, 0] == 1.0
    s = rel("S", [], ["y", "z"], [([], [1.0, 1.0])])
    with pytest.raises(F.rank_error):
        F.recover_q([s], F.build_join_tree([s], 0, [-1]), np.array([[1.0, 1.0], [0.0, 0.0]]))


def test_dangling_and_empty():
    """Dangling parent rows yield no join rows (join.hpp:83); an empty
    relation gives an empty join; no reduction is applied."""
    def rel(name, ka, da, keys, data):
        return F.Relation(name, ka, da, np.array(keys, dtype=np.int64).reshape(-1, len(ka)),
                          np.array(data, dtype=np.float64).reshape(-1, len(da)))

    r1 = rel("R1", ["k"], ["x"], [[1], [2], [3], [2]], [[1.0], [2.0], [3.0], [4.0]])
    r2 = rel("R2", ["k"], ["y"], [[2], [2], [3], [9]], [[5.0], [6.0], [7.0], [8.0]])
    rels = [r1, r2]
    tree = F.build_join_tree(rels, 0, [-1, 0])
    a = F.materialize_join(rels, tree)
    ref = fo.join_rows([fo.Relation(r.name, r.key_attrs, r.data_attrs, r.keys, r.data)
                        for r in rels], fo.build_join_tree(
                            [fo.Relation(r.name, r.key_attrs, r.data_attrs, r.keys, r.data)
                             for r in rels], 0, [-1, 0]))
    np.testing.assert_array_equal(a, ref)
    assert a.shape[0] == 5
    e = rel("R2", ["k"], ["y"], np.zeros((0, 1)), np.zeros((0, 1)))
    assert F.join_size([r1, e], F.build_join_tree([r1, e], 0, [-1, 0])) == 0


def _db(src):
    if src.startswith("big_"):
        return fgdb.read_fgdb(golden(src + ".fgdb"))
    cfg, scale = src.split("@")
    return workloads.make(cfg, seed=5, scale=float(scale))


@pytest.mark.parametrize("src", ["C3@0.0005", "C4@0.0005", "C1@0.3"] + golden_stems("big_"))
def test_join_rows_vs_oracle(src):
    """Multi-level trees (C3: a star under a chain; C4: a chain; big_*: the
    reference's random acyclic generator, up to 6 relations), or the same
    size_error at the cap."""
    db = _db(src)
    cap = 300_000
    orels = [fo.Relation(r.name, r.key_attrs, r.data_attrs, r.keys, r.data) for r in db.relations]
    otree = fo.build_join_tree(orels, db.root, db.parent)
    rels = to_rels(db, True)
    tree = F.build_join_tree(rels, db.root, db.parent)
    try:
        A_ref = fo.join_rows(orels, otree, cap=cap)
    except fo.size_error:
        with pytest.raises(F.size_error):
            F.join_size(rels, tree, cap=cap)
        return
    assert F.join_size(rels, tree, cap=cap) == A_ref.shape[0]
    A = F.materialize_join(rels, tree, cap=cap).cpu().numpy()
    np.testing.assert_array_equal(A, A_ref)


def test_q_properties_at_scale():
    """Q^T Q = I and Q R = A on a C2-shaped join of ~1.4M rows (R from the
    GPU pipeline)."""
    db = workloads.make("C2", seed=3, scale=0.005)
    rels = to_rels(db, True)
    tree = F.build_join_tree(rels, db.root, db.parent)
    R = F.run_pipeline(rels, tree, F.PipelineOptions(assume_reduced=True),
                       fetch_counts=False).factor.r
    A, Q = F.recover_q(rels, tree, R, cap=10_000_000)
    assert A.shape[0] == F.join_size(rels, tree, cap=10_000_000)
    n = Q.shape[1]
    qtq = (Q.T @ Q).cpu().numpy()
    assert np.abs(qtq - np.eye(n)).max() <= 1e-10
    assert rel_fro((Q @ R).cpu().numpy(), A.cpu().numpy()) <= 1e-12
