"""Pipeline parity on the GPU through the C ABI against the compiled reference.

Bars (BASELINE.json north_star): segment offsets, keys and all six count
tables bit-exact; R within relative Frobenius 1e-10 after sign normalisation
(rank-deficient references compare R^T R, since R is then not unique).
Sources of truth: tests/golden (written by oracle/_ref/figaro_ref) and, when
the binary is present, fresh runs of oracle/_ref/figaro_ref on seeded inputs.
"""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import figaro_np as fo  # noqa: E402
from paper_2204_00525_b200 import fgdb, workloads  # noqa: E402
from paper_2204_00525_b200 import figaro as F  # noqa: E402
from tests.conftest import REF_BIN, golden  # noqa: E402
from tests.helpers import golden_stems, r_distance  # noqa: E402

R_TOL = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def to_rels(db, device=True, canonical=False):
    out = []
    for r in db.relations:
        keys, data = r.keys, r.data
        if canonical:
            c = fo.canonicalize(fo.Relation(r.name, r.key_attrs, r.data_attrs, keys, data))
            keys, data = c.keys, c.data
        if device:
            keys, data = torch.from_numpy(np.ascontiguousarray(keys)).cuda(), \
                torch.from_numpy(np.ascontiguousarray(data)).cuda()
        out.append(F.Relation(r.name, r.key_attrs, r.data_attrs, keys, data))
    return out


def run_gpu(db, device=True, canonical=False, keep_r0=False, assume_reduced=True, fuse=True):
    rels = to_rels(db, device, canonical)
    tree = F.build_join_tree(rels, db.root, db.parent)
    res = F.run_pipeline(rels, tree, F.PipelineOptions(assume_reduced=assume_reduced),
                         keep_r0=keep_r0, fuse=fuse)
    R = res.factor.r.cpu().numpy() if device else res.factor.r
    return res, R


def check_counts(res, ref):
    for i, nc in enumerate(ref.nodes):
        c = res.counts[i]
        assert np.array_equal(c.group_begin.astype(np.uint64), nc.group_begin), f"segments node {i}"
        assert np.array_equal(c.keys, nc.keys), f"keys node {i}"
        for name in ("rows_per_key", "theta_down", "full_join_size", "phi_circ", "phi_down", "phi_up"):
            assert np.array_equal(getattr(c, name), getattr(nc, name)), f"{name} node {i}"
        assert np.array_equal(c.parent_keys, nc.pkeys), f"parent keys node {i}"


def match_r0(spans, ref_blocks):
    """Each GPU span equals the vertical concatenation of the next
    reference OutBlocks with the same node / col_begin."""
    it = iter(ref_blocks)
    for sp in spans:
        rows = []
        got = 0
        while got < sp.rows.shape[0]:
            b = next(it)
            assert (b.node, b.col_begin, b.rows.shape[1]) == (sp.node, sp.col_begin, sp.rows.shape[1])
            rows.append(b.rows)
            got += b.rows.shape[0]
        ref = np.vstack(rows)
        scale = max(np.abs(ref).max(), 1e-300)
        np.testing.assert_allclose(sp.rows, ref, rtol=0, atol=1e-12 * scale)
    assert next(it, None) is None


GOLD = golden_stems("rnd_") + golden_stems("hand_") + golden_stems("big_")


@pytest.mark.parametrize("stem", GOLD)
@pytest.mark.parametrize("device,fuse", [(True, True), (False, True), (True, False)])
def test_golden_pipeline(stem, device, fuse):
    db = fgdb.read_fgdb(golden(stem + ".fgdb"))
    ref = fgdb.read_fgrs(golden(stem + ".fgrs"))
    res, R = run_gpu(db, device=device, fuse=fuse)
    assert res.r0_rows == ref.r0_rows and res.input_rows == ref.input_rows
    assert r_distance(R, ref.R) <= R_TOL
    check_counts(res, ref)
    if os.path.exists(golden(stem + ".fgrm")):
        assert r_distance(R, fgdb.read_fgrm(golden(stem + ".fgrm"))) <= R_TOL


@pytest.mark.parametrize("stem", GOLD)
def test_golden_r0_elementwise(stem):
    """With canonically pre-sorted input the R0 spans equal the reference
    blocks element-wise (figaro.hpp:166-329 block order)."""
    db = fgdb.read_fgdb(golden(stem + ".fgdb"))
    ref = fgdb.read_fgrs(golden(stem + ".fgrs"))
    res, _ = run_gpu(db, canonical=True, keep_r0=True)
    match_r0(res.r0, ref.r0)


def test_ground_truth_accuracy():
    # acceptance criterion 6: <= 5e-14 at 512x16 against the fixed factor
    for stem in ("gt_512x16", "gt_64x8"):
        db = fgdb.read_fgdb(golden(stem + ".fgdb"))
        rfix = fgdb.read_fgrm(golden(stem + ".rfix.fgrm"))
        _, R = run_gpu(db)
        n = rfix.shape[0]
        assert fo.rel_frobenius_distance(fo.normalize_signs(R[:n, :n]), fo.normalize_signs(rfix)) <= 5e-14


def test_c1_full_golden():
    db = workloads.config_c1(seed=7)
    ref = fgdb.read_fgrs(golden("c1_seed7.fgrs"))
    res, R = run_gpu(db)
    assert r_distance(R, ref.R) <= R_TOL
    check_counts(res, ref)


def run_ref(db, tmp_path, extra=()):
    p = str(tmp_path / "db.fgdb")
    fgdb.write_fgdb(p, db)
    subprocess.run([REF_BIN, "run", p, p + ".rs", *extra], check=True, capture_output=True)
    return fgdb.read_fgrs(p + ".rs")


@pytest.mark.parametrize("cfg,scale", [("C2", 0.01), ("C3", 0.002), ("C4", 0.02), ("C5", 0.005)])
@pytest.mark.parametrize("fuse", [True, False])
def test_configs_vs_reference(cfg, scale, fuse, tmp_path, ref_bin):
    db = workloads.make(cfg, seed=11, scale=scale)
    ref = run_ref(db, tmp_path)
    res, R = run_gpu(db, fuse=fuse)
    assert res.r0_rows == ref.r0_rows
    assert r_distance(R, ref.R) <= R_TOL
    check_counts(res, ref)


@pytest.mark.parametrize("seed", range(200, 215))
def test_random_reference_databases(seed, tmp_path, ref_bin):
    p = str(tmp_path / "rnd.fgdb")
    subprocess.run([ref_bin, "random", str(seed), p, "--max-rows", "2000", "--max-rel", "6",
                    "--key-domain", "30", "--max-cols", "14"], check=True, capture_output=True)
    db = fgdb.read_fgdb(p)
    ref = run_ref(db, tmp_path)
    res, R = run_gpu(db)
    assert r_distance(R, ref.R) <= R_TOL
    check_counts(res, ref)


def test_unreduced_input_is_reduced(tmp_path, ref_bin):
    """assume_reduced=False runs the semi-join reducer (reduce.hpp:47-74)."""
    db = workloads.make("C5", seed=3, scale=0.002)
    rng = np.random.default_rng(0)
    for r in db.relations:  # dangling keys on both sides
        extra = rng.integers(200_000, 200_050, 40).reshape(-1, 1)
        r.keys = np.vstack([r.keys, extra])
        r.data = np.vstack([r.data, rng.standard_normal((40, r.data.shape[1]))])
    ref = run_ref(db, tmp_path, ["--reduce"])
    res, R = run_gpu(db, assume_reduced=False)
    assert res.input_rows == ref.input_rows
    assert r_distance(R, ref.R) <= R_TOL
    check_counts(res, ref)
    with pytest.raises(F.integrity_error):
        run_gpu(db, assume_reduced=True)


def test_errors_match_reference_taxonomy():
    mk = fgdb.RelationData
    k = lambda *v: np.array(v, dtype=np.int64).reshape(-1, 1)  # noqa: E731
    d = lambda n: np.ones((n, 1))  # noqa: E731
    # unreduced (counts.hpp:143-148 / 211-214)
    for a, b in ((k(1, 2), k(1)), (k(1), k(1, 2))):
        db = fgdb.Database([mk("S", ["X"], ["a"], a, d(len(a))), mk("T", ["X"], ["b"], b, d(len(b)))], 0, [-1, 0])
        with pytest.raises(F.integrity_error):
            run_gpu(db)
    # 300^8 > 2^64 (counts.hpp:47-62)
    rels = [mk(f"S{i}", ["X"], [f"y{i}"], np.ones((300, 1), dtype=np.int64),
               np.arange(300.0).reshape(300, 1)) for i in range(8)]
    with pytest.raises(F.size_error):
        run_gpu(fgdb.Database(rels, 0, [-1] + [0] * 7))
    # empty join after reduction (reduce.hpp:49-53)
    db = fgdb.Database([mk("S", ["X"], ["a"], k(1), d(1)), mk("T", ["X"], ["b"], k(2), d(1))], 0, [-1, 0])
    with pytest.raises(F.empty_join_error):
        run_gpu(db, assume_reduced=False)
    # tree errors (join_tree.hpp:72-180)
    db = fgdb.Database([mk("S", ["X"], ["a"], k(1), d(1)), mk("T", ["Y"], ["b"], k(1), d(1))], 0, [-1, 0])
    with pytest.raises(F.tree_error):
        run_gpu(db)
    db = fgdb.Database([mk("S", ["X"], ["a"], k(1), d(1)), mk("T", ["X"], ["a"], k(1), d(1))], 0, [-1, 0])
    with pytest.raises(F.schema_error):
        run_gpu(db)
    # path property (join_tree.hpp:120-153): X held by S and V but not by the
    # relation between them; the reported relation is the reference's (the
    # first holder pair, first gap along the tree path).
    kk = lambda n: np.ones((1, n), dtype=np.int64)  # noqa: E731
    db = fgdb.Database([mk("S", ["X", "Y"], ["a"], kk(2), d(1)), mk("U", ["Y", "Z"], ["b"], kk(2), d(1)),
                        mk("V", ["X", "Z"], ["c"], kk(2), d(1))], 0, [-1, 0, 1])
    with pytest.raises(F.tree_error, match="relation U does not contain it"):
        run_gpu(db)


@pytest.mark.parametrize("cfg,scale", [("C5", 0.003), ("C2", 0.05), ("C3", 0.002),
                                       ("C4", 0.02)])
def test_determinism_and_launch_evidence(cfg, scale):
    """R bit-identical run to run -- including C2, whose own tails take the
    fused heads/tails -> TSQR kernel (static unit -> warp assignment)."""
    db = workloads.make(cfg, seed=5, scale=scale)
    r1, R1 = run_gpu(db)
    Rs = [run_gpu(db)[1] for _ in range(3)]
    for R2 in Rs:
        assert np.array_equal(R1, R2), "R must be bit-identical run to run"
    assert r1.kernels > 10
    if cfg == "C2":
        assert r1.fused_launches == 2


def test_full_size_c2_gram_property():
    """BASELINE-size C2 (32M rows): R^T R equals the join's A^T A computed
    independently from per-key sums (size-independent property)."""
    db = workloads.config_c2(seed=7)
    res, R = run_gpu(db)
    assert res.input_rows == 32_000_000 and res.r0_rows == 31_000_000
    for c in res.counts:
        assert np.all(c.rows_per_key == 16) and np.all(c.phi_circ == 16)
    ata = np.zeros((32, 32))
    blocks = []
    for r in db.relations:
        k = torch.from_numpy(r.keys[:, 0]).cuda()
        x = torch.from_numpy(r.data).cuda()
        sums = torch.zeros((1_000_000, 16), dtype=torch.float64, device="cuda").index_add_(0, k, x)
        blocks.append((x, sums))
    (x1, s1), (x2, s2) = blocks
    ata[:16, :16] = (16 * (x1.T @ x1)).cpu().numpy()
    ata[16:, 16:] = (16 * (x2.T @ x2)).cpu().numpy()
    cross = (s1.T @ s2).cpu().numpy()
    ata[:16, 16:] = cross
    ata[16:, :16] = cross.T
    assert fo.rel_frobenius_distance(R.T @ R, ata) <= 1e-12


def test_cpp_facade_on_reference_types():
    """include/figaro_gpu.hpp bound to the reference's own Relation/JoinTree
    (tests/cpp/facade_parity.cpp, built by oracle/Makefile)."""
    exe = os.path.join(os.path.dirname(REF_BIN), "facade_parity")
    if not os.path.exists(exe):
        pytest.skip("facade_parity not built")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "PASS" in out.stdout


@pytest.mark.parametrize("w1,w2", [(12, 20), (24, 5), (32, 3), (1, 33), (7, 9), (40, 5), (64, 2)])
@pytest.mark.parametrize("fuse", [True, False])
def test_widths_cover_every_kernel_shape(w1, w2, fuse, tmp_path, ref_bin):
    """2-relation joins whose widths hit each fused / TSQR bucket (4..128),
    odd widths (scalar path) and long groups (carry chains)."""
    rng = np.random.default_rng(w1 * 100 + w2)
    rels = []
    for i, w in enumerate((w1, w2)):
        keys = np.concatenate([rng.integers(0, 300, 4000), np.full(900, 7)]).reshape(-1, 1)
        rng.shuffle(keys)
        data = rng.standard_normal((keys.shape[0], w)) * rng.uniform(0.1, 10.0, w)
        rels.append(fgdb.RelationData(f"R{i}", ["k"], [f"c{i}_{j}" for j in range(w)],
                                      keys.astype(np.int64), data))
    db = fgdb.Database(rels, 0, [-1, 0])
    ref = run_ref(db, tmp_path)
    res, R = run_gpu(db, fuse=fuse)
    assert r_distance(R, ref.R) <= R_TOL
    check_counts(res, ref)


def _write_csv_db(db, d):
    """A database as the reference's config + CSV files (join_tree.hpp:370-445)."""
    names = [r.name for r in db.relations]
    lines = []
    for r in db.relations:
        with open(os.path.join(d, r.name + ".csv"), "w") as f:
            f.write(",".join(list(r.key_attrs) + list(r.data_attrs)) + "\n")
            for k, v in zip(r.keys, r.data):
                f.write(",".join([str(int(x)) for x in k] + ["%.17g" % x for x in v]) + "\n")
        lines.append(f"relation {r.name} file={r.name}.csv keys={','.join(r.key_attrs)} "
                     f"data={','.join(r.data_attrs)}")

    def term(i):
        kids = [c for c, p in enumerate(db.parent) if p == i and c != db.root]
        return names[i] + ("(" + ",".join(term(c) for c in kids) + ")" if kids else "")

    lines.append("tree " + term(db.root))
    p = os.path.join(d, "db.cfg")
    with open(p, "w") as f:
        f.write("\n".join(lines) + "\n")
    return p


def _read_csv_matrix(p):
    with open(p) as f:
        rows = [ln.rstrip("\n").split(",") for ln in f if ln.strip()]
    return rows[0], np.array([[float(x) for x in r] for r in rows[1:]])


@pytest.mark.parametrize("case", ["db1", "C1", "C4", "rnd_8"])
def test_driver_swap(case, tmp_path):
    """The reference CLI driver (driver.hpp:run) with its run_pipeline call
    swapped for figaro::gpu::run_pipeline<PipelineResult> (
    oracle/_ref/driver_swap) against the unmodified driver (driver_ref) on
    the same config: R, the count dump (write_counts_csv, every map of every
    node, text-identical), the R0 dump and the Q output."""
    ref = os.path.join(os.path.dirname(REF_BIN), "driver_ref")
    swap = os.path.join(os.path.dirname(REF_BIN), "driver_swap")
    if not (os.path.exists(ref) and os.path.exists(swap)):
        pytest.skip("driver_ref / driver_swap not built")
    if case == "db1":
        cfg = os.path.join(os.path.dirname(__file__), "golden", "csv", "db1.cfg")
    elif case.startswith("rnd"):
        cfg = _write_csv_db(fgdb.read_fgdb(golden(case + ".fgdb")), str(tmp_path))
    else:
        cfg = _write_csv_db(workloads.make(case, seed=11, scale=0.01), str(tmp_path))
    outs = {}
    for tag, exe in (("ref", ref), ("gpu", swap)):
        o = {k: str(tmp_path / f"{tag}.{k}") for k in ("r", "counts", "r0", "q")}
        p = subprocess.run([exe, cfg, o["r"], "--counts", o["counts"], "--r0", o["r0"],
                            "--q", o["q"]], capture_output=True, text=True, timeout=600)
        outs[tag] = (o, p.stdout, p.returncode, p.stderr)
    if outs["ref"][2] != 0:  # e.g. rank_error in compute-q: same phase and class
        assert outs["gpu"][2] == outs["ref"][2], outs["gpu"][3]
        assert outs["gpu"][3].split(":")[:2] == outs["ref"][3].split(":")[:2]
        return
    assert outs["gpu"][2] == 0, outs["gpu"][1] + outs["gpu"][3]
    outs = {k: v[:2] for k, v in outs.items()}
    (ro, rlog), (go, glog) = outs["ref"], outs["gpu"]
    # Log: same relations / M / N / tree / rows(R0) lines (timings differ).
    keep = lambda s: [ln.split("->")[0] for ln in s.splitlines()  # noqa: E731
                      if ln.startswith(("relations:", "join tree:", "q rows:"))]
    assert keep(rlog) == keep(glog)
    assert [ln.split("rows(R0)=")[1] for ln in rlog.splitlines() if "rows(R0)" in ln] == \
        [ln.split("rows(R0)=")[1] for ln in glog.splitlines() if "rows(R0)" in ln]
    with open(ro["counts"]) as a, open(go["counts"]) as b:
        assert a.read() == b.read()
    hr, Rr = _read_csv_matrix(ro["r"])
    hg, Rg = _read_csv_matrix(go["r"])
    assert hr == hg
    assert r_distance(Rg, Rr) <= 1e-10
    h0r, A0r = _read_csv_matrix(ro["r0"])
    h0g, A0g = _read_csv_matrix(go["r0"])
    assert h0r == h0g and A0r.shape == A0g.shape
    assert np.abs(A0r - A0g).max() <= 1e-12 * max(1.0, np.abs(A0r).max())
    with open(ro["q"]) as a, open(go["q"]) as b:
        Qr = np.array([[float(x) for x in ln.split(",")] for ln in a if ln.strip()])
        Qg = np.array([[float(x) for x in ln.split(",")] for ln in b if ln.strip()])
    assert Qr.shape == Qg.shape
    if Qr.size:
        assert np.linalg.norm(Qr - Qg) <= 1e-8 * max(1.0, np.linalg.norm(Qr))
