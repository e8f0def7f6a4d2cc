"""Phase-level kernel parity on the GPU (called through the C ABI):
K1 grouping vs a stable argsort, K3/K5 heads/tails vs the oracle's
head/tail/generalized transforms, K6/K7 TSQR vs the oracle Householder R.
Tolerances: integer outputs bit-exact; FP64 outputs 1e-12 relative
(summation order differs from the reference's sequential loops)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import figaro_np as fo  # noqa: E402
from paper_2204_00525_b200 import figaro as F  # noqa: E402
from tests.helpers import r_distance  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("n,bits,hi", [(1, 0, 1), (1000, 10, 1000), (100_000, 17, 100_000),
                                       (300_000, 40, 1 << 40), (50_000, 64, None), (0, 5, 1),
                                       # onesweep tile edges (4096 u64 / 6144 u32 keys per tile)
                                       (4096, 33, 1 << 33), (4097, 33, 1 << 33), (6144, 12, 7),
                                       (6145, 20, 1 << 20), (12_289, 9, 512),
                                       # all keys equal with bits > 0; one-bit keys
                                       (20_000, 16, 1), (30_000, 1, 2),
                                       # 7+7+6-bit passes (C2's 20-bit keys), 8x6 passes (C3)
                                       (2_000_003, 20, 1 << 20), (1_500_000, 47, 1 << 47),
                                       (1_000_000, 32, 1 << 32), (700_000, 63, 1 << 63)])
def test_group_keys_stable(n, bits, hi):
    rng = np.random.default_rng(n + bits)
    if hi is None:
        keys = rng.integers(0, 1 << 63, n, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
        keys[: n // 3] = keys[n // 3: 2 * (n // 3)]  # duplicates
    else:
        keys = rng.integers(0, hi, n).astype(np.uint64)
    perm, begins, uniq = F.group_keys(dev(keys.view(np.int64)), bits)
    ref_perm = np.argsort(keys, kind="stable")
    assert np.array_equal(perm.cpu().numpy(), ref_perm.astype(np.int32))
    sk = keys[ref_perm]
    u, first = np.unique(sk, return_index=True)
    assert np.array_equal(uniq.cpu().numpy().view(np.uint64), u)
    assert np.array_equal(begins.cpu().numpy(), np.append(first, n).astype(np.int32))


def segments(sizes):
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)


@pytest.mark.parametrize("w", [1, 3, 4, 16, 20, 33, 64, 130])
@pytest.mark.parametrize("kind", ["small", "heavy", "singletons", "mixed"])
def test_heads_tails_plain(w, kind):
    rng = np.random.default_rng(w * 7 + len(kind))
    sizes = {"small": rng.integers(1, 20, 400), "heavy": np.array([1, 5000, 3, 700, 2]),
             "singletons": np.ones(1000, dtype=int),
             "mixed": np.concatenate([rng.integers(1, 4, 300), [3000], rng.integers(200, 300, 5)])}[kind]
    n = int(sizes.sum())
    data = rng.standard_normal((n, w))
    perm = rng.permutation(n).astype(np.int32)
    cnt = rng.integers(1, 50, len(sizes)).astype(np.uint64)
    begins = segments(sizes)
    heads, tails, scales = F.heads_tails(dev(data), dev(begins), perm=dev(perm), tail_count=dev(cnt))
    heads, tails, scales = heads.cpu().numpy(), tails.cpu().numpy(), scales.cpu().numpy()
    t_off = 0
    for g, m in enumerate(sizes):
        grp = data[perm[begins[g]:begins[g + 1]]]
        np.testing.assert_allclose(heads[g], fo.head(grp), rtol=1e-12, atol=1e-12 * np.abs(grp).max())
        ref_t = fo.tail(grp) * np.sqrt(float(cnt[g]))
        got_t = tails[t_off:t_off + m - 1]
        t_off += m - 1
        scale = max(np.abs(ref_t).max(), 1e-300) if ref_t.size else 1
        np.testing.assert_allclose(got_t, ref_t, rtol=0, atol=1e-12 * scale * max(1, np.sqrt(m)))
        assert scales[g] == pytest.approx(np.sqrt(m), rel=1e-15)
    assert t_off == tails.shape[0]


@pytest.mark.parametrize("w", [2, 5, 16, 40])
def test_heads_tails_generalized(w):
    rng = np.random.default_rng(w)
    sizes = np.concatenate([rng.integers(1, 12, 200), [900, 1]])
    n = int(sizes.sum())
    data = rng.standard_normal((n, w))
    wts = rng.uniform(0.1, 40.0, n)
    begins = segments(sizes)
    heads, tails, scales = F.heads_tails(dev(data), dev(begins), weights=dev(wts))
    heads, tails = heads.cpu().numpy(), tails.cpu().numpy()
    t_off = 0
    for g, m in enumerate(sizes):
        grp = data[begins[g]:begins[g + 1]]
        v = wts[begins[g]:begins[g + 1]]
        np.testing.assert_allclose(heads[g], fo.generalized_head(grp, v), rtol=1e-11, atol=1e-11)
        got = tails[t_off:t_off + m - 1]
        t_off += m - 1
        np.testing.assert_allclose(got, fo.generalized_tail(grp, v), rtol=1e-10, atol=1e-11)
        assert scales.cpu().numpy()[g] == pytest.approx(np.linalg.norm(v), rel=1e-13)


@pytest.mark.parametrize("n,widths", [(8, [(3000, 8, 0)]), (16, [(100_000, 16, 0)]),
                                      (32, [(50_000, 16, 0), (40_000, 16, 16), (5_000, 32, 0)]),
                                      (5, [(7, 5, 0)]), (20, [(2, 20, 0), (300, 12, 8)]),
                                      (64, [(20_000, 64, 0)]), (128, [(3000, 64, 0), (2000, 64, 64), (500, 128, 0)]),
                                      (36, [(10_000, 8, 0), (9_000, 20, 8), (1000, 36, 0)])])
def test_tsqr_matches_householder(n, widths):
    rng = np.random.default_rng(n)
    blocks, dense = [], []
    for rows, cols, cb in widths:
        x = rng.standard_normal((rows, cols)) * rng.uniform(1e-3, 1e3, cols)
        blocks.append((dev(x), cb))
        full = np.zeros((rows, n))
        full[:, cb:cb + cols] = x
        dense.append(full)
    R = F.tsqr(blocks, n).cpu().numpy()
    ref = fo.normalize_signs(fo.householder_r(np.vstack(dense)))
    assert np.all(np.tril(R, -1) == 0)
    assert np.all(np.diag(R) >= 0)
    assert r_distance(R, ref) <= 1e-12  # Gram comparison when rank-deficient


def test_tsqr_rank_deficient_and_empty():
    x = np.zeros((50, 4))
    x[:, 0] = 1.0
    x[:, 2] = np.arange(50.0)
    R = F.tsqr([(dev(x), 0)], 4).cpu().numpy()
    np.testing.assert_allclose(R.T @ R, x.T @ x, rtol=1e-12, atol=1e-9)
    assert R[1, 1] == 0.0 and R[3, 3] == 0.0
    R = F.tsqr([], 3).cpu().numpy()
    assert np.array_equal(R, np.zeros((3, 3)))


@pytest.mark.parametrize("w", [40, 48, 64, 128])
def test_tsqr_wide_large_spans(w):
    """The look-ahead blocked TSQR at span sizes that select its large-span
    configurations (>= 512k rows: triangular-R, 2-warp CTAs at W = 64/128),
    with exactly zero, duplicated and badly scaled columns (downdate repairs,
    zero panels).  R is compared through the Gram matrix (rank-deficient)."""
    rows = 600_000
    rng = np.random.default_rng(w)
    x = rng.standard_normal((rows, w)) * np.logspace(-3, 3, w)
    x[:, 1] = x[:, 0]
    x[:, w // 2: w // 2 + 8] = 0.0  # one whole zero panel
    R = F.tsqr([(dev(x), 0)], w).cpu().numpy()
    assert np.all(np.tril(R, -1) == 0) and np.all(np.diag(R) >= 0)
    G = x.T @ x
    assert np.linalg.norm(R.T @ R - G) / np.linalg.norm(G) <= 1e-13
    # full-rank part: compare with numpy's Householder R on the same columns
    keep = [j for j in range(w) if j != 1 and not (w // 2 <= j < w // 2 + 8)]
    xr = np.ascontiguousarray(x[:, keep])
    Rk = F.tsqr([(dev(xr), 0)], len(keep)).cpu().numpy()
    ref = fo.normalize_signs(np.linalg.qr(xr, mode="r"))
    assert r_distance(Rk, ref) <= 1e-12


@pytest.mark.parametrize("bits", [20, 47])
def test_group_keys_zipf(bits):
    """Heavily skewed keys (Zipf 1.1 / 1.3, as C3's fact keys and C5) through
    the onesweep sort: stable permutation and offsets bit-exact."""
    rng = np.random.default_rng(bits)
    n = 3_000_000
    z = rng.zipf(1.1 if bits > 32 else 1.3, n) % (1 << min(bits, 40))
    keys = (z.astype(np.uint64) * np.uint64(2654435761)) & np.uint64((1 << bits) - 1)
    perm, begins, uniq = F.group_keys(dev(keys.view(np.int64)), bits)
    ref_perm = np.argsort(keys, kind="stable")
    assert np.array_equal(perm.cpu().numpy(), ref_perm.astype(np.int32))
    sk = keys[ref_perm]
    u, first = np.unique(sk, return_index=True)
    assert np.array_equal(uniq.cpu().numpy().view(np.uint64), u)
    assert np.array_equal(begins.cpu().numpy(), np.append(first, n).astype(np.int32))
