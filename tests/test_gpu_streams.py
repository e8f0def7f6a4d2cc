"""Stream ordering between torch and the library (the context binds to
torch's current stream): inputs produced by a just-launched torch kernel are
complete before the pipeline reads them, on the default and on a side
stream, and results are ordered before torch's next op."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2204_00525_b200 import figaro as F  # noqa: E402
from paper_2204_00525_b200 import workloads  # noqa: E402
from tests.helpers import r_distance  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _host_R(db):
    rels = [F.Relation(r.name, r.key_attrs, r.data_attrs, r.keys, r.data) for r in db.relations]
    tree = F.build_join_tree(rels, db.root, db.parent)
    return F.run_pipeline(rels, tree, F.PipelineOptions(assume_reduced=True),
                          fetch_counts=False).factor.r


def _produced_late(db, stream):
    """Device relations whose data is written by a slow torch kernel chain
    enqueued just before the pipeline call (0 * big + data)."""
    out = []
    with torch.cuda.stream(stream):
        big = torch.randn(4096, 4096, device="cuda", dtype=torch.float64)
        for _ in range(3):
            big = big @ big / 64.0
        z = big.sum() * 0.0
        for r in db.relations:
            d = torch.from_numpy(r.data).to("cuda", non_blocking=True) + z
            k = torch.from_numpy(r.keys).to("cuda", non_blocking=True)
            out.append(F.Relation(r.name, r.key_attrs, r.data_attrs, k, d))
    return out


@pytest.mark.parametrize("side", [False, True], ids=["default_stream", "side_stream"])
def test_pipeline_reads_torch_outputs_in_order(side):
    db = workloads.make("C2", seed=21, scale=0.01)
    want = _host_R(db)
    s = torch.cuda.Stream() if side else torch.cuda.current_stream()
    rels = _produced_late(db, s)
    with torch.cuda.stream(s):
        tree = F.build_join_tree(rels, db.root, db.parent)
        res = F.run_pipeline(rels, tree, F.PipelineOptions(assume_reduced=True),
                             fetch_counts=False)
        R2 = res.factor.r * 2.0  # torch op on the same stream consumes R
    s.synchronize()
    assert r_distance(res.factor.r.cpu().numpy(), want) <= 1e-10
    assert np.allclose(R2.cpu().numpy(), 2.0 * res.factor.r.cpu().numpy())


def test_tsqr_reads_torch_outputs_in_order():
    s = torch.cuda.Stream()
    g = torch.Generator(device="cuda").manual_seed(3)
    with torch.cuda.stream(s):
        big = torch.randn(4096, 4096, device="cuda", dtype=torch.float64, generator=g)
        for _ in range(3):
            big = big @ big / 64.0
        A = torch.randn(20000, 24, device="cuda", dtype=torch.float64, generator=g) + \
            big.sum() * 0.0
        R = F.tsqr([(A, 0)], 24)
    s.synchronize()
    Rn = np.linalg.qr(A.cpu().numpy(), mode="r")
    Rn = Rn * np.sign(np.diag(Rn))[:, None]
    assert r_distance(R.cpu().numpy(), Rn) <= 1e-12
