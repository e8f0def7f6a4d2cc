"""Host ingestion (paper_2204_00525_b200/ingest.py) against the reference's
CSV loader, config parser and tree terms (relation.hpp:169-258,
join_tree.hpp:221-445) and its writers (io.hpp).  CPU only, except the last
test which runs the loaded database through the GPU pipeline."""
import io
import json
import os

import numpy as np
import pytest

from oracle import figaro_np as fo
from paper_2204_00525_b200 import fgdb, ingest
from paper_2204_00525_b200 import figaro as F
from tests.conftest import golden
from tests.helpers import r_distance

CSV = golden("csv")


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_load_relation_pins(tmp_path):
    # test_relational.cpp:45-66
    rel = ingest.load_relation(_write(tmp_path, "a.csv", "X,Y\na,1.0\na,3.0\n"), "S", ["X"], ["Y"])
    assert rel.keys == [("a",), ("a",)] and rel.data[:, 0].tolist() == [1.0, 3.0]
    a = ingest.load_relation(_write(tmp_path, "b.csv", "X,Y,Z\n2,0.5,1e3\n1,-2.25,4.0\n1,-3.0,0.25\n2,0.5,99\n"),
                             "S", ["X"], ["Y", "Z"])
    b = ingest.load_relation(_write(tmp_path, "c.csv", "X,Y,Z\n1,-3.0,0.25\n2,0.5,99\n2,0.5,1e3\n1,-2.25,4.0\n"),
                             "S", ["X"], ["Y", "Z"])
    assert a.keys == b.keys and np.array_equal(a.data, b.data)
    assert a.keys == [(1,), (1,), (2,), (2,)] and a.data[:, 0].tolist() == [-3.0, -2.25, 0.5, 0.5]
    d = ingest.load_relation(_write(tmp_path, "d.csv", "X,Y\n1,2.0\n1,2.0\n"), "S", ["X"], ["Y"])
    assert len(d.keys) == 2 and d.data[0, 0] == d.data[1, 0]


def test_load_errors_pins(tmp_path):
    # test_relational.cpp:68-91
    p = _write(tmp_path, "m.csv", "X,Y\n1,2.0\n")
    with pytest.raises(F.schema_error, match=f"^'{p}': column 'Y2' not found in header$"):
        ingest.load_relation(p, "S", ["X"], ["Y2"])
    with pytest.raises(F.parse_error, match="line 3"):
        ingest.load_relation(_write(tmp_path, "b.csv", "X,Y\n1,2.0\n2,oops\n"), "S", ["X"], ["Y"])
    with pytest.raises(F.schema_error):
        ingest.load_relation(_write(tmp_path, "x.csv", "X,Y\n1,2.0\nfoo,3.0\n"), "S", ["X"], ["Y"])
    with pytest.raises(F.parse_error):
        ingest.load_relation(_write(tmp_path, "i.csv", "X,Y\n1,inf\n"), "S", ["X"], ["Y"])


def test_cell_rules():
    """from_chars semantics: no '+', no hex, no spaces inside, int64 range."""
    assert ingest.parse_double("1e3") == 1000.0 and ingest.parse_double("-.5") == -0.5
    for bad in ["+1", "0x10", "1 2", "", "1e", "nan", "1e999"]:
        assert ingest.parse_double(bad) is None, bad
    assert ingest.parse_int64("-12") == -12 and ingest.parse_int64("+1") is None
    assert ingest.parse_int64(str(1 << 63)) is None and ingest.parse_int64(str(-(1 << 63))) == -(1 << 63)
    assert ingest.split_csv_line(" a ,b\r,, c") == ["a", "b", "", "c"]


def test_tree_terms_and_config():
    # test_relational.cpp:130-137
    t = ingest.parse_tree_term("S1(S2(S3,S4))")
    assert t.name == "S1" and len(t.children) == 1 and len(t.children[0].children) == 2
    for bad in ["S1(S2", "S1)x", "", "S1(,S2)"]:
        with pytest.raises(F.parse_error):
            ingest.parse_tree_term(bad)
    root, parent = ingest.join_tree_parents(["A", "B", "C"], ingest.parse_tree_term("B(C, A)"))
    assert root == 1 and parent == [1, -1, 1]
    with pytest.raises(F.tree_error):
        ingest.join_tree_parents(["A", "B"], ingest.parse_tree_term("A(A)"))
    with pytest.raises(F.tree_error):
        ingest.join_tree_parents(["A", "B"], ingest.parse_tree_term("A"))
    cfg = ingest.parse_config("# c\n\nrelation R file=r.csv keys=a,b data=x\ntree R\n")
    assert cfg.relations[0].keys == ["a", "b"] and cfg.tree_term == "R"
    for bad in ["relation R keys=a\ntree R", "relation R file=x bogus=1\ntree R",
                "relation R file=x\n", "tree R\n", "frobnicate\n"]:
        with pytest.raises(F.parse_error):
            ingest.parse_config(bad)


def _dump(loaded):
    lines = []
    for r in loaded:
        for k, d in zip(r.keys, r.data):
            lines.append(f"{r.name}|{';'.join(str(x) for x in k)}|"
                         f"{';'.join(ingest.format_value(x) for x in d)}")
    return lines


def test_reference_loaded_database_matches(tmp_path):
    """db1: the relations as the reference loaded and canonicalised them
    (exact text), and R of the encoded database through the numpy oracle
    (with semi-join reduction) against the reference's R."""
    with open(os.path.join(CSV, "db1.cfg")) as f:
        cfg = ingest.parse_config(f.read())
    loaded = [ingest.load_relation(os.path.join(CSV, s.file), s.name, s.keys, s.data)
              for s in cfg.relations]
    with open(os.path.join(CSV, "db1.txt"), encoding="utf-8") as f:
        ref_lines = f.read().splitlines()
    assert _dump(loaded) == ref_lines
    rels, tree = ingest.load_database(cfg, CSV)
    orels = [fo.Relation(r.name, r.key_attrs, r.data_attrs, r.keys, r.data) for r in rels]
    res = fo.run_pipeline(orels, tree.root, tree.parent, reduce=True)
    assert r_distance(res.R, fgdb.read_fgrm(os.path.join(CSV, "db1.fgrm"))) <= 1e-10


def test_bad_files_match_reference_errors():
    with open(os.path.join(CSV, "bad.json")) as f:
        expect = json.load(f)
    cls = {6: F.parse_error, 7: F.schema_error}
    for name, e in expect.items():
        with open(os.path.join(CSV, name + ".cfg")) as f:
            cfg = ingest.parse_config(f.read())
        with pytest.raises(cls[e["rc"]]) as ei:
            ingest.load_database(cfg, CSV)
        ref_msg = e["stderr"].split(": ", 2)[2]
        ref_msg = ref_msg.replace(ref_msg[ref_msg.index("'") + 1:ref_msg.index(".csv'") + 4],
                                  os.path.join(CSV, name + ".csv"))
        assert str(ei.value) == ref_msg


def test_writers():
    assert ingest.format_value(0.1) == "0.10000000000000001"
    assert ingest.format_value(-2.0) == "-2"
    out = io.StringIO()
    ingest.write_triangular_csv(out, np.array([[1.5, 2.0], [0.0, 3.0]]), ["a", "b"])
    assert out.getvalue() == "a,b\n1.5,2\n0,3\n"
    out = io.StringIO()
    ingest.write_matrix_csv(out, np.array([[1.0, 0.25]]))
    assert out.getvalue() == "1,0.25\n"


@pytest.mark.gpu
def test_csv_database_on_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    with open(os.path.join(CSV, "db1.cfg")) as f:
        cfg = ingest.parse_config(f.read())
    rels, tree = ingest.load_database(cfg, CSV)
    res = F.run_pipeline(rels, tree, F.PipelineOptions(assume_reduced=False))
    assert r_distance(res.factor.r, fgdb.read_fgrm(os.path.join(CSV, "db1.fgrm"))) <= 1e-10
