"""CPU-side checks of the drop-in boundary: the C-ABI library exists, loads,
exports every entry point include/figaro_cuda.h declares, and refuses to
compute without a B200 (no CPU fallback).  Also the host-side tree/layout
logic of the Python mirror against the oracle restatement."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2204_00525_b200 import _lib
from paper_2204_00525_b200 import figaro as F
from oracle import figaro_np as fo
from paper_2204_00525_b200 import fgdb
from tests.conftest import ROOT, golden
from tests.helpers import golden_stems

HEADER = os.path.join(ROOT, "include", "figaro_cuda.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"FG_API\s+[\w\s\*]+?\b(fg_\w+)\s*\(", text)))


def test_header_declares_the_exported_list():
    assert declared_symbols() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libfigaro_cuda.so not built (run __graft_entry__.build())")
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_no_cpu_fallback_without_gpu():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    lib = _lib.load()
    h = C.c_void_p()
    assert lib.fg_ctx_create(0, C.byref(h)) == _lib.FG_E_CUDA
    assert lib.fg_version() == 1
    with pytest.raises(F.cuda_error):
        F.Context(0)


@pytest.mark.parametrize("stem", golden_stems("rnd_")[:10] + golden_stems("hand_"))
def test_host_tree_and_layout_mirror(stem):
    db = fgdb.read_fgdb(golden(stem + ".fgdb"))
    rels = [F.Relation(r.name, r.key_attrs, r.data_attrs, r.keys, r.data) for r in db.relations]
    orels, root, parent = fo.from_fgdb(db)
    t = F.build_join_tree(rels, root, parent)
    ot = fo.build_join_tree(orels, root, parent)
    assert t.preorder == ot.preorder and t.children == ot.children
    assert t.parent_attrs == ot.parent_attrs
    lay, olay = F.make_layout(rels, t), fo.Layout(orels, ot)
    assert (lay.total, lay.node_offset, lay.subtree_begin, lay.subtree_end) == \
        (olay.total, olay.node_offset, olay.subtree_begin, olay.subtree_end)


def test_host_tree_errors():
    r = F.Relation("S", ["X"], ["a"], np.zeros((1, 1), np.int64), np.zeros((1, 1)))
    with pytest.raises(F.tree_error):
        F.build_join_tree([r, r], 0, [0, 0])
    with pytest.raises(F.tree_error):
        F.build_join_tree([r, r], 0, [-1, 5])
    with pytest.raises(F.tree_error):
        F.build_join_tree([], 0, [])
