"""Host ingestion and dumps: the data formats on either side of the path
(SURVEY 8f, rank 4).

Restates, on the host, the reference's
  * CSV relation loader   load_relation        (relation.hpp:169-258)
    with its cell rules (trim, split_csv_line, parse_int64, parse_double:
    relation.hpp:71-107) and canonical order (relation.hpp:109-167);
  * config / tree term    parse_config, parse_tree_term, join_tree_from_term,
                          load_database        (join_tree.hpp:221-445);
  * CSV writers           format_value, write_triangular_csv,
                          write_matrix_csv     (io.hpp:18-62).
String-typed key columns are dictionary-encoded per attribute across all
relations of a database (order-preserving byte order), so the int64 C ABI
sees keys that sort, group and join exactly as the reference's
std::variant<int64, string> keys do.
"""
from __future__ import annotations

import dataclasses
import math
import os
import re
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from .figaro import (JoinTree, Relation, build_join_tree, error, parse_error,
                     schema_error, tree_error, unsupported_error)

_INT = re.compile(r"-?[0-9]+\Z")
# std::from_chars(double) in general format: no leading '+', no hex, no
# whitespace; inf/nan spellings parse but are rejected as non-finite.
_DBL = re.compile(r"-?(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?\Z")
_NONFINITE = re.compile(r"-?(?:inf|infinity|nan(?:\([0-9A-Za-z_]*\))?)\Z", re.I)


def trim(s: str) -> str:
    """relation.hpp:71-79: strip ' ', '\\t', '\\r' at both ends."""
    return s.strip(" \t\r")


def split_csv_line(line: str) -> List[str]:
    """relation.hpp:81-91: split on every ',', trim each cell (no quoting)."""
    return [trim(c) for c in line.split(",")]


def parse_int64(s: str) -> Optional[int]:
    """relation.hpp:93-99: the whole cell is a base-10 int64."""
    if not _INT.match(s):
        return None
    v = int(s)
    return v if -(1 << 63) <= v < (1 << 63) else None


def parse_double(s: str) -> Optional[float]:
    """relation.hpp:101-107 (+ the isfinite check of load_relation)."""
    if _DBL.match(s):
        x = float(s)
        return x if math.isfinite(x) else None  # overflow -> inf
    return None


@dataclasses.dataclass
class LoadedRelation:
    """A relation as load_relation returns it: keys are int or str tuples,
    rows in canonical order (key tuple, then data)."""
    name: str
    key_attrs: List[str]
    data_attrs: List[str]
    keys: List[tuple]
    data: np.ndarray


def load_relation(path: str, name: str, key_attrs: Sequence[str],
                  data_attrs: Sequence[str]) -> LoadedRelation:
    """relation.hpp:169-258."""
    try:
        f = open(path, "r", newline="")
    except OSError:
        raise error(f"cannot open '{path}'")
    with f:
        lines = f.read().split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    if not lines:
        raise parse_error(f"'{path}': missing header line")
    header = split_csv_line(lines[0])

    def col_of(attr):
        for i, h in enumerate(header):
            if h == attr:
                return i
        raise schema_error(f"'{path}': column '{attr}' not found in header")

    kc = [col_of(a) for a in key_attrs]
    dc = [col_of(a) for a in data_attrs]
    raw_keys: List[List[str]] = []
    raw_data: List[List[float]] = []
    for lineno, line in enumerate(lines[1:], start=2):
        if trim(line) == "":
            continue
        cells = split_csv_line(line)
        if len(cells) != len(header):
            raise parse_error(f"'{path}' line {lineno}: expected {len(header)} cells, "
                              f"got {len(cells)}")
        raw_keys.append([cells[c] for c in kc])
        row = []
        for c in dc:
            x = parse_double(cells[c])
            if x is None:
                raise parse_error(f"'{path}' line {lineno}: cannot parse data cell "
                                  f"'{cells[c]}' as a finite real")
            row.append(x)
        raw_data.append(row)
    rows = len(raw_keys)
    typed_cols = []
    for c, attr in enumerate(key_attrs):
        ints = [parse_int64(raw_keys[i][c]) for i in range(rows)]
        any_int = any(v is not None for v in ints)
        any_str = any(v is None for v in ints)
        if any_int and any_str:
            raise schema_error(f"'{path}': key column '{attr}' mixes integers and strings")
        typed_cols.append(ints if any_int else [raw_keys[i][c] for i in range(rows)])
    keys = [tuple(col[i] for col in typed_cols) for i in range(rows)]
    data = np.array(raw_data, dtype=np.float64).reshape(rows, len(data_attrs))
    # canonicalize (relation.hpp:109-167): key tuple, then data values.
    def sort_key(i):
        return (tuple(k.encode() if isinstance(k, str) else k for k in keys[i]),
                tuple(data[i]))
    order = sorted(range(rows), key=sort_key)
    return LoadedRelation(name, list(key_attrs), list(data_attrs),
                          [keys[i] for i in order], data[order] if rows else data)


# ---------------------------------------------------------------- config

@dataclasses.dataclass
class TreeTerm:
    name: str
    children: List["TreeTerm"] = dataclasses.field(default_factory=list)


def parse_tree_term(text: str) -> TreeTerm:
    """join_tree.hpp:238-290: term := name | name(term, term, ...)."""
    pos = 0

    def fail(what):
        raise parse_error(f"tree term: {what} at offset {pos} in '{text}'")

    def skip_ws():
        nonlocal pos
        while pos < len(text) and text[pos] in " \t":
            pos += 1

    def ident():
        nonlocal pos
        skip_ws()
        start = pos
        while pos < len(text) and text[pos] not in "(), \t":
            pos += 1
        if pos == start:
            fail("expected relation name")
        return text[start:pos]

    def term():
        nonlocal pos
        t = TreeTerm(ident())
        skip_ws()
        if pos < len(text) and text[pos] == "(":
            pos += 1
            while True:
                t.children.append(term())
                skip_ws()
                if pos < len(text) and text[pos] == ",":
                    pos += 1
                    continue
                if pos < len(text) and text[pos] == ")":
                    pos += 1
                    break
                fail("expected ',' or ')'")
        return t

    t = term()
    skip_ws()
    if pos != len(text):
        fail("trailing input")
    return t


def to_term_string(tree: JoinTree, names: Sequence[str], node: Optional[int] = None) -> str:
    """join_tree.hpp:292-306."""
    node = tree.root if node is None else node
    out = names[node]
    if tree.children[node]:
        out += "(" + ",".join(to_term_string(tree, names, c) for c in tree.children[node]) + ")"
    return out


def join_tree_parents(names: Sequence[str], term: TreeTerm) -> Tuple[int, List[int]]:
    """join_tree_from_term (join_tree.hpp:308-339) without the validation:
    (root, parent[]) for build_join_tree."""
    index: Dict[str, int] = {}
    for i, n in enumerate(names):
        if n in index:
            raise schema_error(f"duplicate relation name '{n}'")
        index[n] = i
    parent = [-2] * len(names)

    def resolve(n):
        if n not in index:
            raise tree_error(f"tree term names unknown relation '{n}'")
        return index[n]

    def walk(t, par):
        node = resolve(t.name)
        if parent[node] != -2:
            raise tree_error(f"relation '{t.name}' appears twice in the tree")
        parent[node] = par
        for c in t.children:
            walk(c, node)

    root = resolve(term.name)
    walk(term, -1)
    for i, p in enumerate(parent):
        if p == -2:
            raise tree_error(f"relation '{names[i]}' missing from the tree term")
    return root, parent


@dataclasses.dataclass
class RelationSpec:
    name: str
    file: str = ""
    keys: List[str] = dataclasses.field(default_factory=list)
    data: List[str] = dataclasses.field(default_factory=list)


@dataclasses.dataclass
class DatabaseConfig:
    relations: List[RelationSpec]
    tree_term: str


def _split_names(s: str) -> List[str]:
    """join_tree.hpp split_names: comma list, empty items dropped."""
    return [trim(x) for x in s.split(",") if trim(x)]


def parse_config(text: str) -> DatabaseConfig:
    """join_tree.hpp:370-424."""
    rels: List[RelationSpec] = []
    term = ""
    for lineno, line in enumerate(text.split("\n"), start=1):
        t = trim(line)
        if not t or t.startswith("#"):
            continue
        words = t.split()
        if words[0] == "relation":
            if len(words) < 2:
                raise parse_error(f"config line {lineno}: relation needs a name")
            spec = RelationSpec(words[1])
            for kv in words[2:]:
                if "=" not in kv:
                    raise parse_error(f"config line {lineno}: expected key=value, got '{kv}'")
                k, v = kv.split("=", 1)
                if k == "file":
                    spec.file = v
                elif k == "keys":
                    spec.keys = _split_names(v)
                elif k == "data":
                    spec.data = _split_names(v)
                else:
                    raise parse_error(f"config line {lineno}: unknown option '{k}'")
            if not spec.file:
                raise parse_error(f"config line {lineno}: relation '{spec.name}' needs file=")
            rels.append(spec)
        elif words[0] == "tree":
            term = trim(t[len("tree"):])
            if not term:
                raise parse_error(f"config line {lineno}: tree needs a term")
        else:
            raise parse_error(f"config line {lineno}: unknown directive '{words[0]}'")
    if not rels:
        raise parse_error("config: no relations")
    if not term:
        raise parse_error("config: no tree directive")
    return DatabaseConfig(rels, term)


def encode_relations(loaded: Sequence[LoadedRelation]) -> List[Relation]:
    """int64 relations for the C ABI: string key attributes are replaced by
    their rank among the attribute's distinct strings (byte order) across
    all relations, which preserves order and equality."""
    kinds: Dict[str, set] = {}
    for r in loaded:
        for c, a in enumerate(r.key_attrs):
            for k in r.keys:
                kinds.setdefault(a, set()).add(type(k[c]))
    for a, ks in kinds.items():
        if len(ks) > 1:
            raise unsupported_error(f"key attribute '{a}' is an integer in one relation "
                                    "and a string in another")
    dicts: Dict[str, Dict[str, int]] = {}
    for a, ks in kinds.items():
        if str in ks:
            vals = sorted({k[c] for r in loaded for c, b in enumerate(r.key_attrs) if b == a
                           for k in r.keys}, key=lambda s: s.encode())
            dicts[a] = {s: i for i, s in enumerate(vals)}
    out = []
    for r in loaded:
        keys = np.array([[dicts[a][k[c]] if a in dicts else k[c]
                          for c, a in enumerate(r.key_attrs)] for k in r.keys],
                        dtype=np.int64).reshape(len(r.keys), len(r.key_attrs))
        out.append(Relation(r.name, r.key_attrs, r.data_attrs, keys,
                            np.ascontiguousarray(r.data)))
    return out


def load_database(cfg: DatabaseConfig, base_dir: str = "") -> Tuple[List[Relation], JoinTree]:
    """join_tree.hpp:432-445: CSVs of the config (relative paths against
    base_dir) and the join tree of its term, ready for run_pipeline."""
    loaded = []
    for spec in cfg.relations:
        path = spec.file
        if base_dir and path and not path.startswith("/"):
            path = os.path.join(base_dir, path)
        loaded.append(load_relation(path, spec.name, spec.keys, spec.data))
    rels = encode_relations(loaded)
    root, parent = join_tree_parents([r.name for r in rels], parse_tree_term(cfg.tree_term))
    return rels, build_join_tree(rels, root, parent)


# ---------------------------------------------------------------- writers

def format_value(x: float) -> str:
    """io.hpp:18-23: %.17g."""
    return "%.17g" % x


def write_triangular_csv(out, R, column_names: Sequence[str]) -> None:
    """io.hpp:34-49: header, then rows with a literal 0 below the diagonal."""
    R = np.asarray(R)
    out.write(",".join(column_names) + "\n")
    n = R.shape[0]
    for i in range(n):
        out.write(",".join("0" if j < i else format_value(R[i, j]) for j in range(n)) + "\n")


def write_matrix_csv(out, M, names: Sequence[str] = ()) -> None:
    """io.hpp:51-62."""
    M = np.asarray(M)
    if names:
        out.write(",".join(names) + "\n")
    for row in M:
        out.write(",".join(format_value(x) for x in row) + "\n")
