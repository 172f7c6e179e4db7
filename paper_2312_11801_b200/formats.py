"""Instance file formats of the reference front end (problem.py:546-681):
MatrixMarket coordinate graphs and QAPLIB-style assignment instances.

Host-side I/O only (not part of the iteration).  The readers accept and
reject the same files as the reference -- symmetric or general coordinate
matrices with pattern / real / integer fields, one-based indices, comments
and blank lines skipped, a general file's off-diagonal entries required in
mirrored pairs -- and raise ``ParseError`` (a ``ValueError``) carrying the
offending line number.  Writers emit what the readers read back exactly
(17 significant digits).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np

from .instances import Graph, Qap

__all__ = ["ParseError", "parse_graph_mm", "write_graph_mm", "parse_qaplib", "write_qaplib"]


class ParseError(ValueError):
    """Malformed instance file (problem.py:43-50); ``line`` is 1-based."""

    def __init__(self, message: str, line=None):
        super().__init__(message if line is None else f"line {line}: {message}")
        self.line = line


def _data_lines(lines: List[str], start: int):
    """(1-based line number, stripped text) of the non-blank, non-comment
    lines from ``start`` on."""
    for ln in range(start, len(lines) + 1):
        text = lines[ln - 1].strip()
        if text and not text.startswith("%"):
            yield ln, text


def parse_graph_mm(path) -> Graph:
    """MatrixMarket coordinate matrix -> undirected graph (problem.py:546-622).
    Symmetric files list each edge once (either triangle); general files
    list both (i, j) and (j, i) with equal values, the lower one is kept.
    Diagonal entries count towards nnz but are not edges; duplicate edges
    sum (Graph.from_edge_list)."""
    with open(path, "r") as fh:
        lines = fh.readlines()
    if not lines:
        raise ParseError("empty file", 1)
    head = lines[0].split()
    if len(head) < 5 or not head[0].startswith("%%MatrixMarket"):
        raise ParseError("missing MatrixMarket header", 1)
    obj, layout, field, symmetry = (t.lower() for t in head[1:5])
    if obj != "matrix" or layout != "coordinate":
        raise ParseError("only coordinate matrices are supported", 1)
    if field not in ("real", "integer", "pattern"):
        raise ParseError(f"unsupported field {field}", 1)
    if symmetry not in ("symmetric", "general"):
        raise ParseError(f"unsupported symmetry {symmetry}", 1)
    body = _data_lines(lines, 2)
    try:
        size_ln, size_text = next(body)
    except StopIteration:
        raise ParseError("missing size line", len(lines)) from None
    fields = size_text.split()
    if len(fields) != 3:
        raise ParseError("size line must have three fields", size_ln)
    try:
        nrows, ncols, nnz = (int(f) for f in fields)
    except ValueError as exc:
        raise ParseError(f"bad size line: {exc}", size_ln) from exc
    if nrows != ncols:
        raise ParseError(f"matrix must be square, got {nrows}x{ncols}", size_ln)
    need = 2 if field == "pattern" else 3
    edges: List[Tuple[int, int, float]] = []
    entries = {}  # general symmetry: (i, j) -> (value, line)
    count = 0
    for ln, text in body:
        parts = text.split()
        if len(parts) < need:
            raise ParseError("entry line has too few fields", ln)
        try:
            i, j = int(parts[0]) - 1, int(parts[1]) - 1
            w = 1.0 if field == "pattern" else float(parts[2])
        except ValueError as exc:
            raise ParseError(f"bad entry: {exc}", ln) from exc
        if not (0 <= i < nrows and 0 <= j < ncols):
            raise ParseError(f"entry ({i + 1},{j + 1}) out of range", ln)
        count += 1
        if symmetry == "general":
            entries[(i, j)] = (w, ln)
        if i != j:
            edges.append((i, j, w))
    if count != nnz:
        raise ParseError(f"expected {nnz} entries, found {count}", len(lines))
    if symmetry == "general":
        for (i, j), (w, ln) in entries.items():
            if i == j:
                continue
            mate = entries.get((j, i))
            if mate is None:
                raise ParseError(f"entry ({i + 1},{j + 1}) has no mirror", ln)
            if abs(mate[0] - w) > 1e-12 * (1 + abs(w)):
                raise ParseError(f"entry ({i + 1},{j + 1}) mirror mismatch", ln)
        edges = [e for e in edges if e[0] > e[1]]  # one of each mirrored pair
    return Graph.from_edge_list(nrows, edges)


def write_graph_mm(g, path) -> None:
    """Symmetric real coordinate file, one line per edge as (larger, smaller)
    one-based indices (problem.py:625-630)."""
    n, eu, ev, ew = _graph_arrays(g)
    with open(path, "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate real symmetric\n")
        fh.write(f"{n} {n} {len(ew)}\n")
        for u, v, w in zip(eu, ev, ew):
            fh.write(f"{int(v) + 1} {int(u) + 1} {float(w):.17g}\n")


def _graph_arrays(g):
    if hasattr(g, "eu"):
        return g.n, g.eu, g.ev, g.ew
    return g.n, g.edges_u, g.edges_v, g.edges_w  # reference GraphInstance


def parse_qaplib(path) -> Qap:
    """Whitespace-separated tokens: the size l, then the l x l weight matrix,
    then the l x l distance matrix, line breaks anywhere (problem.py:633-668)."""
    toks: List[Tuple[str, int]] = []
    with open(path, "r") as fh:
        for ln, line in enumerate(fh, start=1):
            toks.extend((t, ln) for t in line.split())
    if not toks:
        raise ParseError("empty file", 1)
    try:
        l = int(toks[0][0])
    except ValueError as exc:
        raise ParseError(f"bad size field: {exc}", toks[0][1]) from exc
    if l < 1:
        raise ParseError("size must be positive", toks[0][1])
    need = 1 + 2 * l * l
    if len(toks) < need:
        raise ParseError(f"expected {need - 1} matrix entries, found {len(toks) - 1}", toks[-1][1])
    if len(toks) > need:
        raise ParseError("trailing data after matrices", toks[need][1])
    vals = np.empty(need - 1)
    for x, (t, ln) in enumerate(toks[1:need]):
        try:
            vals[x] = float(t)
        except ValueError as exc:
            raise ParseError(f"bad matrix entry {t!r}", ln) from exc
    try:
        return Qap(vals[:l * l].reshape(l, l), vals[l * l:].reshape(l, l))
    except ValueError as exc:
        raise ParseError(str(exc)) from exc


def write_qaplib(q, path) -> None:
    """Size line, blank line, weight block, blank line, distance block
    (problem.py:671-681)."""
    def block(a):
        return "\n".join(" ".join(f"{float(x):.17g}" for x in row) for row in np.asarray(a))

    l = int(np.asarray(q.weights).shape[0])
    with open(path, "w") as fh:
        fh.write(f"{l}\n\n{block(q.weights)}\n\n{block(q.distances)}\n")
