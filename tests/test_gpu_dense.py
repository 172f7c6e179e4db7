"""Tall-skinny dense kernels against numpy: the Gram A^T B (TMA-fed path for
16-byte-aligned operands of at least 1024 rows, the v1 kernel otherwise) on
the shapes, leading dimensions and views the solver uses (V^T Y, F^T Psi,
orthonormalisation Grams, column views)."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    (1_000_003, 11, 11, 0, 0),   # C4-sized V^T Y (odd row count)
    (200_001, 10, 10, 1, 0),     # F = tmp[:, :kc] (lda = kc + 1) against Psi
    (63_000, 20, 20, 0, 0),      # C5
    (4_099, 64, 64, 0, 0),       # largest k
    (5_000, 11, 1, 0, 0),        # basis^T v
    (3_001, 1, 1, 0, 5),         # a column of a wider block
    (777, 11, 11, 0, 0),         # below the TMA threshold (v1 kernel)
]


@pytest.mark.parametrize("n,ka,kb,pada,padb", CASES)
@pytest.mark.parametrize("sym", [False, True])
def test_gram_matches_numpy(n, ka, kb, pada, padb, sym):
    if sym and ka != kb:
        pytest.skip("symmetric output needs ka == kb")
    from paper_2312_11801_b200.engine import Engine
    from paper_2312_11801_b200.runtime import runtime
    rt = runtime()
    rng = np.random.default_rng(n + ka)
    a_full = rng.standard_normal((n, ka + pada))
    b_full = rng.standard_normal((n, kb + padb))
    A = rt.upload(a_full)[:, :ka]
    B = rt.upload(b_full)[:, padb:padb + kb] if padb else rt.upload(b_full)
    a, b = a_full[:, :ka], b_full[:, padb:padb + kb]
    G = rt.empty(ka, kb)
    eng = Engine.__new__(Engine)
    eng.rt, eng.lib, eng.h, eng.comm = rt, rt.lib, rt.h, None
    eng.gram(A, B, G, sym=sym)
    want = a.T @ b
    if sym:
        want = 0.5 * (want + want.T)
    got = G.cpu().numpy()
    scale = np.sqrt(np.outer((a * a).sum(0), (b * b).sum(0)))
    assert np.max(np.abs(got - want) / scale) <= 64 * np.sqrt(n) * 2.0 ** -53
