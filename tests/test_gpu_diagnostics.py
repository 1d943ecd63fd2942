"""Plan / selection quality diagnostics on the device:
ground_truth_topB and overlap_rate (reference kvcompress.py:112-123), ported
from the reference's own tests (test_kvcompress.py:122-149) with the oracle
(oracle/kvcompress.py) as the checker."""

from __future__ import annotations

import itertools

import numpy as np
import pytest

from oracle import kvcompress as okv
from paper_2507_13681_b200 import kvcompress as kv
from paper_2507_13681_b200.errors import SizeMismatch

pytestmark = pytest.mark.gpu


def _exhaustive_best(total, budget):
    """Brute-force best subset by (score desc, id asc) -- test_kvcompress.py's oracle."""
    best = None
    for sub in itertools.combinations(range(len(total)), budget):
        key = (-sum(total[list(sub)]), sub)
        if best is None or key < best[0]:
            best = (key, sub)
    return np.array(sorted(best[1]))


def test_ground_truth_reduces_to_obs_selection(cuda_lib):  # test_kvcompress.py:122-126
    rows = np.random.Generator(np.random.PCG64(1)).random((1, 6))
    got = kv.ground_truth_topB([rows], 2)
    assert got.tolist() == okv.select_topB_obs(rows, 2, "summed_over_heads").tolist()


@pytest.mark.parametrize("seed", range(12))
def test_ground_truth_matches_exhaustive(cuda_lib, seed):  # test_kvcompress.py:128-135
    rng = np.random.Generator(np.random.PCG64(seed))
    heads = [rng.random((4, 10)) for _ in range(3)]
    got = kv.ground_truth_topB(heads, 3)
    total = sum(okv.token_scores(h) for h in heads)
    assert got.tolist() == _exhaustive_best(total, 3).tolist()


def test_ground_truth_at_decode_scale(cuda_lib):
    """32 heads x 16 observation rows x 15,256 columns, B = 1024 (C2 turn 3)."""
    rng = np.random.Generator(np.random.PCG64(7))
    heads = [rng.random((16, 15256)) ** 8 for _ in range(32)]
    got = kv.ground_truth_topB(heads, 1024)
    want = okv.select_topB_obs(np.stack([okv.token_scores(h) for h in heads]), 1024, "summed_over_heads")
    assert got.tolist() == want.tolist()


def test_overlap_rate_cases(cuda_lib):  # test_kvcompress.py:139-149
    assert kv.overlap_rate([1, 2], [1, 2], 2) == 1.0
    assert kv.overlap_rate([1, 2], [3, 4], 2) == 0.0
    assert kv.overlap_rate([1, 2], [2, 3], 2) == 0.5
    with pytest.raises(SizeMismatch):
        kv.overlap_rate([1], [2, 3], 2)
    rng = np.random.Generator(np.random.PCG64(3))
    a = rng.choice(20000, 1024, replace=False)
    b = rng.choice(20000, 1024, replace=False)
    assert kv.overlap_rate(a, b, 1024) == len(set(a.tolist()) & set(b.tolist())) / 1024
