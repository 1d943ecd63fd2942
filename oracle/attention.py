"""Attention oracle (test infrastructure only).

Restates reference tensor_ops.py:
  * `softmax_rows`              tensor_ops.py:24-40
  * `scaled_dot_attention`      tensor_ops.py:104-127
  * `_row_columns`              tensor_ops.py:130-138
  * `masked_sparse_attention`   tensor_ops.py:141-183
and `_obs_seed_from_blocks`     session.py:89-95.

`masked_sparse_attention` here evaluates the gather form row-chunk by
row-chunk with an explicit cell mask (vertical bit OR slash bit, causal,
diagonal fallback for empty rows), which selects exactly the cells of
`_row_columns` and normalises over them; tests pin it to the reference's
per-row loop within 1e-12.
"""

from __future__ import annotations

import math

import numpy as np


class AllMaskedRow(Exception):
    pass


class EmptyPlan(Exception):
    pass


class NonFiniteInput(Exception):
    pass


def softmax_rows(logits: np.ndarray) -> np.ndarray:
    """tensor_ops.py:24-40."""
    a = np.asarray(logits, dtype=np.float64)
    if np.isnan(a).any() or np.isposinf(a).any():
        raise NonFiniteInput("logits contain NaN or +inf")
    row_max = a.max(axis=1)
    if np.isneginf(row_max).any():
        raise AllMaskedRow("a row is entirely -inf")
    w = np.exp(a - row_max[:, None])
    return w / w.sum(axis=1, keepdims=True)


def scaled_dot_attention(Q, K, V, row_offset: int):
    """tensor_ops.py:104-127 -> (Z, weights)."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    n_new, n_total = Q.shape[0], K.shape[0]
    logits = (Q @ K.T) / math.sqrt(Q.shape[1])
    cols = np.arange(n_total)
    rows = row_offset + np.arange(n_new)
    logits[cols[None, :] > rows[:, None]] = -np.inf
    A = softmax_rows(logits)
    return A @ V, A


def row_columns(slashes, verticals, g: int) -> np.ndarray:
    """tensor_ops.py:130-138."""
    cols = {c for c in verticals if 0 <= c <= g}
    cols.update(g - d for d in slashes if 0 <= g - d)
    if not cols:
        cols = {g}
    return np.fromiter(sorted(cols), dtype=np.intp)


def plan_mask(slashes, verticals, row_offset: int, n_rows: int, n_total: int,
              r0: int = 0) -> np.ndarray:
    """Boolean cell mask of rows [r0, r0+n_rows): exactly the `_row_columns` cells."""
    vbit = np.zeros(n_total, dtype=bool)
    sbit = np.zeros(n_total, dtype=bool)
    v = np.asarray(sorted(verticals), dtype=np.intp)
    s = np.asarray(sorted(slashes), dtype=np.intp)
    vbit[v[(v >= 0) & (v < n_total)]] = True
    sbit[s[(s >= 0) & (s < n_total)]] = True
    g = row_offset + r0 + np.arange(n_rows)
    c = np.arange(n_total)
    d = g[:, None] - c[None, :]
    causal = d >= 0
    M = causal & (vbit[None, :] | sbit[np.clip(d, 0, n_total - 1)])
    empty = ~M.any(axis=1)
    M[np.nonzero(empty)[0], g[empty]] = True  # diagonal fallback
    return M


def masked_sparse_attention(Q, K, V, slashes, verticals, row_offset: int,
                            return_weights: bool = False, chunk: int = 512):
    """tensor_ops.py:141-183 -> Z (and the dense weights, and the cell count)."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    if not slashes and not verticals:
        raise EmptyPlan("plan selects no lines")
    n_new, n_total = Q.shape[0], K.shape[0]
    scale = 1.0 / math.sqrt(Q.shape[1])
    Z = np.zeros((n_new, V.shape[1]))
    W = np.zeros((n_new, n_total)) if return_weights else None
    cells = 0
    for r0 in range(0, n_new, chunk):
        nr = min(chunk, n_new - r0)
        M = plan_mask(slashes, verticals, row_offset, nr, n_total, r0)
        cells += int(M.sum())
        S = (Q[r0:r0 + nr] @ K.T) * scale
        S = np.where(M, S, -np.inf)
        P = np.exp(S - S.max(axis=1, keepdims=True))
        P /= P.sum(axis=1, keepdims=True)
        Z[r0:r0 + nr] = P @ V
        if return_weights:
            W[r0:r0 + nr] = P
    return Z, W, cells


def obs_seed_rows(weights: np.ndarray, window: int):
    """session.py:89-95 for one head: last `window` rows as dense (ids, row)."""
    n_new, n_total = weights.shape
    lo = max(0, n_new - window)
    cols = np.arange(n_total)
    return [(cols, weights[r]) for r in range(lo, n_new)]
