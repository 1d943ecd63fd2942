"""Attention-only turn driver (test infrastructure only).

Restates the LoopServe branch of `run_turn` (reference session.py:113-201)
for one attention layer with synthetic Q/K/V instead of the toy model's
projections (model.py:227-231):
  * row policy + sparsifier closure   session.py:135-147
  * sparse branch of forward_extend   model.py:242-251
  * observation seeds                 session.py:89-95 (last W rows only)
  * op counts                         session.py:185-191
GQA mapping (a build decision): reference "head" h
is q-head h; it reads K/V of kv-head h // (n_q / n_kv).
"""

from __future__ import annotations

import math

import numpy as np

from .attention import masked_sparse_attention, plan_mask
from .prefill import sparsify_head
from .seeding import turn_rows


class OpCounter:
    """opcount.py:12-17."""

    def __init__(self):
        self.scores = 0

    def add(self, n: int) -> None:
        self.scores += int(n)


def seed_rows_for_plan(Q, K, slashes, verticals, row_offset: int, window: int):
    """Dense weights of the block's last `window` rows under the plan
    (session.py:92-94 reads block.weights[r] for r in [n_new-W, n_new))."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    n_new, n_total = Q.shape[0], K.shape[0]
    lo = max(0, n_new - window)
    M = plan_mask(slashes, verticals, row_offset, n_new - lo, n_total, lo)
    S = (Q[lo:] @ K.T) / math.sqrt(Q.shape[1])
    S = np.where(M, S, -np.inf)
    P = np.exp(S - S.max(axis=1, keepdims=True))
    P /= P.sum(axis=1, keepdims=True)
    cols = np.arange(n_total)
    return [(cols, P[i]) for i in range(P.shape[0])]


def prefill_head(Q, K, V, row_offset: int, alpha: float, rate: float, floor: int,
                 session_seed: int, turn: int, layer: int, head: int, window: int,
                 counter: OpCounter | None = None):
    """One (layer, head) of the sparse prefill: plan, Z, decode seed rows."""
    Q = np.asarray(Q, dtype=np.float64)
    n_new = Q.shape[0]
    positions = row_offset + np.arange(n_new)
    rows = turn_rows(n_new, alpha, rate, floor, session_seed, turn, layer, head)
    plan = sparsify_head(Q[rows], K, alpha, positions[rows], counter=counter)
    Z, _, cells = masked_sparse_attention(Q, K, V, plan.selected_slashes,
                                          plan.selected_verticals, row_offset)
    if counter is not None:
        counter.add(cells)
    seeds = seed_rows_for_plan(Q, K, plan.selected_slashes, plan.selected_verticals,
                               row_offset, window)
    return dict(rows=rows, plan=plan, Z=Z, seeds=seeds, cells=cells)
