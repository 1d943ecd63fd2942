"""Prefill sparsification oracle (test infrastructure only).

Restates reference prefill.py:
  * `Line`                     prefill.py:24-37
  * `SparsePlan` (fields)      prefill.py:40-61
  * `vertical_length` / `slash_length`  prefill.py:94-99
  * `_BlockView.cell`          prefill.py:102-122
  * `_line_sums`               prefill.py:138-169
  * `_greedy`                  prefill.py:178-229
  * `_coverage`                prefill.py:258-281
  * `sparsify_head`            prefill.py:363-393
  * `plan_for_block`           prefill.py:396-410
with two additions used only for parity diagnostics: the greedy also returns
its pick sequence with the two gains compared at every step, so a test can
prove that the first divergence from the CUDA path is a near-tie.

The per-cell Python loop of `_line_sums` (prefill.py:149-157) is vectorised
here with the same summation order (rows ascending, fp64), so slash and
vertical sums are bit-identical to the reference for the same weights.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .attention import softmax_rows


class InvalidAlpha(Exception):
    pass


@dataclass(frozen=True)
class Line:
    """prefill.py:24-37."""

    kind: str
    index: int
    weight: float
    length: int
    max_cell: float


@dataclass(frozen=True)
class Plan:
    """Field-for-field SparsePlan (prefill.py:40-61) plus the pick trace."""

    selected_slashes: frozenset
    selected_verticals: frozenset
    achieved_coverage: float
    approx_sum: float
    total_weight: float
    n_total: int
    # ((kind, index, gain_s, gain_v, approx, exact, target) after each pick, ...)
    picks: tuple = field(default=(), compare=False)

    def cost(self, n_new: int, n_total: int | None = None) -> int:
        n = self.n_total if n_total is None else n_total
        return sum(slash_length(n_new, n, d) for d in self.selected_slashes) + sum(
            vertical_length(n_new, n, c) for c in self.selected_verticals)


def vertical_length(n_new: int, n_total: int, col: int) -> int:
    """prefill.py:94-95."""
    return max(0, min(n_new, n_total - col))


def slash_length(n_new: int, n_total: int, offset: int) -> int:
    """prefill.py:98-99."""
    return max(0, min(n_new, n_total - offset))


class BlockView:
    """prefill.py:102-122: weights plus explicit global row positions."""

    def __init__(self, weights: np.ndarray, positions: np.ndarray):
        self.weights = np.asarray(weights, dtype=np.float64)
        self.positions = np.asarray(positions, dtype=np.intp)
        self.n_total = self.weights.shape[1]
        self.local_row = {int(g): r for r, g in enumerate(self.positions)}

    def cell(self, offset: int, col: int) -> float:
        r = self.local_row.get(col + offset)
        if r is None:
            return 0.0
        return float(self.weights[r, col])


def line_arrays(weights: np.ndarray, positions: np.ndarray):
    """Unsorted per-index line statistics (prefill.py:138-167), vectorised.

    Returns dict of arrays indexed by vertical column c / slash offset d:
    v_w, v_max, v_len (length n_total) and s_w, s_max, s_len (length max(g)+1).
    """
    w = np.asarray(weights, dtype=np.float64)
    pos = np.asarray(positions, dtype=np.intp)
    n_rows, n_total = w.shape
    v_w = w.sum(axis=0)                      # prefill.py:141 (same call)
    v_max = w.max(axis=0)                    # prefill.py:142
    v_len = n_rows - np.searchsorted(np.sort(pos), np.arange(n_total), side="left")
    g_top = int(min(pos.max(), n_total - 1))
    n_d = g_top + 1
    # A[r, d] = w[r, g_r - d] for 0 <= d <= min(g_r, n_total-1), else 0.0.
    # Summing A over axis 0 adds rows in ascending order starting from 0.0,
    # which is the accumulation order of prefill.py:149-157; adding an
    # explicit 0.0 for missing cells leaves an fp64 sum unchanged.
    d = np.arange(n_d)
    cols = pos[:, None] - d[None, :]
    valid = (cols >= 0) & (d[None, :] <= np.minimum(pos, n_total - 1)[:, None])
    A = np.where(valid, w[np.arange(n_rows)[:, None], np.clip(cols, 0, n_total - 1)], 0.0)
    s_w = A.sum(axis=0)
    s_max = np.maximum(A.max(axis=0), 0.0)   # prefill.py:156-157 starts max at 0.0
    s_len = valid.sum(axis=0)
    return dict(v_w=v_w, v_max=v_max, v_len=v_len, s_w=s_w, s_max=s_max, s_len=s_len)


def line_sums_view(weights: np.ndarray, positions: np.ndarray):
    """prefill.py:138-169: two lists sorted by (-weight, index)."""
    a = line_arrays(weights, positions)
    verticals = [Line("vertical", c, float(a["v_w"][c]), int(a["v_len"][c]), float(a["v_max"][c]))
                 for c in range(len(a["v_w"])) if a["v_len"][c] > 0]
    slashes = [Line("slash", d, float(a["s_w"][d]), int(a["s_len"][d]), float(a["s_max"][d]))
               for d in range(len(a["s_w"])) if a["s_len"][d] > 0]
    key = lambda ln: (-ln.weight, ln.index)
    return sorted(slashes, key=key), sorted(verticals, key=key)


def greedy(slashes, verticals, alpha: float, total_weight: float, view: BlockView) -> Plan:
    """prefill.py:178-229 (same update order, same fp64 arithmetic)."""
    if not (0.0 <= alpha <= 1.0):
        raise InvalidAlpha(f"alpha={alpha} outside [0, 1]")
    target = alpha * total_weight
    eps = 1e-12
    s_idx = v_idx = 0
    sel_s: list[int] = []
    sel_v: list[int] = []
    ol_s = ol_v = 0.0
    approx = 0.0
    exact = 0.0
    picks = []
    while approx < target - eps and exact < target - eps:
        s = slashes[s_idx] if s_idx < len(slashes) else None
        v = verticals[v_idx] if v_idx < len(verticals) else None
        if s is None and v is None:
            break
        gain_s = gain_v = float("nan")
        if s is None:
            take_slash = False
        elif v is None:
            take_slash = True
        else:
            gain_s = (s.weight - ol_v) / max(1, s.length - len(sel_v))
            gain_v = (v.weight - ol_s) / max(1, v.length - len(sel_s))
            take_slash = gain_s >= gain_v
        if take_slash:
            approx += s.weight - ol_v
            exact += s.weight - sum(view.cell(s.index, c) for c in sel_v)
            ol_s += s.max_cell
            sel_s.append(s.index)
            s_idx += 1
            picks.append(("slash", s.index, gain_s, gain_v, approx, exact, target))
        else:
            approx += v.weight - ol_s
            exact += v.weight - sum(view.cell(d, v.index) for d in sel_s)
            ol_v += v.max_cell
            sel_v.append(v.index)
            v_idx += 1
            picks.append(("vertical", v.index, gain_s, gain_v, approx, exact, target))
    coverage = exact / total_weight if total_weight > 0 else 0.0
    return Plan(frozenset(sel_s), frozenset(sel_v), min(coverage, 1.0), approx,
                total_weight, view.n_total, tuple(picks))


def coverage(weights: np.ndarray, positions: np.ndarray, plan) -> float:
    """prefill.py:258-281 (inclusion-exclusion over single crossings)."""
    view = BlockView(weights, positions)
    w = view.weights
    total = float(w.sum())
    if total <= 0:
        return 0.0
    mass = 0.0
    for c in sorted(plan.selected_verticals):
        mass += float(w[:, c].sum())
    for d in sorted(plan.selected_slashes):
        rows = view.positions - d
        valid = rows >= 0
        if valid.any():
            mass += float(w[np.arange(len(rows))[valid], rows[valid]].sum())
    for d in sorted(plan.selected_slashes):
        for c in sorted(plan.selected_verticals):
            mass -= view.cell(d, c)
    return mass / total


def sampled_logits(Q_sampled: np.ndarray, K_all: np.ndarray, row_positions) -> np.ndarray:
    """prefill.py:377-389: causal logits of the sampled rows, -inf beyond g."""
    Q_sampled = np.asarray(Q_sampled, dtype=np.float64)
    K_all = np.asarray(K_all, dtype=np.float64)
    positions = np.asarray(row_positions, dtype=np.intp)
    n_total = K_all.shape[0]
    scale = 1.0 / math.sqrt(K_all.shape[1])
    logits = np.full((Q_sampled.shape[0], n_total), -np.inf)
    for r, g in enumerate(positions):
        hi = min(int(g), n_total - 1) + 1
        logits[r, :hi] = (K_all[:hi] @ Q_sampled[r]) * scale
    return logits


def sparsify_head(Q_sampled, K_all, alpha: float, row_positions, counter=None) -> Plan:
    """prefill.py:363-393."""
    positions = np.asarray(row_positions, dtype=np.intp)
    if np.asarray(Q_sampled).shape[0] != positions.shape[0]:
        raise ValueError("one global position is required per sampled row")
    n_total = np.asarray(K_all).shape[0]
    logits = sampled_logits(Q_sampled, K_all, positions)
    if counter is not None:
        counter.add(int(sum(min(int(g), n_total - 1) + 1 for g in positions)))
    weights = softmax_rows(logits)
    view = BlockView(weights, positions)
    slashes, verticals = line_sums_view(weights, positions)
    return greedy(slashes, verticals, alpha, float(weights.sum()), view)


def plan_for_block(weights: np.ndarray, row_offset: int, alpha: float) -> Plan:
    """prefill.py:396-410 without sampling (diagnostics/tests)."""
    w = np.asarray(weights, dtype=np.float64)
    positions = row_offset + np.arange(w.shape[0])
    view = BlockView(w, positions)
    slashes, verticals = line_sums_view(w, positions)
    return greedy(slashes, verticals, alpha, float(w.sum()), view)
