"""Progressive decode KV-compression oracle (test infrastructure only).

Restates reference kvcompress.py:
  * `CompressionConfig`         kvcompress.py:22-36
  * `token_scores`              kvcompress.py:58-64
  * `accumulate_scores`         kvcompress.py:67-83
  * `_top_by_score`             kvcompress.py:86-90
  * `select_topB_obs`           kvcompress.py:93-109
  * `retained_union`            kvcompress.py:126-130
  * `compact_cache`             kvcompress.py:133-147
  * `progressive_decode`        kvcompress.py:167-240, restated for
    attention-only shapes: the per-head decode step is model.py:232-241
    (cols = working set + new position, softmax of K[cols].q/sqrt(d),
    out = w.V[cols], obs row = (cols, w)); q and the appended K/V row of every
    step are inputs instead of coming from the toy model's projections.
"""

from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass, field

import numpy as np


class EmptyWindow(Exception):
    pass


class InvalidConfig(Exception):
    pass


class InvalidIds(Exception):
    pass


@dataclass(frozen=True)
class CompressionConfig:
    """kvcompress.py:22-36."""

    budget: int | None = 1024
    interval: int = 16
    warmup: int = 16
    obs_window: int | None = None

    def window(self) -> int:
        return self.interval if self.obs_window is None else self.obs_window

    def validate(self) -> None:
        if self.budget is not None and self.budget < 1:
            raise InvalidConfig("budget must be >= 1 (or None for unlimited)")
        if self.interval < 1 or self.warmup < 1 or self.window() < 1:
            raise InvalidConfig("interval, warmup, and obs_window must be >= 1")


def token_scores(window_rows) -> np.ndarray:
    """kvcompress.py:58-64."""
    rows = np.asarray(window_rows, dtype=np.float64)
    if rows.ndim != 2 or rows.shape[0] == 0:
        raise EmptyWindow("need at least one observation row")
    return rows.sum(axis=0)


def accumulate_scores(buffered_rows):
    """kvcompress.py:67-83, vectorised: rows are added oldest -> newest per id
    in fp64 (np.add.at is unbuffered and applies in order), so the sums are
    bit-identical to the dict loop. Only touched ids are candidates."""
    rows = list(buffered_rows)
    if not rows:
        raise EmptyWindow("need at least one observation row")
    hi = max((int(np.max(ids)) + 1 if len(ids) else 0) for ids, _ in rows)
    acc = np.zeros(hi)
    touched = np.zeros(hi, dtype=bool)
    for ids, w in rows:
        ids = np.asarray(ids, dtype=np.intp)
        np.add.at(acc, ids, np.asarray(w, dtype=np.float64))
        touched[ids] = True
    ids = np.nonzero(touched)[0].astype(np.intp)
    return ids, acc[ids]


def top_by_score(ids: np.ndarray, scores: np.ndarray, budget: int) -> np.ndarray:
    """kvcompress.py:86-90: B highest by (score desc, id asc), returned sorted."""
    ids = np.asarray(ids)
    if budget >= len(ids):
        return np.sort(ids)
    order = np.lexsort((ids, -np.asarray(scores)))
    return np.sort(ids[order[:budget]])


def select_topB_obs(scores, budget: int, aggregate: str = "per_head", candidate_ids=None):
    """kvcompress.py:93-109."""
    s = np.atleast_2d(np.asarray(scores, dtype=np.float64))
    ids = np.arange(s.shape[1]) if candidate_ids is None else np.asarray(candidate_ids)
    if aggregate == "summed_over_heads":
        return top_by_score(ids, s.sum(axis=0), budget)
    if aggregate == "per_head":
        return [top_by_score(ids, s[h], budget) for h in range(s.shape[0])]
    raise ValueError(f"unknown aggregate mode {aggregate!r}")


def retained_union(selected, recent_window: int, full_len: int) -> np.ndarray:
    """kvcompress.py:126-130."""
    recent = np.arange(max(0, full_len - recent_window), full_len)
    return np.union1d(np.asarray(selected, dtype=np.intp), recent).astype(np.intp)


def compact_cache(keys, values, retained_ids, full_len, new_ids, recent_window):
    """kvcompress.py:133-147 -> (keys, values, keep)."""
    keep = retained_union(new_ids, recent_window, full_len)
    have = {int(g): i for i, g in enumerate(retained_ids)}
    try:
        rows = np.array([have[int(g)] for g in keep], dtype=np.intp)
    except KeyError as exc:
        raise InvalidIds(f"position {exc} is not present in the cache") from exc
    return np.asarray(keys)[rows], np.asarray(values)[rows], keep


@dataclass
class DecodeStats:
    """kvcompress.py:159-164."""

    events: list = field(default_factory=list)
    step_head_scores: list = field(default_factory=list)
    step_retained: list = field(default_factory=list)
    compressed: bool = False


def decode_head_step(k_arch, v_arch, q, cols):
    """model.py:233-241 for one head: returns (out, w)."""
    scores = (k_arch[cols] @ q) / math.sqrt(q.shape[0])
    w = np.exp(scores - scores.max())
    w /= w.sum()
    return w @ v_arch[cols], w


def progressive_decode_attn(k_arch, v_arch, kv_of_head, L0: int, obs_seed, comp: CompressionConfig,
                            max_new: int, q_steps, counter=None, score_log=None):
    """kvcompress.py:167-240 at attention-only shapes.

    k_arch, v_arch: [n_kv, L0 + max_new, d] fp64; rows >= L0 are the decode
    steps' appended K/V (step t appends row L0 + t before attending).
    kv_of_head: q-head -> kv-head map.  obs_seed: per q-head list of (ids, w).
    q_steps: [max_new, n_heads, d].  Returns (outs [max_new, n_heads, d], stats).
    score_log: if a list, each event appends (n_o, head, candidate ids, scores)
    (the parity tests classify a differing retained set as a top-B near-tie).
    """
    comp.validate()
    n_heads = len(kv_of_head)
    window = comp.window()
    stats = DecodeStats()
    length = L0
    heads = list(range(n_heads))
    working = {h: np.arange(length, dtype=np.intp) for h in heads}
    selected = {h: None for h in heads}
    obs_buf = {h: deque(obs_seed[h], maxlen=window) for h in heads}
    outs = np.zeros((max_new, n_heads, np.asarray(v_arch).shape[2]))
    n_answer = 0
    # first token comes from the prefill logits (kvcompress.py:199); every loop
    # iteration appends it and runs one decode step (kvcompress.py:200-228)
    while n_answer < max_new:
        n_answer += 1
        n_o = n_answer
        if comp.budget is not None and n_o >= comp.warmup and (n_o - comp.warmup) % comp.interval == 0:
            for h in heads:
                ids, scores = accumulate_scores(obs_buf[h])
                if score_log is not None:
                    score_log.append((n_o, h, ids, scores))
                picked = top_by_score(ids, scores, comp.budget)
                selected[h] = picked
                working[h] = retained_union(picked, window, length)
                kept_mass = float(scores[np.isin(ids, working[h])].sum())
                total_mass = float(scores.sum())
                stats.events.append({
                    "step": n_o,
                    "head": h,
                    "retained_ids": [int(g) for g in working[h]],
                    "score_coverage": kept_mass / total_mass if total_mass > 0 else 1.0,
                })
            stats.compressed = True
        pre_counts = {h: len(working[h]) + 1 for h in heads}
        pos = length
        length += 1
        t = n_answer - 1
        for h in heads:
            kv = kv_of_head[h]
            cols = np.append(working[h], pos)
            out, w = decode_head_step(k_arch[kv], v_arch[kv], q_steps[t][h], cols)
            if counter is not None:
                counter.add(len(cols))
            outs[t, h] = out
            obs_buf[h].append((cols, w))
            if stats.compressed:
                working[h] = retained_union(selected[h], window, length)
            else:
                working[h] = np.arange(length, dtype=np.intp)
        stats.step_head_scores.append(max(pre_counts.values()))
        stats.step_retained.append(max(len(working[h]) for h in heads))
    return outs, stats


def obswindow_select(obs_seed, budget, window: int, length: int):
    """session.py:204-230 (the obswindow baseline's one-shot selection):
    obs_seed: per (layer, head), in (layer, head) order, the list of buffered
    (ids, w) rows. Each head's scores go into a dense length-`length` array,
    the arrays are summed over all heads (numpy axis-0 order) and one top-B
    (summed_over_heads) is taken; base = retained_union(picked, W, length)
    is every head's working set. Returns (picked, base, summed)."""
    if budget is None:
        base = np.arange(length, dtype=np.intp)
        return base, base, None
    per_head = []
    for rows in obs_seed:
        ids, scores = accumulate_scores(rows)
        full = np.zeros(length)
        full[ids] = scores
        per_head.append(full)
    summed = np.stack(per_head).sum(axis=0)
    picked = top_by_score(np.arange(length), summed, budget)
    return picked, retained_union(picked, window, length), summed


def obswindow_decode_attn(k_arch, v_arch, kv_of_head, L0: int, base, max_new: int, q_steps, counter=None):
    """session.py:239-257 at attention-only shapes: every head attends to
    working = base + every position appended since (no re-selection), plus the
    new position (model.py:232-241). Returns outs [max_new, n_heads, d]."""
    n_heads = len(kv_of_head)
    working = np.asarray(base, dtype=np.intp)
    outs = np.zeros((max_new, n_heads, np.asarray(v_arch).shape[2]))
    length = L0
    for t in range(max_new):
        pos = length
        length += 1
        cols = np.append(working, pos)
        for h in range(n_heads):
            kv = kv_of_head[h]
            out, _ = decode_head_step(k_arch[kv], v_arch[kv], q_steps[t][h], cols)
            outs[t, h] = out
            if counter is not None:
                counter.add(len(cols))
        working = np.append(working, pos)
    return outs
