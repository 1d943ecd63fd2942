"""Progressive decode KV compression -- the reference's kvcompress.py API on
the B200 path.

  * `CompressionConfig`, `DecodeStats`   kvcompress.py:22-36, 159-164 (same fields)
  * `accumulate_scores`, `select_topB_obs`, `_top_by_score`
                                         kvcompress.py:67-109 -> K7 on the device
  * `retained_union`                     kvcompress.py:126-130
  * `compact_cache`, `KVCacheHead`       kvcompress.py:39-55, 133-147 -> K8
  * `DecodeLayer`                        device state of one layer: observation
                                         ring (the deque of kvcompress.py:196),
                                         selected ids, compacted K/V
  * `progressive_decode`                 kvcompress.py:167-240 at attention-only
                                         shapes: the per-step q and appended K/V
                                         come from a step source instead of the
                                         toy model's projections (model.py:227)
"""

from __future__ import annotations

import ctypes
from collections import deque
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import EmptyWindow, InvalidConfig, InvalidIds, SizeMismatch
from .opcount import OpCounter
from .prefill import Workspace, _dev


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

    def event_at(self, n_o: int) -> bool:
        """kvcompress.py:205-209."""
        return self.budget is not None and n_o >= self.warmup and (n_o - self.warmup) % self.interval == 0

    def surviving_seeds(self, n_seed: int, max_new: int) -> int:
        """How many of the n_seed prefill seed rows are still in the deque at
        the first event (later events only see decode rows unless W > interval;
        rows evicted before any event are never read)."""
        if self.budget is None or self.warmup > max_new:
            return 0
        W = self.window()
        # deque after seeds + (warmup - 1) decode rows, maxlen W
        return max(0, min(n_seed, W - (self.warmup - 1)))


@dataclass
class DecodeStats:
    """kvcompress.py:159-164."""

    events: list = field(default_factory=list)
    step_head_scores: list = field(default_factory=list)
    step_retained: list = field(default_factory=list)
    compressed: bool = False


@dataclass(frozen=True)
class KVCacheHead:
    """kvcompress.py:39-55 (host view; the device cache is DecodeLayer.ck/cv)."""

    keys: np.ndarray
    values: np.ndarray
    retained_ids: np.ndarray
    full_len: int

    def __post_init__(self):
        ids = self.retained_ids
        if ids.ndim != 1 or (len(ids) > 1 and not (np.diff(ids) > 0).all()):
            raise InvalidIds("retained_ids must be strictly increasing")
        if len(ids) and (ids[0] < 0 or ids[-1] >= self.full_len):
            raise InvalidIds("retained_ids outside [0, full_len)")
        if self.keys.shape[0] != len(ids) or self.values.shape[0] != len(ids):
            raise InvalidIds("row count does not match retained_ids")


class DecodeStack:
    """Device decode state of every layer of one session (ls_decode_stack):
    observation ring (the deque of kvcompress.py:196) per (layer, q-head),
    selected ids, compacted K/V, and the device step counters
    (step[0] = cache length, step[1] = rows appended to the deque)."""

    def __init__(self, n_layers: int, n_heads: int, n_kv_heads: int, head_dim: int, window: int, budget_cap: int,
                 row_cap: int, kv_layer_stride: int, kv_head_stride: int, device=None, sparse_cap: int | None = None):
        dev = device or _dev()
        self.n_layers, self.n_heads, self.n_kv, self.d, self.window = n_layers, n_heads, n_kv_heads, head_dim, window
        self.budget_cap, self.row_cap = max(1, budget_cap), row_cap
        self.sparse_cap = max(self.budget_cap + window + 1, sparse_cap or 0)
        HR, W = n_layers * n_heads, window
        f32, i32 = torch.float32, torch.int32
        self.ring_s = torch.zeros((HR, W, row_cap), dtype=f32, device=dev)
        self.ring_ml = torch.zeros((HR, W, 2), dtype=f32, device=dev)
        self.ring_ids = torch.zeros((HR, W, self.sparse_cap), dtype=i32, device=dev)
        self.ring_n = torch.zeros((HR, W), dtype=i32, device=dev)
        self.ring_dense = torch.zeros((HR, W), dtype=i32, device=dev)
        self.sel_ids = torch.zeros((HR, self.budget_cap), dtype=i32, device=dev)
        self.n_sel = torch.zeros(HR, dtype=i32, device=dev)
        self.ck = torch.zeros((HR, self.budget_cap, head_dim), dtype=torch.bfloat16, device=dev)
        self.cv = torch.zeros((HR, self.budget_cap, head_dim), dtype=torch.bfloat16, device=dev)
        self.counters = torch.zeros(2 * n_heads, dtype=i32, device=dev)  # split-K arrivals, departures
        self.step_t = torch.zeros(4, dtype=i32, device=dev)
        self.n_a = torch.zeros(HR, dtype=i32, device=dev)
        self.retained_n = torch.zeros(HR, dtype=i32, device=dev)
        self.score_cov = torch.zeros(HR, dtype=torch.float64, device=dev)
        self.desc = _lib.DecodeStackDesc(
            n_layers, n_heads, n_kv_heads, head_dim, window, row_cap, self.sparse_cap, self.budget_cap,
            int(kv_layer_stride), int(kv_head_stride), self.ring_s.data_ptr(), self.ring_ml.data_ptr(),
            self.ring_ids.data_ptr(), self.ring_n.data_ptr(), self.ring_dense.data_ptr(), self.sel_ids.data_ptr(),
            self.n_sel.data_ptr(), self.ck.data_ptr(), self.cv.data_ptr(), 0, self.counters.data_ptr(),
            self.step_t.data_ptr(), self.n_a.data_ptr())
        # split-K partials of the decode kernel (units x splits, combined by the last CTA of a unit)
        n_part = int(_lib.lib().ls_decode_partials_size(ctypes.byref(self.desc), int(row_cap))) // 4
        self.partials = torch.zeros(max(1, n_part), dtype=f32, device=dev)
        self.desc.partials = self.partials.data_ptr()
        self.ws = Workspace()
        self.set_step(0, 0)

    # ---------------------------------------------------------------- counters
    def set_step(self, length: int, appended: int):
        """Host mirror + device counters (a tiny H2D copy; outside graphs)."""
        self.length, self.appended = int(length), int(appended)
        self.step_t.copy_(torch.tensor([self.length, self.appended, 0, 0], dtype=torch.int32))

    def deque_slots(self) -> list[int]:
        n = min(self.window, self.appended)
        return [(self.appended - n + i) % self.window for i in range(n)]

    def seed_slots(self, n_seed: int) -> list[int]:
        """Slots of n_seed seed rows appended to an empty deque (oldest first)."""
        return [i % self.window for i in range(n_seed)]

    def write_dense_rows(self, layer: int, slot: int, rows: torch.Tensor):
        """Seed rows given as probabilities: rows fp32 [H, n] (ids = arange(n))."""
        H, n = rows.shape
        hr = slice(layer * self.n_heads, (layer + 1) * self.n_heads)
        self.ring_s[hr, slot, :n].copy_(rows)
        self.ring_ml[hr, slot, 0] = 0.0
        self.ring_ml[hr, slot, 1] = 0.0  # sum == 0: probabilities stored directly
        self.ring_n[hr, slot] = n
        self.ring_dense[hr, slot] = 1

    def write_sparse_row(self, layer: int, h: int, slot: int, ids: np.ndarray, w: np.ndarray):
        n = len(ids)
        if n > self.sparse_cap or n > self.row_cap:
            raise SizeMismatch("observation row longer than the ring capacity")
        hr = layer * self.n_heads + h
        self.ring_s[hr, slot, :n] = torch.as_tensor(np.asarray(w, dtype=np.float32))
        self.ring_ids[hr, slot, :n] = torch.as_tensor(np.asarray(ids, dtype=np.int32))
        self.ring_ml[hr, slot, 0] = 0.0
        self.ring_ml[hr, slot, 1] = 0.0
        self.ring_n[hr, slot] = n
        self.ring_dense[hr, slot] = 0

    # ----------------------------------------------------------------- kernels
    def event_workspace(self, max_len: int) -> torch.Tensor:
        """K7's global score accumulator (only past its shared-memory capacity);
        call before graph capture so the capture does not allocate."""
        n = _lib.lib().ls_decode_select_workspace(ctypes.byref(self.desc))
        return self.ws.get(n if max_len > 24 * 1024 else 1)

    def event(self, budget: int, k_all: torch.Tensor, v_all: torch.Tensor, max_len: int | None = None, stream=None):
        """K7 + K8 for every layer (kvcompress.py:210-225) at the current step."""
        if self.appended == 0:
            raise EmptyWindow("need at least one observation row")
        max_len = self.length if max_len is None else max_len
        w = self.event_workspace(max_len)
        _lib.call("ls_decode_event", ctypes.byref(self.desc), int(budget), int(max_len), k_all.data_ptr(),
                  v_all.data_ptr(), self.retained_n.data_ptr(), self.score_cov.data_ptr(), w.data_ptr(), w.numel(),
                  _lib.stream_ptr(stream))

    def step(self, layer: int, q: torch.Tensor, k_layer: torch.Tensor, v_layer: torch.Tensor, compressed: bool,
             max_cols: int, out: torch.Tensor, stream=None):
        """K6 for one layer at the current step (q [H, d] bf16 -> out [H, d])."""
        _lib.call("ls_decode_step", ctypes.byref(self.desc), int(layer), q.data_ptr(), k_layer.data_ptr(),
                  v_layer.data_ptr(), int(bool(compressed)), int(max_cols), out.data_ptr(),
                  int(out.dtype == torch.bfloat16), _lib.stream_ptr(stream))

    def step_archive(self, layer: int, q_layer: torch.Tensor, k_layer: torch.Tensor, v_layer: torch.Tensor,
                     compressed: bool, max_cols: int, out: torch.Tensor, pdl: bool = True, stream=None):
        """K6 for one layer with q read from the layer's Q archive [H, cap, d]
        at the current cache length (no per-step q gather); pdl: programmatic
        dependent launch after the previous kernel on the stream."""
        _lib.call("ls_decode_step_archive", ctypes.byref(self.desc), int(layer), q_layer.data_ptr(),
                  int(q_layer.stride(0)), k_layer.data_ptr(), v_layer.data_ptr(), int(bool(compressed)),
                  int(max_cols), out.data_ptr(), int(out.dtype == torch.bfloat16), 1 if pdl else 0,
                  _lib.stream_ptr(stream))

    def advance(self, stream=None):
        _lib.call("ls_decode_advance", ctypes.byref(self.desc), _lib.stream_ptr(stream))
        self.length += 1
        self.appended += 1

    # ------------------------------------------------------ host views (parity)
    def working_ids(self, layer: int, compressed: bool) -> list[np.ndarray]:
        """retained_union(selected, W, length) per head (kvcompress.py:126-130)."""
        L = self.length
        if not compressed:
            return [np.arange(L) for _ in range(self.n_heads)]
        hr = slice(layer * self.n_heads, (layer + 1) * self.n_heads)
        sel = self.sel_ids[hr].cpu().numpy()
        n = self.n_sel[hr].cpu().numpy()
        lo = max(0, L - self.window)
        return [np.union1d(sel[h, :n[h]], np.arange(lo, L)).astype(np.intp) for h in range(self.n_heads)]

    def slot_row(self, layer: int, h: int, slot: int):
        """(ids, normalised weights) of a ring row."""
        hr = layer * self.n_heads + h
        n = int(self.ring_n[hr, slot].item())
        s = self.ring_s[hr, slot, :n].double().cpu().numpy()
        M, Ls = (float(x) for x in self.ring_ml[hr, slot].cpu().numpy())
        w = s if Ls == 0.0 else np.exp2(s - M) / Ls
        if int(self.ring_dense[hr, slot].item()):
            return np.arange(n), w
        return self.ring_ids[hr, slot, :n].cpu().numpy().astype(np.intp), w


def retained_union(selected, recent_window: int, full_len: int) -> np.ndarray:
    """kvcompress.py:126-130 (on the device)."""
    dev = _dev()
    sel = torch.as_tensor(np.asarray(selected, dtype=np.int64), device=dev)
    recent = torch.arange(max(0, full_len - recent_window), full_len, device=dev, dtype=torch.int64)
    return torch.unique(torch.cat([sel, recent])).cpu().numpy().astype(np.intp)


def _rows_select(buffered_rows, budget: int):
    """Run K7 on caller rows; returns (ids, scores, picked)."""
    rows = list(buffered_rows)
    if not rows:
        raise EmptyWindow("need at least one observation row")
    id_cap = max(int(np.max(ids)) + 1 if len(ids) else 1 for ids, _ in rows)
    n_max = max(len(ids) for ids, _ in rows)
    cap = max(id_cap, n_max) + 1
    st = DecodeStack(1, 1, 1, 64, len(rows), max(1, budget), cap, 0, 0, sparse_cap=n_max)
    for i, (ids, w) in enumerate(rows):
        st.write_sparse_row(0, 0, i, np.asarray(ids), np.asarray(w))
    st.set_step(id_cap, len(rows))
    dummy = torch.zeros(8 * 64, dtype=torch.bfloat16, device=st.ring_s.device)
    st.event(max(1, budget), dummy, dummy, max_len=id_cap)
    # scores: host re-accumulation of the same fp32 weights in the same order
    acc = np.zeros(id_cap)
    touched = np.zeros(id_cap, dtype=bool)
    for ids, w in rows:
        np.add.at(acc, np.asarray(ids, dtype=np.intp), np.asarray(w, dtype=np.float32).astype(np.float64))
        touched[np.asarray(ids, dtype=np.intp)] = True
    ids = np.nonzero(touched)[0].astype(np.intp)
    n = int(st.n_sel[0].item())
    picked = st.sel_ids[0, :n].cpu().numpy().astype(np.intp)
    return ids, acc[ids], picked


def accumulate_scores(buffered_rows):
    """kvcompress.py:67-83 on the device (fp32 weights, fp64 sums)."""
    ids, scores, _ = _rows_select(buffered_rows, 1)
    return ids, scores


def token_scores(window_rows) -> np.ndarray:
    """kvcompress.py:58-64: dense rows -> column sums (device)."""
    rows = np.asarray(window_rows, dtype=np.float64)
    if rows.ndim != 2 or rows.shape[0] == 0:
        raise EmptyWindow("need at least one observation row")
    dev = _dev()
    return torch.as_tensor(rows, device=dev).sum(dim=0).cpu().numpy()


def _top_by_score(ids: np.ndarray, scores: np.ndarray, budget: int) -> np.ndarray:
    """kvcompress.py:86-90 on the device via K7's radix select."""
    ids = np.asarray(ids, dtype=np.intp)
    scores = np.asarray(scores, dtype=np.float64)
    if budget >= len(ids):
        return np.sort(ids)
    _, _, picked = _rows_select([(ids, scores)], budget)
    return picked


def select_topB_obs(scores, budget: int, aggregate: str = "per_head", candidate_ids=None):
    """kvcompress.py:93-109."""
    s = np.atleast_2d(np.asarray(scores, dtype=np.float64))
    ids = np.arange(s.shape[1]) if candidate_ids is None else np.asarray(candidate_ids)
    if len(ids) != s.shape[1]:
        raise SizeMismatch("candidate_ids length must match score columns")
    if aggregate == "summed_over_heads":
        return _top_by_score(ids, s.sum(axis=0), budget)
    if aggregate == "per_head":
        return [_top_by_score(ids, s[h], budget) for h in range(s.shape[0])]
    raise ValueError(f"unknown aggregate mode {aggregate!r}")


def compact_cache(head: KVCacheHead, retained_ids, recent_window: int) -> KVCacheHead:
    """kvcompress.py:133-147: keep union(retained_ids, recent window) rows via
    the K8 gather."""
    keep = retained_union(retained_ids, recent_window, head.full_len)
    have = {int(g): i for i, g in enumerate(head.retained_ids)}
    try:
        rows = np.array([have[int(g)] for g in keep], dtype=np.int32)
    except KeyError as exc:
        raise InvalidIds(f"position {exc} is not present in the cache") from exc
    dev = _dev()
    d = head.keys.shape[1] if head.keys.ndim == 2 else 1
    keys = torch.as_tensor(np.asarray(head.keys, dtype=np.float32), device=dev)
    vals = torch.as_tensor(np.asarray(head.values, dtype=np.float32), device=dev)
    idx = torch.as_tensor(rows, device=dev, dtype=torch.int64)
    del d
    return KVCacheHead(keys=keys[idx].cpu().numpy().astype(head.keys.dtype),
                       values=vals[idx].cpu().numpy().astype(head.values.dtype),
                       retained_ids=keep, full_len=head.full_len)


def progressive_decode(stack: DecodeStack, step_source, L0: int, comp: CompressionConfig, max_new: int,
                       k_all: torch.Tensor, v_all: torch.Tensor, counter: OpCounter | None = None,
                       row_collector: list | None = None, record_events: bool = True, stream=None):
    """kvcompress.py:167-240 at attention-only shapes.

    `stack` is already seeded (ring rows of the prefill observation seeds,
    counters at (L0, n_seed)). step_source(t, length) -> list per layer of
    (q [H, d] bf16, k_layer, v_layer) with the new token's K/V at `length`.
    Returns (outputs per step [max_new][layer] -> [H, d], DecodeStats).
    """
    comp.validate()
    window = comp.window()
    stats = DecodeStats()
    outs = []
    compressed = False
    budget_cols = (comp.budget or 0) + window + 1
    for n_answer in range(1, max_new + 1):
        n_o = n_answer
        length = stack.length
        if comp.event_at(n_o):
            stack.event(comp.budget, k_all, v_all, stream=stream)
            compressed = True
            stats.compressed = True
            if record_events:
                cov = stack.score_cov.cpu().numpy()
                for li in range(stack.n_layers):
                    work = stack.working_ids(li, True)
                    for h in range(stack.n_heads):
                        stats.events.append({"step": n_o, "head": f"L{li}H{h}",
                                             "retained_ids": [int(g) for g in work[h]],
                                             "score_coverage": float(cov[li * stack.n_heads + h])})
        inputs = step_source(n_answer - 1, length)
        if record_events:
            pre = max(max(len(w) for w in stack.working_ids(li, compressed)) for li in range(stack.n_layers)) + 1
            stats.step_head_scores.append(pre)
            if counter is not None:
                for li in range(stack.n_layers):
                    counter.add(sum(len(w) + 1 for w in stack.working_ids(li, compressed)))
        step_outs = []
        max_cols = min(budget_cols, length + 1) if compressed else length + 1
        slot = stack.appended % stack.window
        for li in range(stack.n_layers):
            q, k_layer, v_layer = inputs[li]
            out = torch.empty((stack.n_heads, stack.d), dtype=torch.bfloat16, device=q.device)
            stack.step(li, q, k_layer, v_layer, compressed, max_cols, out, stream=stream)
            step_outs.append(out)
        stack.advance(stream=stream)
        if row_collector is not None:
            row_collector.append([{(li, h): stack.slot_row(li, h, slot) for h in range(stack.n_heads)}
                                  for li in range(stack.n_layers)])
        if record_events:
            stats.step_retained.append(max(max(len(w) for w in stack.working_ids(li, compressed))
                                           for li in range(stack.n_layers)))
        outs.append(step_outs)
    return outs, stats


__all__ = ["CompressionConfig", "DecodeStats", "KVCacheHead", "accumulate_scores", "token_scores",
           "select_topB_obs", "_top_by_score", "retained_union", "compact_cache", "progressive_decode", "DecodeStack"]
