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


class DecodeLayer:
    """Device decode state of one attention layer (all q-heads)."""

    def __init__(self, n_heads: int, n_kv_heads: int, head_dim: int, window: int, budget_cap: int,
                 row_cap: int, kv_head_stride: int, device=None):
        dev = device or _dev()
        self.n_heads, self.n_kv, self.d, self.window = n_heads, n_kv_heads, head_dim, window
        self.budget_cap, self.row_cap = max(1, budget_cap), row_cap
        self.sparse_cap = self.budget_cap + window + 1
        H, W = n_heads, window
        self.ring_w = torch.zeros((H, W, row_cap), dtype=torch.float32, device=dev)
        self.ring_ids = torch.zeros((H, W, self.sparse_cap), dtype=torch.int32, device=dev)
        self.ring_n = torch.zeros((H, W), dtype=torch.int32, device=dev)
        self.ring_dense = torch.zeros((H, W), dtype=torch.int32, device=dev)
        self.sel_ids = torch.zeros((H, self.budget_cap), dtype=torch.int32, device=dev)
        self.n_sel = torch.zeros(H, dtype=torch.int32, device=dev)
        self.ck = torch.zeros((H, self.budget_cap, head_dim), dtype=torch.bfloat16, device=dev)
        self.cv = torch.zeros((H, self.budget_cap, head_dim), dtype=torch.bfloat16, device=dev)
        self.retained_n = torch.zeros(H, dtype=torch.int32, device=dev)
        self.score_cov = torch.zeros(H, dtype=torch.float64, device=dev)
        self.desc = _lib.DecodeStateDesc(
            n_heads, n_kv_heads, head_dim, window, row_cap, self.sparse_cap, self.budget_cap, int(kv_head_stride),
            self.ring_w.data_ptr(), self.ring_ids.data_ptr(), self.ring_n.data_ptr(), self.ring_dense.data_ptr(),
            self.sel_ids.data_ptr(), self.n_sel.data_ptr(), self.ck.data_ptr(), self.cv.data_ptr())
        self.ws = Workspace()
        self.reset()

    def reset(self):
        self.appended = 0
        self.order: deque = deque(maxlen=self.window)

    # ring / deque bookkeeping (kvcompress.py:196, 233)
    def push_slot(self) -> int:
        slot = self.appended % self.window
        self.appended += 1
        self.order.append(slot)
        return slot

    def seed_slots(self, n_seed: int) -> list[int]:
        """Append n_seed seed rows; returns their slots (oldest first)."""
        return [self.push_slot() for _ in range(n_seed)]

    def write_dense_row(self, slot: int, rows: torch.Tensor):
        """rows: fp32 [H, n] dense observation rows (ids = arange(n))."""
        n = rows.shape[1]
        self.ring_w[:, slot, :n].copy_(rows)
        self.ring_n[:, slot] = n
        self.ring_dense[:, slot] = 1

    def write_sparse_row(self, slot: int, h: int, ids: np.ndarray, w: np.ndarray):
        n = len(ids)
        if n > self.sparse_cap:
            raise SizeMismatch("observation row longer than the sparse ring capacity")
        self.ring_w[h, slot, :n] = torch.as_tensor(np.asarray(w, dtype=np.float32))
        self.ring_ids[h, slot, :n] = torch.as_tensor(np.asarray(ids, dtype=np.int32))
        self.ring_n[h, slot] = n
        self.ring_dense[h, slot] = 0

    def event(self, length: int, budget: int, stream=None):
        """K7 + K8: select per head from the buffered rows, compact K/V."""
        if not self.order:
            raise EmptyWindow("need at least one observation row")
        order = torch.tensor(list(self.order), dtype=torch.int32, device=self.ring_w.device)
        n = _lib.lib().ls_decode_select_workspace(ctypes.byref(self.desc), length)
        w = self.ws.get(n)
        _lib.call("ls_decode_select", ctypes.byref(self.desc), order.data_ptr(), len(self.order), int(length),
                  int(budget), self.retained_n.data_ptr(), self.score_cov.data_ptr(), w.data_ptr(), w.numel(),
                  _lib.stream_ptr(stream))
        self._order_keepalive = order
        return w

    def compact(self, k_arch: torch.Tensor, v_arch: torch.Tensor, stream=None):
        _lib.call("ls_kv_compact", ctypes.byref(self.desc), k_arch.data_ptr(), v_arch.data_ptr(),
                  _lib.stream_ptr(stream))

    def step(self, q: torch.Tensor, k_arch: torch.Tensor, v_arch: torch.Tensor, length: int, compressed: bool,
             out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """K6: attend one new token (K/V already at position `length` of the
        archive); q [H, d] bf16 -> out [H, d]."""
        slot = self.push_slot()
        if out is None:
            out = torch.empty((self.n_heads, self.d), dtype=torch.bfloat16, device=q.device)
        n = _lib.lib().ls_decode_attention_workspace(ctypes.byref(self.desc), length)
        w = self.ws.get(n)
        _lib.call("ls_decode_attention", ctypes.byref(self.desc), q.data_ptr(), k_arch.data_ptr(),
                  v_arch.data_ptr(), int(length), int(bool(compressed)), slot, out.data_ptr(),
                  int(out.dtype == torch.bfloat16), w.data_ptr(), w.numel(), _lib.stream_ptr(stream))
        return out

    # ------------------------------------------------------ host views (parity)
    def working_ids(self, length: int, compressed: bool) -> list[np.ndarray]:
        """retained_union(selected, W, length) per head (kvcompress.py:126-130)."""
        if not compressed:
            return [np.arange(length) for _ in range(self.n_heads)]
        sel = self.sel_ids.cpu().numpy()
        n = self.n_sel.cpu().numpy()
        lo = max(0, length - self.window)
        return [np.union1d(sel[h, :n[h]], np.arange(lo, length)).astype(np.intp) for h in range(self.n_heads)]

    def slot_row(self, h: int, slot: int):
        n = int(self.ring_n[h, slot].item())
        w = self.ring_w[h, slot, :n].double().cpu().numpy()
        if int(self.ring_dense[h, slot].item()):
            return np.arange(n), w
        return self.ring_ids[h, slot, :n].cpu().numpy().astype(np.intp), w


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
    layer = DecodeLayer(1, 1, 64, len(rows), max(1, budget), max(id_cap, n_max) + 1, 0)
    layer.sparse_cap = max(layer.sparse_cap, n_max)
    if n_max > layer.ring_ids.shape[2]:
        layer.ring_ids = torch.zeros((1, len(rows), n_max), dtype=torch.int32, device=layer.ring_w.device)
        layer.desc.ring_ids = layer.ring_ids.data_ptr()
        layer.desc.sparse_cap = n_max
        layer.sparse_cap = n_max
    for ids, w in rows:
        slot = layer.push_slot()
        layer.write_sparse_row(slot, 0, np.asarray(ids), np.asarray(w))
    ws = layer.event(id_cap, max(1, budget))
    torch.cuda.synchronize()
    acc = ws[: 8 * layer.row_cap].view(torch.float64)[:id_cap].cpu().numpy()
    off = (8 * layer.row_cap + 255) // 256 * 256
    touched = ws[off: off + id_cap].cpu().numpy().astype(bool)
    ids = np.nonzero(touched)[0].astype(np.intp)
    n = int(layer.n_sel[0].item())
    picked = layer.sel_ids[0, :n].cpu().numpy().astype(np.intp)
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


def progressive_decode(layers: list[DecodeLayer], step_source, L0: int, comp: CompressionConfig, max_new: int,
                       counter: OpCounter | None = None, row_collector: list | None = None,
                       record_events: bool = True, stream=None):
    """kvcompress.py:167-240 at attention-only shapes.

    layers: one DecodeLayer per attention layer, already seeded (ring holds the
    prefill observation seeds). step_source(t, length) -> list per layer of
    (q [H, d] bf16, k_arch, v_arch) with the new token's K/V at `length`.
    Returns (outputs per step [max_new][layer] -> [H, d], DecodeStats).
    """
    comp.validate()
    window = comp.window()
    stats = DecodeStats()
    length = L0
    outs = []
    compressed = False
    for n_answer in range(1, max_new + 1):
        n_o = n_answer
        inputs = step_source(n_answer - 1, length)
        if comp.event_at(n_o):
            for li, layer in enumerate(layers):
                layer.event(length, comp.budget, stream=stream)
                _, k_arch, v_arch = inputs[li]
                layer.compact(k_arch, v_arch, stream=stream)
                if record_events:
                    work = layer.working_ids(length, True)
                    cov = layer.score_cov.cpu().numpy()
                    for h in range(layer.n_heads):
                        stats.events.append({"step": n_o, "head": f"L{li}H{h}",
                                             "retained_ids": [int(g) for g in work[h]],
                                             "score_coverage": float(cov[h])})
            compressed = True
            stats.compressed = True
        step_outs = []
        for li, layer in enumerate(layers):
            q, k_arch, v_arch = inputs[li]
            step_outs.append(layer.step(q, k_arch, v_arch, length, compressed, stream=stream))
        if record_events:
            pre = max(len(w) for w in layers[0].working_ids(length, compressed)) + 1 if compressed else length + 1
            if compressed:
                pre = max(max(len(w) for w in layer.working_ids(length, True)) for layer in layers) + 1
            stats.step_head_scores.append(pre)
            if counter is not None:
                for layer in layers:
                    counter.add(sum(len(w) + 1 for w in layer.working_ids(length, compressed)))
        if row_collector is not None:
            row_collector.append([{(li, h): layer.slot_row(h, layer.order[-1]) for h in range(layer.n_heads)}
                                  for li, layer in enumerate(layers)])
        length += 1
        if record_events:
            stats.step_retained.append(max(max(len(w) for w in layer.working_ids(length, compressed))
                                           for layer in layers))
        outs.append(step_outs)
    return outs, stats


__all__ = ["CompressionConfig", "DecodeStats", "KVCacheHead", "DecodeLayer", "accumulate_scores", "token_scores",
           "select_topB_obs", "_top_by_score", "retained_union", "compact_cache", "progressive_decode"]
