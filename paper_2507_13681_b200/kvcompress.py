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


RING_WORKING_SET = 2  # ring_dense kind: ids derived from the selection (LS_RING_WORKING_SET)


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
        # compressed steps record (n_a, lo) per observation row instead of its ids
        # (K7 derives them from the selection): only valid when every buffered
        # row is consumed before the next selection, i.e. interval >= window;
        # the owner (SessionEngine) sets it from its CompressionConfig
        self.derived_ids = False
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
        flags = (1 if pdl else 0) | (2 if self.derived_ids else 0)  # LS_DECODE_PDL, LS_DECODE_DERIVED_IDS
        _lib.call("ls_decode_step_archive", ctypes.byref(self.desc), int(layer), q_layer.data_ptr(),
                  int(q_layer.stride(0)), k_layer.data_ptr(), v_layer.data_ptr(), int(bool(compressed)),
                  int(max_cols), out.data_ptr(), int(out.dtype == torch.bfloat16), flags,
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
        kind = int(self.ring_dense[hr, slot].item())
        if kind == 1:
            return np.arange(n), w
        if kind == RING_WORKING_SET:  # ids from the current selection: sel_ids[:n_a] then lo, lo + 1, ...
            n_a, lo = (int(x) for x in self.ring_ids[hr, slot, :2].cpu().numpy())
            sel = self.sel_ids[hr, :n_a].cpu().numpy().astype(np.intp)
            return np.concatenate([sel, lo + np.arange(n - n_a)]), w
        return self.ring_ids[hr, slot, :n].cpu().numpy().astype(np.intp), w


def _i32_dev(x) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.int32), device=_dev())


def _f64_dev(x) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device=_dev())


def _check_id_range(ids: np.ndarray, what: str) -> None:
    if len(ids) and (ids.min() < 0 or ids.max() >= 2 ** 31 - 1):
        raise InvalidIds(f"{what}: ids must lie in [0, 2^31 - 1) on the device path")


def retained_union(selected, recent_window: int, full_len: int) -> np.ndarray:
    """kvcompress.py:126-130 on the device (ls_retained_union: bitmap union,
    ids emitted in ascending order)."""
    sel = np.asarray(selected, dtype=np.int64).ravel()
    _check_id_range(sel, "retained_union")
    recent_window, full_len = int(recent_window), int(full_len)
    cap = max(full_len, int(sel.max()) + 1 if len(sel) else 0, 1)
    dev = _dev()
    out = torch.empty(len(sel) + max(0, min(recent_window, full_len)) + 1, dtype=torch.int32, device=dev)
    n_out = torch.empty(1, dtype=torch.int32, device=dev)
    ws = torch.empty((cap + 31) // 32 * 4, dtype=torch.uint8, device=dev)
    sel_t = _i32_dev(sel) if len(sel) else torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("ls_retained_union", len(sel), sel_t.data_ptr(), recent_window, full_len, cap, out.data_ptr(),
              n_out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    n = int(n_out.item())
    return out[:n].cpu().numpy().astype(np.intp)


def _accumulate_device(rows):
    """ls_accumulate_scores on (ids, weights) rows -> (acc, touched) numpy."""
    ids_l, w_l = [], []
    for ids, w in rows:
        ids = np.asarray(ids, dtype=np.int64).ravel()
        w = np.asarray(w, dtype=np.float64).ravel()
        if len(w) < len(ids):
            raise SizeMismatch("observation row has fewer weights than ids")
        ids_l.append(ids)
        w_l.append(w[:len(ids)])
    if not ids_l:
        raise EmptyWindow("need at least one observation row")
    flat_ids = np.concatenate(ids_l) if ids_l else np.zeros(0, np.int64)
    _check_id_range(flat_ids, "accumulate_scores")
    flat_w = np.concatenate(w_l)
    row_ptr = np.zeros(len(ids_l) + 1, dtype=np.int64)
    row_ptr[1:] = np.cumsum([len(i) for i in ids_l])
    id_cap = int(flat_ids.max()) + 1 if len(flat_ids) else 1
    dev = _dev()
    acc = torch.empty(id_cap, dtype=torch.float64, device=dev)
    touched = torch.empty(id_cap, dtype=torch.uint8, device=dev)
    ids_t = _i32_dev(flat_ids) if len(flat_ids) else torch.zeros(1, dtype=torch.int32, device=dev)
    w_t = _f64_dev(flat_w) if len(flat_w) else torch.zeros(1, dtype=torch.float64, device=dev)
    ptr_t = torch.as_tensor(row_ptr, device=dev)  # kept alive until the kernel has read it
    _lib.call("ls_accumulate_scores", len(ids_l), ptr_t.data_ptr(), ids_t.data_ptr(), w_t.data_ptr(), id_cap,
              acc.data_ptr(), touched.data_ptr(), _lib.stream_ptr())
    return acc.cpu().numpy(), touched.cpu().numpy().astype(bool)


def accumulate_scores(buffered_rows):
    """kvcompress.py:67-83 on the device: fp64 sums in the reference's order
    (rows oldest -> newest per id); only touched ids are candidates. Ids must
    be distinct within a row (the reference's rows are working-set columns)."""
    acc, touched = _accumulate_device(list(buffered_rows))
    ids = np.nonzero(touched)[0].astype(np.intp)
    return ids, acc[ids]


def token_scores(window_rows) -> np.ndarray:
    """kvcompress.py:58-64: dense rows -> column sums, added row by row on the
    device (the order of numpy's axis-0 sum)."""
    rows = np.asarray(window_rows, dtype=np.float64)
    if rows.ndim != 2 or rows.shape[0] == 0:
        raise EmptyWindow("need at least one observation row")
    cols = np.arange(rows.shape[1])
    acc, _ = _accumulate_device([(cols, r) for r in rows])
    return acc[:rows.shape[1]]


def _top_by_score(ids: np.ndarray, scores: np.ndarray, budget: int) -> np.ndarray:
    """kvcompress.py:86-90 on the device (ls_top_by_score: radix select on
    (score desc, id asc), ids emitted ascending). Ids must be distinct."""
    ids = np.asarray(ids, dtype=np.int64).ravel()
    scores = np.asarray(scores, dtype=np.float64).ravel()
    if len(ids) != len(scores):
        raise SizeMismatch("ids and scores differ in length")
    if len(ids) == 0:
        return np.zeros(0, dtype=np.intp)
    _check_id_range(ids, "_top_by_score")
    b = int(min(int(budget), len(ids)))
    if b < 1:
        return np.zeros(0, dtype=np.intp)
    lo = int(ids.min())
    rng = int(ids.max()) - lo + 1
    dev = _dev()
    out = torch.empty(b, dtype=torch.int32, device=dev)
    n_out = torch.empty(1, dtype=torch.int32, device=dev)
    ws = torch.empty(int(_lib.lib().ls_top_by_score_workspace(rng)), dtype=torch.uint8, device=dev)
    ids_t, sc_t = _i32_dev(ids), _f64_dev(scores)  # named: a temporary's memory could be reused before the kernel runs
    _lib.call("ls_top_by_score", len(ids), ids_t.data_ptr(), sc_t.data_ptr(), b, lo, rng, out.data_ptr(),
              n_out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    if int(n_out.item()) != b:
        raise InvalidIds("_top_by_score: ids must be distinct")
    return out.cpu().numpy().astype(np.intp)


def select_topB_obs(scores, budget: int, aggregate: str = "per_head", candidate_ids=None):
    """kvcompress.py:93-109 (summed_over_heads: the head sum runs on the device
    in head order, as numpy's axis-0 sum)."""
    s = np.atleast_2d(np.asarray(scores, dtype=np.float64))
    ids = np.arange(s.shape[1]) if candidate_ids is None else np.asarray(candidate_ids)
    if len(ids) != s.shape[1]:
        raise SizeMismatch("candidate_ids length must match score columns")
    if aggregate == "summed_over_heads":
        return _top_by_score(ids, token_scores(s), budget)
    if aggregate == "per_head":
        return [_top_by_score(ids, s[h], budget) for h in range(s.shape[0])]
    raise ValueError(f"unknown aggregate mode {aggregate!r}")


def ground_truth_topB(output_rows_per_head, budget: int) -> np.ndarray:
    """kvcompress.py:112-116 on the device: per-head column sums of the output
    rows' attention, summed over heads, top-B."""
    stacked = np.stack([token_scores(rows) for rows in output_rows_per_head])
    return select_topB_obs(stacked, budget, aggregate="summed_over_heads")


def overlap_rate(selected, truth, budget: int) -> float:
    """kvcompress.py:119-123: |a & b| / B, with |a & b| = |a| + |b| - |a U b|
    and the union on the device."""
    a = np.unique(np.asarray(selected, dtype=np.int64))
    b = np.unique(np.asarray(truth, dtype=np.int64))
    if len(a) != budget or len(b) != budget:
        raise SizeMismatch(f"both sets must have exactly {budget} elements")
    u = retained_union(np.concatenate([a, b]), 0, 0)
    return (len(a) + len(b) - len(u)) / budget


def compact_cache(head: KVCacheHead, retained_ids, recent_window: int) -> KVCacheHead:
    """kvcompress.py:133-147: keep = retained_union(...) (device), then the K8
    gather (ls_kv_compact) of those rows from the head's cache; a kept id the
    cache does not hold raises InvalidIds."""
    keep = retained_union(retained_ids, recent_window, head.full_len)
    keys = np.ascontiguousarray(head.keys)
    vals = np.ascontiguousarray(head.values)
    n_src, n_keep = len(head.retained_ids), len(keep)
    dev = _dev()

    def rows_dev(a):
        """[n_src, ...] -> uint8 rows padded to 16 bytes (the vectorised gather)."""
        rb = int(np.prod(a.shape[1:])) * a.dtype.itemsize if a.ndim > 1 else a.dtype.itemsize
        b = np.zeros((max(n_src, 1), rb + (-rb) % 16), dtype=np.uint8)
        if n_src:
            b[:n_src, :rb] = np.ascontiguousarray(a).reshape(n_src, -1).view(np.uint8).reshape(n_src, rb)
        return torch.as_tensor(b, device=dev), rb

    (src_k, kb), (src_v, vb) = rows_dev(keys), rows_dev(vals)
    dst_k = torch.empty((max(n_keep, 1), src_k.shape[1]), dtype=torch.uint8, device=dev)
    dst_v = torch.empty((max(n_keep, 1), src_v.shape[1]), dtype=torch.uint8, device=dev)
    status = torch.empty(1, dtype=torch.int32, device=dev)
    src_ids = _i32_dev(head.retained_ids) if n_src else torch.zeros(1, dtype=torch.int32, device=dev)
    keep_t = _i32_dev(keep) if n_keep else torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("ls_kv_compact", n_src, src_ids.data_ptr(), src_k.data_ptr(), src_v.data_ptr(), n_keep,
              keep_t.data_ptr(), src_k.shape[1], src_v.shape[1], dst_k.data_ptr(), dst_v.data_ptr(),
              status.data_ptr(), _lib.stream_ptr())
    st = int(status.item())
    if st:
        raise InvalidIds(f"position {int(keep[st - 1])} is not present in the cache")

    def back(t, like, rb):
        raw = np.ascontiguousarray(t[:n_keep, :rb].cpu().numpy())
        return raw.view(like.dtype).reshape((n_keep,) + like.shape[1:])

    cls = type(head) if hasattr(type(head), "__dataclass_fields__") else KVCacheHead  # the caller's class
    return cls(keys=back(dst_k, keys, kb), values=back(dst_v, vals, vb), retained_ids=keep, full_len=head.full_len)


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
           "select_topB_obs", "_top_by_score", "retained_union", "compact_cache", "ground_truth_topB",
           "overlap_rate", "progressive_decode", "DecodeStack"]
