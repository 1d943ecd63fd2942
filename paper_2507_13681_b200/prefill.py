"""Prefill sparsification -- the reference's prefill.py API on the B200 path.

Same names, fields and errors as reference prefill.py; every compute call goes
to the CUDA library (K0 sampler, K1 scoring/line sums, K2-K4 sort/greedy/plan):
  * `Line`, `SparsePlan`               prefill.py:24-91
  * `vertical_length`, `slash_length`  prefill.py:94-99
  * `sample_rows`                      prefill.py:125-135  (K0, bit-exact)
  * `sparsify_head`                    prefill.py:363-393  (K1 + K2-K4)
  * `sparsify_layer`                   the batched form the engine uses: all
                                       q-heads of a layer in one launch chain,
                                       plans stay on the device.
Inputs may be numpy arrays (converted to bf16 on the device, which is the
precision of the B200 path) or torch CUDA bf16 tensors.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import EmptyBlock, InvalidAlpha
from .opcount import OpCounter


@dataclass(frozen=True)
class Line:
    """prefill.py:24-37."""

    kind: str  # "slash" | "vertical"
    index: int
    weight: float
    length: int
    max_cell: float


@dataclass(frozen=True)
class SparsePlan:
    """prefill.py:40-91 (same fields, same JSON)."""

    selected_slashes: frozenset
    selected_verticals: frozenset
    achieved_coverage: float
    approx_sum: float
    total_weight: float
    n_total: int

    def cost(self, n_new: int, n_total: int | None = None) -> int:
        n = self.n_total if n_total is None else n_total
        return sum(slash_length(n_new, n, d) for d in self.selected_slashes) + sum(
            vertical_length(n_new, n, c) for c in self.selected_verticals)

    def lines(self) -> frozenset:
        return frozenset([("slash", d) for d in self.selected_slashes]
                         + [("vertical", c) for c in self.selected_verticals])

    def to_json(self, head: str | None = None) -> dict:
        doc = {"slashes": sorted(self.selected_slashes), "verticals": sorted(self.selected_verticals),
               "coverage": self.achieved_coverage, "approx_sum": self.approx_sum,
               "total_weight": self.total_weight, "n_total": self.n_total}
        if head is not None:
            doc["head"] = head
        return doc

    @staticmethod
    def from_json(doc: dict) -> "SparsePlan":
        return SparsePlan(frozenset(doc["slashes"]), frozenset(doc["verticals"]), doc["coverage"],
                          doc["approx_sum"], doc["total_weight"], doc["n_total"])


def vertical_length(n_new: int, n_total: int, col: int) -> int:
    return max(0, min(n_new, n_total - col))


def slash_length(n_new: int, n_total: int, offset: int) -> int:
    return max(0, min(n_new, n_total - offset))


def plans_to_jsonl(plans: dict, path: str) -> None:
    """prefill.py:420-423."""
    with open(path, "w") as fh:
        for head in sorted(plans):
            fh.write(json.dumps(plans[head].to_json(head=head), sort_keys=True) + "\n")


# ---------------------------------------------------------------- helpers
def _dev():
    if not torch.cuda.is_available():
        from .errors import NativeLibraryMissing

        raise NativeLibraryMissing("no CUDA device: the B200 path has no CPU fallback")
    return torch.device("cuda")


def to_bf16(x) -> torch.Tensor:
    """numpy / torch -> contiguous CUDA bf16."""
    if isinstance(x, torch.Tensor):
        t = x.to(device=_dev())
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32))).to(_dev())
    return t.to(torch.bfloat16).contiguous()


def sample_size(n_new: int, rate: float, floor: int) -> int:
    import ctypes

    n = ctypes.c_int32()
    _lib.check(_lib.lib().ls_sample_size(int(n_new), float(rate), int(floor), ctypes.byref(n)),
               "sample_rows")
    return int(n.value)


def sample_rows_device(n_new: int, rate: float, floor: int, session_seed: int, turn: int, layer: int,
                       head_begin: int, n_heads: int, n_layers: int = 1, stream=None,
                       ws: "Workspace | None" = None) -> torch.Tensor:
    """K0 for layers [layer, layer+n_layers) x heads [head_begin, +n_heads):
    int32 [n_layers, n_heads, n_s] sorted local rows (squeezed to 2-D when
    n_layers == 1)."""
    n_s = sample_size(n_new, rate, floor)
    dev = _dev()
    out = torch.empty((n_layers, n_heads, n_s), dtype=torch.int32, device=dev)
    ws_n = _lib.lib().ls_sample_rows_workspace(n_layers * n_heads, n_new)
    w = (ws or Workspace()).get(ws_n)
    _lib.call("ls_sample_rows", int(session_seed) & (2 ** 64 - 1), int(turn), int(layer), int(n_layers),
              int(head_begin), int(n_heads), int(n_new), float(rate), int(floor), out.data_ptr(), w.data_ptr(),
              w.numel(), _lib.stream_ptr(stream))
    return out[0] if n_layers == 1 else out


def sample_rows(n_new: int, rate: float, floor: int, seed: int) -> np.ndarray:
    """prefill.py:125-135 with an explicit PCG64 seed (turn = -1 selects the
    raw-seed mode of the device generator)."""
    if n_new <= 0:
        raise EmptyBlock("cannot sample rows of an empty block")
    if not (0.0 < rate <= 1.0) or floor < 1:
        raise ValueError("need 0 < rate <= 1 and floor >= 1")
    rows = sample_rows_device(n_new, rate, floor, seed, -1, 0, 0, 1)
    return rows[0].cpu().numpy().astype(np.intp)


# --------------------------------------------------------------- layer API
@dataclass
class LayerPlans:
    """Device-resident plans of one layer (all heads)."""

    slash_ids: torch.Tensor   # int32 [H, n_total], sorted prefix of length counts[h, 0]
    vert_ids: torch.Tensor    # int32 [H, n_total]
    counts: torch.Tensor      # int32 [H, 2]
    coverage: torch.Tensor    # f64 [H]
    approx: torch.Tensor      # f64 [H]
    total: torch.Tensor       # f64 [H]
    score_count: torch.Tensor  # i64 [H]
    picks: torch.Tensor       # int32 [H, 2*n_total] selection order (kind<<31 | index)
    n_picks: torch.Tensor     # int32 [H]
    n_total: int

    @staticmethod
    def cat(parts: list["LayerPlans"]) -> "LayerPlans":
        """Plans of consecutive head groups -> one layer's plans (head order)."""
        if len(parts) == 1:
            return parts[0]
        f = lambda name: torch.cat([getattr(p, name) for p in parts])
        out = LayerPlans(f("slash_ids"), f("vert_ids"), f("counts"), f("coverage"), f("approx"), f("total"),
                         f("score_count"), f("picks"), f("n_picks"), parts[0].n_total)
        if all(hasattr(p, "line_arrays") for p in parts):
            out.line_arrays = tuple(torch.cat([p.line_arrays[i] for p in parts]) for i in range(4))
            out.row_stats = torch.cat([p.row_stats for p in parts])
        return out

    def to_host(self) -> list[SparsePlan]:
        sl, vt, cn = self.slash_ids.cpu().numpy(), self.vert_ids.cpu().numpy(), self.counts.cpu().numpy()
        cov, ap, tot = self.coverage.cpu().numpy(), self.approx.cpu().numpy(), self.total.cpu().numpy()
        out = []
        for h in range(cn.shape[0]):
            out.append(SparsePlan(frozenset(int(x) for x in sl[h, :cn[h, 0]]),
                                  frozenset(int(x) for x in vt[h, :cn[h, 1]]),
                                  float(cov[h]), float(ap[h]), float(tot[h]), self.n_total))
        return out

    def pick_sequences(self) -> list[list[tuple[str, int]]]:
        pk, n = self.picks.cpu().numpy(), self.n_picks.cpu().numpy()
        seqs = []
        for h in range(pk.shape[0]):
            s = []
            for code in pk[h, :n[h]]:
                code = int(code)
                s.append(("vertical", code & 0x7FFFFFFF) if code < 0 else ("slash", code))
            seqs.append(s)
        return seqs


class Workspace:
    """Grow-only device scratch buffer."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(int(nbytes * 1.25) + 4096, dtype=torch.uint8, device=_dev())
        return self.buf


def layer_desc(n_heads, n_kv_heads, d, n_new, n_total, q_head_stride, kv_head_stride, out_row_stride=0):
    return _lib.LayerDesc(int(n_heads), int(n_kv_heads), int(d), int(n_new), int(n_total),
                          int(n_total - n_new), int(q_head_stride), int(kv_head_stride), int(out_row_stride))


def sparsify_layer(q_block: torch.Tensor, k: torch.Tensor, rows: torch.Tensor, alpha: float,
                   n_new: int, n_total: int, n_kv_heads: int, q_head_stride: int | None = None,
                   kv_head_stride: int | None = None, ws: Workspace | None = None,
                   stream=None, on_scored=None, select_stream=None, plan_ready: torch.Tensor | None = None,
                   epoch: int = 0) -> LayerPlans:
    """Batched sparsify_head for every q-head of a layer (K1 + K2-K4).
    on_scored(): called once the line sums (K1) are enqueued, before the
    selection (the engine's head-group pipeline records an event there).
    select_stream: run the selection (K2-K4) there (ordered after K1 and
    before anything later on `stream` by events).
    plan_ready / epoch: int32 [H] device flags; each head's K3 CTA writes its
    plan and then sets plan_ready[h] = epoch (ls_select_lines_ready), so a
    consumer stream can start on a head as soon as its plan exists.

    q_block: bf16, head h row r at q_block.data_ptr() + (h*q_head_stride + r*d)*2
    k:       bf16 archive, kv-head j position c at (j*kv_head_stride + c*d)*2
    rows:    int32 [H, n_s] sorted local block rows.
    """
    if not (0.0 <= alpha <= 1.0):
        raise InvalidAlpha(f"alpha={alpha} outside [0, 1]")
    H, n_s = rows.shape
    d = q_block.shape[-1]
    dev = q_block.device
    qhs = q_block.stride(0) if q_head_stride is None else q_head_stride
    khs = k.stride(0) if kv_head_stride is None else kv_head_stride
    L = layer_desc(H, n_kv_heads, d, n_new, n_total, qhs, khs)
    ws = ws or Workspace()
    lib = _lib.lib()
    f64, f32, i32 = torch.float64, torch.float32, torch.int32
    v_w = torch.empty((H, n_total), dtype=f64, device=dev)
    s_w = torch.empty((H, n_total), dtype=f64, device=dev)
    v_max = torch.empty((H, n_total), dtype=f32, device=dev)
    s_max = torch.empty((H, n_total), dtype=f32, device=dev)
    row_stats = torch.empty((H, n_s, 2), dtype=f32, device=dev)
    total = torch.empty(H, dtype=f64, device=dev)
    score_count = torch.empty(H, dtype=torch.int64, device=dev)
    sp = _lib.stream_ptr(stream)
    n1 = lib.ls_score_lines_workspace(C_ref(L), n_s)
    w1 = ws.get(n1)
    _lib.call("ls_score_lines", C_ref(L), n_s, q_block.data_ptr(), k.data_ptr(), rows.data_ptr(),
              v_w.data_ptr(), v_max.data_ptr(), s_w.data_ptr(), s_max.data_ptr(), row_stats.data_ptr(),
              total.data_ptr(), score_count.data_ptr(), w1.data_ptr(), w1.numel(), sp)
    if on_scored is not None:
        on_scored()
    if select_stream is not None:
        ev = torch.cuda.Event()
        ev.record(stream)
        select_stream.wait_event(ev)
        sp = _lib.stream_ptr(select_stream)
    slash_ids = torch.empty((H, n_total), dtype=i32, device=dev)
    vert_ids = torch.empty((H, n_total), dtype=i32, device=dev)
    counts = torch.empty((H, 2), dtype=i32, device=dev)
    coverage = torch.empty(H, dtype=f64, device=dev)
    approx = torch.empty(H, dtype=f64, device=dev)
    picks = torch.empty((H, 2 * n_total), dtype=i32, device=dev)
    n_picks = torch.empty(H, dtype=i32, device=dev)
    n2 = lib.ls_select_lines_workspace(C_ref(L), n_s)
    w2 = ws.get(n2)
    if plan_ready is None:
        _lib.call("ls_select_lines", C_ref(L), n_s, float(alpha), q_block.data_ptr(), k.data_ptr(),
                  rows.data_ptr(), v_w.data_ptr(), v_max.data_ptr(), s_w.data_ptr(), s_max.data_ptr(),
                  row_stats.data_ptr(), total.data_ptr(), slash_ids.data_ptr(), vert_ids.data_ptr(),
                  counts.data_ptr(), coverage.data_ptr(), approx.data_ptr(), picks.data_ptr(),
                  n_picks.data_ptr(), w2.data_ptr(), w2.numel(), sp)
    else:
        _lib.call("ls_select_lines_ready", C_ref(L), n_s, float(alpha), q_block.data_ptr(), k.data_ptr(),
                  rows.data_ptr(), v_w.data_ptr(), v_max.data_ptr(), s_w.data_ptr(), s_max.data_ptr(),
                  row_stats.data_ptr(), total.data_ptr(), slash_ids.data_ptr(), vert_ids.data_ptr(),
                  counts.data_ptr(), coverage.data_ptr(), approx.data_ptr(), picks.data_ptr(),
                  n_picks.data_ptr(), plan_ready.data_ptr(), int(epoch), w2.data_ptr(), w2.numel(), sp)
    if select_stream is not None:
        ev = torch.cuda.Event()
        ev.record(select_stream)
        (stream if stream is not None else torch.cuda.current_stream()).wait_event(ev)
    plans = LayerPlans(slash_ids, vert_ids, counts, coverage, approx, total, score_count, picks,
                       n_picks, n_total)
    plans.line_arrays = (v_w, v_max, s_w, s_max)  # kept for diagnostics / parity tests
    plans.row_stats = row_stats
    return plans


def line_arrays_device(Qt: torch.Tensor, Kt: torch.Tensor, row_offset: int):
    """Line weights of a block over ALL its rows (every row "sampled"), one
    head: (v_w, s_w) fp64 numpy arrays of length n_total (K1 through the C ABI;
    diagnostics such as metrics.recovery_curve)."""
    n_new, n_total = Qt.shape[0], Kt.shape[0]
    dev = Qt.device
    rows = torch.arange(n_new, dtype=torch.int32, device=dev).unsqueeze(0)
    L = layer_desc(1, 1, Qt.shape[-1], n_new, n_total, 0, 0)
    f64, f32 = torch.float64, torch.float32
    v_w, s_w = torch.empty(n_total, dtype=f64, device=dev), torch.empty(n_total, dtype=f64, device=dev)
    v_max, s_max = torch.empty(n_total, dtype=f32, device=dev), torch.empty(n_total, dtype=f32, device=dev)
    row_stats = torch.empty((n_new, 2), dtype=f32, device=dev)
    total = torch.empty(1, dtype=f64, device=dev)
    count = torch.empty(1, dtype=torch.int64, device=dev)
    ws = Workspace().get(_lib.lib().ls_score_lines_workspace(C_ref(L), n_new))
    _lib.call("ls_score_lines", C_ref(L), n_new, Qt.data_ptr(), Kt.data_ptr(), rows.data_ptr(), v_w.data_ptr(),
              v_max.data_ptr(), s_w.data_ptr(), s_max.data_ptr(), row_stats.data_ptr(), total.data_ptr(),
              count.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    return v_w.cpu().numpy(), s_w.cpu().numpy()


def C_ref(x):
    import ctypes

    return ctypes.byref(x)


# ------------------------------------------------------------ drop-in API
def sparsify_head(Q_sampled, K_all, alpha: float, row_positions, counter: OpCounter | None = None) -> SparsePlan:
    """prefill.py:363-393 on the device, one head.

    Q_sampled [n_s, d] rows at global positions row_positions (any order
    accepted, sorted internally as the reference's line sums are order-free),
    K_all [n_total, d]."""
    positions = np.asarray(row_positions, dtype=np.int64)
    Qs = to_bf16(Q_sampled)
    K = to_bf16(K_all)
    if Qs.shape[0] != positions.shape[0]:
        raise EmptyBlock("one global position is required per sampled row")
    if not (0.0 <= alpha <= 1.0):
        raise InvalidAlpha(f"alpha={alpha} outside [0, 1]")
    n_total, d = K.shape
    order = np.argsort(positions, kind="stable")
    positions = positions[order]
    row_offset = int(positions.min())
    n_new = n_total - row_offset
    block = torch.zeros((n_new, d), dtype=torch.bfloat16, device=K.device)
    local = torch.from_numpy(positions - row_offset).to(K.device)
    block[local] = Qs[torch.from_numpy(order).to(K.device)]
    rows = local.to(torch.int32).reshape(1, -1).contiguous()
    plans = sparsify_layer(block.unsqueeze(0), K.unsqueeze(0), rows, alpha, n_new, n_total, 1)
    _lib.device_status(what="sparsify_head")  # NonFiniteInput / AllMaskedRow (tensor_ops.py:34-38)
    if counter is not None:
        counter.add(int(plans.score_count[0].item()))
    return plans.to_host()[0]


def line_sums_device(Q_sampled, K_all, row_positions):
    """Unsorted line weights of the sampled block (diagnostics): returns
    (v_w, v_max, s_w, s_max, total) as numpy arrays."""
    positions = np.sort(np.asarray(row_positions, dtype=np.int64))
    Qs, K = to_bf16(Q_sampled), to_bf16(K_all)
    n_total, d = K.shape
    row_offset = int(positions.min())
    n_new = n_total - row_offset
    block = torch.zeros((n_new, d), dtype=torch.bfloat16, device=K.device)
    local = torch.from_numpy(positions - row_offset).to(K.device)
    block[local] = Qs
    rows = local.to(torch.int32).reshape(1, -1).contiguous()
    plans = sparsify_layer(block.unsqueeze(0), K.unsqueeze(0), rows, 1.0, n_new, n_total, 1)
    v_w, v_max, s_w, s_max = (t[0].cpu().numpy() for t in plans.line_arrays)
    return v_w, v_max, s_w, s_max, float(plans.total[0].item())


def greedy_select_lines(slashes, verticals, alpha: float, total_weight: float, weights, positions) -> SparsePlan:
    """prefill.py:178-251 on the device with caller-provided sorted Line lists
    and a dense fp64 weight matrix as the crossing-cell source (one head)."""
    if not (0.0 <= alpha <= 1.0):
        raise InvalidAlpha(f"alpha={alpha} outside [0, 1]")
    dev = _dev()
    W = torch.as_tensor(np.ascontiguousarray(weights, dtype=np.float64), device=dev)
    pos = torch.as_tensor(np.asarray(positions, dtype=np.int32), device=dev)
    n_rows, n_total = W.shape

    def arr(lines, attr, dt):
        return torch.as_tensor(np.array([getattr(l, attr) for l in lines]), dtype=dt, device=dev)

    s = [arr(slashes, a, t) for a, t in (("index", torch.int32), ("weight", torch.float64),
                                         ("length", torch.int32), ("max_cell", torch.float64))]
    v = [arr(verticals, a, t) for a, t in (("index", torch.int32), ("weight", torch.float64),
                                           ("length", torch.int32), ("max_cell", torch.float64))]
    slash_ids = torch.empty(n_total, dtype=torch.int32, device=dev)
    vert_ids = torch.empty(n_total, dtype=torch.int32, device=dev)
    counts = torch.empty(2, dtype=torch.int32, device=dev)
    cov = torch.empty(1, dtype=torch.float64, device=dev)
    ap = torch.empty(1, dtype=torch.float64, device=dev)
    ws = torch.empty(64 * n_total * 8 + (1 << 20), dtype=torch.uint8, device=dev)
    _lib.call("ls_greedy_dense", len(slashes), *(t.data_ptr() for t in s), len(verticals),
              *(t.data_ptr() for t in v), float(alpha), float(total_weight), W.data_ptr(), pos.data_ptr(),
              n_rows, n_total, slash_ids.data_ptr(), vert_ids.data_ptr(), counts.data_ptr(), cov.data_ptr(),
              ap.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    cn = counts.cpu().numpy()
    return SparsePlan(frozenset(int(x) for x in slash_ids[:cn[0]].cpu().numpy()),
                      frozenset(int(x) for x in vert_ids[:cn[1]].cpu().numpy()),
                      float(cov.item()), float(ap.item()), float(total_weight), n_total)


__all__ = ["Line", "SparsePlan", "vertical_length", "slash_length", "sample_rows", "sample_size",
           "sample_rows_device", "sparsify_head", "sparsify_layer", "LayerPlans", "greedy_select_lines",
           "line_sums_device", "plans_to_jsonl", "math"]
