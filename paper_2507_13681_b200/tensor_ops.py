"""Attention primitives -- the reference's tensor_ops.py API on the B200 path.

  * `masked_sparse_attention`  tensor_ops.py:141-183 -> K5 (vertical/slash
                               sparse attention, exact `_row_columns` cells
                               incl. the diagonal fallback)
  * `scaled_dot_attention`     tensor_ops.py:104-127 -> dense causal K5 mode
  * `AttentionBlock`           tensor_ops.py:43-88, host-side validated view
                               of dense weights (diagnostics only; the device
                               path never materialises it unless asked)
  * `attention_layer`          the batched form: all q-heads of a layer,
                               plans on the device, token-major output
                               [n_new, H, d] (the head concat of model.py:259)
Inputs may be numpy (rounded to bf16 on the device) or CUDA bf16 tensors.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from types import SimpleNamespace

import numpy as np
import torch

from . import _lib
from .errors import DimensionMismatch, EmptyPlan, NonFiniteInput
from .opcount import OpCounter
from .prefill import C_ref, Workspace, layer_desc, to_bf16


@dataclass(frozen=True)
class AttentionBlock:
    """tensor_ops.py:43-88 (same validation)."""

    weights: np.ndarray
    row_offset: int

    def __post_init__(self):
        w = self.weights
        if w.ndim != 2:
            raise DimensionMismatch("weights must be 2-D")
        n_new, n_total = w.shape
        if n_new > n_total:
            raise DimensionMismatch(f"n_new={n_new} exceeds n_total={n_total}")
        if self.row_offset != n_total - n_new:
            raise DimensionMismatch(f"row_offset={self.row_offset} != n_total-n_new={n_total - n_new}")
        if not np.isfinite(w).all():
            raise NonFiniteInput("attention weights must be finite")
        if np.abs(w.sum(axis=1) - 1.0).max() > 1e-6:  # fp32 device weights: 1e-6 instead of 1e-9
            raise DimensionMismatch("attention rows must each sum to 1")
        cols = np.arange(n_total)
        rows = self.row_offset + np.arange(n_new)
        if np.any(w[cols[None, :] > rows[:, None]] != 0.0):
            raise DimensionMismatch("nonzero weight above the causal boundary")

    @property
    def n_new(self) -> int:
        return self.weights.shape[0]

    @property
    def n_total(self) -> int:
        return self.weights.shape[1]

    @property
    def total_weight(self) -> float:
        return float(self.weights.sum())

    def row_positions(self) -> np.ndarray:
        return self.row_offset + np.arange(self.n_new)


def _check_qkv(Q, K, V, row_offset):
    if Q.dim() != 2 or K.dim() != 2 or V.dim() != 2:
        raise DimensionMismatch("Q, K, V must be 2-D")
    if Q.shape[1] != K.shape[1]:
        raise DimensionMismatch(f"Q cols {Q.shape[1]} != K cols {K.shape[1]}")
    if V.shape[0] != K.shape[0]:
        raise DimensionMismatch(f"V rows {V.shape[0]} != K rows {K.shape[0]}")
    if row_offset != K.shape[0] - Q.shape[0] or row_offset < 0:
        raise DimensionMismatch(f"row_offset={row_offset} must equal K rows - Q rows >= 0")
    if V.shape[1] != K.shape[1]:
        raise DimensionMismatch("the B200 kernels require d_v == d_k")


def plan_tensors(plan, n_total: int, device):
    """SparsePlan (or any object with selected_slashes / selected_verticals,
    tensor_ops.py:158-159) -> device (slash_ids, vert_ids, counts) for 1 head."""
    s = sorted(int(x) for x in plan.selected_slashes if 0 <= int(x) < n_total)
    v = sorted(int(x) for x in plan.selected_verticals if 0 <= int(x) < n_total)
    sl = torch.zeros((1, n_total), dtype=torch.int32)
    vt = torch.zeros((1, n_total), dtype=torch.int32)
    sl[0, :len(s)] = torch.tensor(s, dtype=torch.int32)
    vt[0, :len(v)] = torch.tensor(v, dtype=torch.int32)
    counts = torch.tensor([[len(s), len(v)]], dtype=torch.int32)
    return sl.to(device), vt.to(device), counts.to(device)


def attention_layer(q_block: torch.Tensor, k: torch.Tensor, v: torch.Tensor, slash_ids, vert_ids, counts,
                    n_new: int, n_total: int, n_kv_heads: int, out: torch.Tensor | None = None,
                    out_dtype=torch.bfloat16, q_head_stride=None, kv_head_stride=None,
                    ws: Workspace | None = None, stream=None, tiles: torch.Tensor | None = None,
                    cells: torch.Tensor | None = None):
    """K5 for every q-head of a layer -> (out [n_new, H, d], cells [H]); with
    `tiles` (int64 [H]) also the 128x128 tensor-core tiles each head executed.
    `out` may be a head-column view of a wider [n_new, H_all, d] output."""
    H = counts.shape[0]
    d = q_block.shape[-1]
    dev = q_block.device
    L = layer_desc(H, n_kv_heads, d, n_new, n_total,
                   q_block.stride(0) if q_head_stride is None else q_head_stride,
                   k.stride(0) if kv_head_stride is None else kv_head_stride,
                   out.stride(0) if out is not None else 0)
    if out is None:
        out = torch.empty((n_new, H, d), dtype=out_dtype, device=dev)
    if cells is None:
        cells = torch.empty(H, dtype=torch.int64, device=dev)
    ws = ws or Workspace()
    n = _lib.lib().ls_vs_attention_workspace(C_ref(L))
    w = ws.get(n)
    if tiles is None:
        _lib.call("ls_vs_attention", C_ref(L), q_block.data_ptr(), k.data_ptr(), v.data_ptr(), slash_ids.data_ptr(),
                  vert_ids.data_ptr(), counts.data_ptr(), out.data_ptr(), int(out.dtype == torch.bfloat16),
                  cells.data_ptr(), w.data_ptr(), w.numel(), _lib.stream_ptr(stream))
    else:
        _lib.call("ls_vs_attention_ex", C_ref(L), q_block.data_ptr(), k.data_ptr(), v.data_ptr(),
                  slash_ids.data_ptr(), vert_ids.data_ptr(), counts.data_ptr(), out.data_ptr(),
                  int(out.dtype == torch.bfloat16), cells.data_ptr(), tiles.data_ptr(), w.data_ptr(), w.numel(),
                  _lib.stream_ptr(stream))
    return out, cells


def plan_rows(q_block, k, slash_ids, vert_ids, counts, n_new, n_total, n_kv_heads, n_rows, out=None,
              out_row_stride=None, out_head_stride=None, q_head_stride=None, kv_head_stride=None, stream=None):
    """Dense probability rows of the block's last n_rows rows under the plan
    (session.py:89-95 observation seeds): fp32 [H, n_rows, n_total]."""
    H = counts.shape[0]
    d = q_block.shape[-1]
    L = layer_desc(H, n_kv_heads, d, n_new, n_total,
                   q_block.stride(0) if q_head_stride is None else q_head_stride,
                   k.stride(0) if kv_head_stride is None else kv_head_stride)
    if out is None:
        out = torch.empty((H, n_rows, n_total), dtype=torch.float32, device=q_block.device)
        out_row_stride, out_head_stride = n_total, n_rows * n_total
    _lib.call("ls_plan_rows", C_ref(L), int(n_rows), q_block.data_ptr(), k.data_ptr(), slash_ids.data_ptr(),
              vert_ids.data_ptr(), counts.data_ptr(), out.data_ptr(), int(out_row_stride), int(out_head_stride),
              _lib.stream_ptr(stream))
    return out


def plan_coverage_layer(q_block, k, v, slash_ids, vert_ids, counts, n_new, n_total, n_kv_heads,
                        q_head_stride=None, kv_head_stride=None, ws: Workspace | None = None,
                        stream=None) -> torch.Tensor:
    """coverage_ratio (prefill.py:254-281) of every head's plan over the block's
    full causal attention: fp64 [H] on the device."""
    H = counts.shape[0]
    d = q_block.shape[-1]
    L = layer_desc(H, n_kv_heads, d, n_new, n_total,
                   q_block.stride(0) if q_head_stride is None else q_head_stride,
                   k.stride(0) if kv_head_stride is None else kv_head_stride)
    cov = torch.empty(H, dtype=torch.float64, device=q_block.device)
    ws = ws or Workspace()
    w = ws.get(_lib.lib().ls_plan_coverage_workspace(C_ref(L)))
    _lib.call("ls_plan_coverage", C_ref(L), q_block.data_ptr(), k.data_ptr(), v.data_ptr(), slash_ids.data_ptr(),
              vert_ids.data_ptr(), counts.data_ptr(), cov.data_ptr(), w.data_ptr(), w.numel(),
              _lib.stream_ptr(stream))
    return cov


def coverage_ratio(Q, K, V, plan, row_offset: int) -> float:
    """prefill.coverage_ratio(block, plan) (prefill.py:254-257) for one head,
    with the block given as its Q/K/V instead of a dense AttentionBlock: the
    dense weights are never materialised."""
    Qt, Kt, Vt = to_bf16(Q), to_bf16(K), to_bf16(V)
    _check_qkv(Qt, Kt, Vt, row_offset)
    n_new, n_total = Qt.shape[0], Kt.shape[0]
    sl, vt, cn = plan_tensors(plan, n_total, Qt.device)
    cov = plan_coverage_layer(Qt.unsqueeze(0), Kt.unsqueeze(0), Vt.unsqueeze(0), sl, vt, cn, n_new, n_total, 1)
    return float(cov[0].item())


def recovery_curve(qkv_per_head: dict, row_offset: int, etas) -> list[tuple[float, float]]:
    """metrics.recovery_curve (metrics.py:71-96) with each head's block given
    as its (Q, K, V) instead of a dense AttentionBlock: for each eta, the
    head-averaged full-block coverage of the top floor(eta * 2 n_total) lines of
    both kinds ranked together by (weight desc, kind, index). Line sums over ALL
    block rows come from K1 (rows = every row), coverage from ls_plan_coverage;
    only the ranking of the 2 n_total lines runs on the host (diagnostic path)."""
    from .prefill import line_arrays_device  # noqa: PLC0415

    curves = {float(e): [] for e in etas}
    for Q, K, V in qkv_per_head.values():
        Qt, Kt, Vt = to_bf16(Q), to_bf16(K), to_bf16(V)
        _check_qkv(Qt, Kt, Vt, row_offset)
        n_new, n_total = Qt.shape[0], Kt.shape[0]
        v_w, s_w = line_arrays_device(Qt, Kt, row_offset)
        # every row sampled: all n_total lines of each kind exist (prefill.py:159-167)
        w = np.concatenate([s_w, v_w])
        kind = np.concatenate([np.zeros(n_total, np.int8), np.ones(n_total, np.int8)])  # "slash" < "vertical"
        idx = np.concatenate([np.arange(n_total), np.arange(n_total)])
        order = np.lexsort((idx, kind, -w))
        for eta in curves:
            k = int(np.floor(eta * 2 * n_total + 1e-9))
            chosen = order[:k]
            sl = idx[chosen[kind[chosen] == 0]]
            vt = idx[chosen[kind[chosen] == 1]]
            plan = SimpleNamespace(selected_slashes=frozenset(int(x) for x in sl),
                                   selected_verticals=frozenset(int(x) for x in vt))
            if not plan.selected_slashes and not plan.selected_verticals:
                curves[eta].append(0.0)
                continue
            sl_t, vt_t, cn = plan_tensors(plan, n_total, Qt.device)
            cov = plan_coverage_layer(Qt.unsqueeze(0), Kt.unsqueeze(0), Vt.unsqueeze(0), sl_t, vt_t, cn, n_new,
                                      n_total, 1)
            curves[eta].append(float(cov[0].item()))
    return [(eta, float(np.mean(r))) for eta, r in curves.items()]


def masked_sparse_attention(Q, K, V, plan, row_offset: int, counter: OpCounter | None = None,
                            return_weights: bool = False):
    """tensor_ops.py:141-183 on the device (one head). Returns numpy fp64 Z
    (and an AttentionBlock of the fp32 device weights when asked)."""
    Qt, Kt, Vt = to_bf16(Q), to_bf16(K), to_bf16(V)
    _check_qkv(Qt, Kt, Vt, row_offset)
    if not plan.selected_slashes and not plan.selected_verticals:
        raise EmptyPlan("plan selects no lines")
    n_new, n_total = Qt.shape[0], Kt.shape[0]
    sl, vt, cn = plan_tensors(plan, n_total, Qt.device)
    out, cells = attention_layer(Qt.unsqueeze(0), Kt.unsqueeze(0), Vt.unsqueeze(0), sl, vt, cn, n_new, n_total, 1,
                                 out_dtype=torch.float32)
    Z = out[:, 0, :].double().cpu().numpy()
    if counter is not None:
        counter.add(int(cells[0].item()))
    if return_weights:
        W = plan_rows(Qt.unsqueeze(0), Kt.unsqueeze(0), sl, vt, cn, n_new, n_total, 1, n_new)
        return Z, AttentionBlock(weights=W[0].double().cpu().numpy(), row_offset=row_offset)
    return Z


def scaled_dot_attention(Q, K, V, row_offset: int, counter: OpCounter | None = None):
    """tensor_ops.py:104-127: dense causal attention on the device -> (Z, AttentionBlock)."""
    Qt, Kt, Vt = to_bf16(Q), to_bf16(K), to_bf16(V)
    _check_qkv(Qt, Kt, Vt, row_offset)
    n_new, n_total = Qt.shape[0], Kt.shape[0]
    L = layer_desc(1, 1, Qt.shape[1], n_new, n_total, 0, 0)
    out = torch.empty((n_new, 1, Qt.shape[1]), dtype=torch.float32, device=Qt.device)
    _lib.call("ls_dense_attention", C_ref(L), Qt.data_ptr(), Kt.data_ptr(), Vt.data_ptr(), out.data_ptr(), 0,
              _lib.stream_ptr())
    if counter is not None:
        counter.add(n_new * n_total)
    # dense weights through the plan-rows kernel with the all-lines plan
    allp = type("AllLines", (), {"selected_slashes": range(n_total), "selected_verticals": ()})()
    sl, vt, cn = plan_tensors(allp, n_total, Qt.device)
    W = plan_rows(Qt.unsqueeze(0), Kt.unsqueeze(0), sl, vt, cn, n_new, n_total, 1, n_new)
    return out[:, 0, :].double().cpu().numpy(), AttentionBlock(weights=W[0].double().cpu().numpy(),
                                                               row_offset=row_offset)


def dense_attention_layer(q_block, k, v, n_new, n_total, n_kv_heads, out=None, out_dtype=torch.bfloat16,
                          q_head_stride=None, kv_head_stride=None, stream=None):
    """Dense causal attention for every q-head of a layer (the lossless
    baseline, §8f.1): out [n_new, H, d]."""
    H = q_block.shape[0]
    d = q_block.shape[-1]
    L = layer_desc(H, n_kv_heads, d, n_new, n_total,
                   q_block.stride(0) if q_head_stride is None else q_head_stride,
                   k.stride(0) if kv_head_stride is None else kv_head_stride)
    if out is None:
        out = torch.empty((n_new, H, d), dtype=out_dtype, device=q_block.device)
    _lib.call("ls_dense_attention", C_ref(L), q_block.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
              int(out.dtype == torch.bfloat16), _lib.stream_ptr(stream))
    return out


__all__ = ["AttentionBlock", "masked_sparse_attention", "scaled_dot_attention", "attention_layer",
           "dense_attention_layer", "plan_rows", "plan_tensors", "plan_coverage_layer", "coverage_ratio", "recovery_curve", "math"]
