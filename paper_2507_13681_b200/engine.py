"""Device-resident multi-layer LoopServe turn engine (attention-only shapes).

Restates the LoopServe branch of `run_turn` (reference session.py:113-201)
for models whose attention layers are given as Q/K/V tensors in HBM (the
synthetic Llama/Qwen shapes of BASELINE.json; projections/MLP are out of
scope):

  prefill (per layer, all q-heads, no host sync):
    K0 sample rows        session.py:135-144 / prefill.py:125-135 (all layers, one launch)
    K1 score + line sums  prefill.py:377-390, 138-169
    K2-K4 sort + greedy   prefill.py:168-169, 178-229
    K5 sparse attention   model.py:242-251 -> tensor_ops.py:141-183
    seeds                 session.py:163 / 89-95 (only rows that survive to the first event)
  decode (per token, per layer):
    event: K7 + K8        kvcompress.py:205-225
    K6 decode attention   kvcompress.py:227-237 / model.py:232-241
  rollback                session.py:180 (the archive only grows; positions past the
                          block are simply not read by the next turn's prefill)

Layouts in HBM (bf16): Q [L, n_q, cap, d], K/V [L, n_kv, cap, d]; a q-head
h reads kv-head h // (n_q / n_kv). Outputs are token-major [n_new, n_q, d].
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

from .kvcompress import CompressionConfig, DecodeLayer
from .prefill import LayerPlans, Workspace, sample_rows_device, sample_size, sparsify_layer
from .tensor_ops import attention_layer, dense_attention_layer, plan_rows

MODES = ("dense", "loopserve")


@dataclass(frozen=True)
class SessionParams:
    """session.py:42-57 (same field names and defaults)."""

    mode: str = "loopserve"
    alpha: float = 0.955
    comp: CompressionConfig = field(default_factory=CompressionConfig)
    sample_rate: float = 0.1
    sample_floor: int = 32
    max_new: int = 24
    eos_id: int | None = None
    seed: int = 0
    collect_timings: bool = False

    def validate(self) -> None:
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        self.comp.validate()


@dataclass(frozen=True)
class AttnShape:
    n_layers: int
    n_q: int
    n_kv: int
    d: int


class QKVStore:
    """Q/K/V of every position of a dialogue, per layer, resident in HBM."""

    def __init__(self, shape: AttnShape, cap: int, device="cuda", q=None, k=None, v=None):
        self.shape, self.cap = shape, cap
        L, d = shape.n_layers, shape.d
        self.q = q if q is not None else torch.empty((L, shape.n_q, cap, d), dtype=torch.bfloat16, device=device)
        self.k = k if k is not None else torch.empty((L, shape.n_kv, cap, d), dtype=torch.bfloat16, device=device)
        self.v = v if v is not None else torch.empty((L, shape.n_kv, cap, d), dtype=torch.bfloat16, device=device)

    @staticmethod
    def synthetic(shape: AttnShape, cap: int, n_ref: int | None = None, seed: int = 0, device="cuda"):
        from .synth import SynthSpec, layer_qkv_torch

        st = QKVStore(shape, cap, device)
        spec = SynthSpec(shape.n_q, shape.n_kv, shape.d, cap, n_ref=n_ref, seed=seed)
        for l in range(shape.n_layers):
            q, k, v = layer_qkv_torch(spec, l, device=device)
            st.q[l].copy_(q)
            st.k[l].copy_(k)
            st.v[l].copy_(v)
        return st


@dataclass
class PrefillOut:
    out: list          # per layer [n_new, n_q, d] bf16
    plans: list        # per layer LayerPlans (None in dense mode)
    cells: list        # per layer int64 [n_q] (K5 OpCounter increments)
    rows: torch.Tensor | None
    n_new: int
    n_total: int


class SessionEngine:
    def __init__(self, shape: AttnShape, params: SessionParams, cap: int, device="cuda",
                 out_dtype=torch.bfloat16):
        params.validate()
        self.shape, self.params, self.cap = shape, params, cap
        self.device = device
        self.out_dtype = out_dtype
        comp = params.comp
        self.window = comp.window()
        budget_cap = comp.budget if comp.budget is not None else 1
        self.decode_layers = [DecodeLayer(shape.n_q, shape.n_kv, shape.d, self.window, budget_cap, cap + 1,
                                          cap * shape.d, device=device) for _ in range(shape.n_layers)]
        self.ws = Workspace()
        self.rows_ws = Workspace()
        self.clear_logs()

    def clear_logs(self):
        """Work logs (device tensors / host counts) used by bench.py's roofline."""
        self.cell_log, self.score_log, self.decode_cols = [], [], 0
        self.decode_launches = 0

    # ------------------------------------------------------------- prefill
    def prefill(self, store: QKVStore, turn: int, row_offset: int, n_new: int, seed_rows: bool = True,
                stream=None, turn_offset_heads: int = 0) -> PrefillOut:
        """Sparse prefill of one turn block for every layer. `turn_offset_heads`
        is the global index of local q-head 0 (head-sharded runs): sampling
        seeds use global head ids (session.py:84-86)."""
        p, sh = self.params, self.shape
        n_total = row_offset + n_new
        outs, plans_all, cells_all = [], [], []
        rows = None
        if p.mode == "loopserve":
            if p.alpha >= 1.0:  # session.py:136-137: every row
                rows = torch.arange(n_new, dtype=torch.int32, device=self.device).expand(
                    sh.n_layers, sh.n_q, n_new).contiguous()
            else:
                rows = sample_rows_device(n_new, p.sample_rate, p.sample_floor, p.seed, turn, 0,
                                          turn_offset_heads, sh.n_q, n_layers=sh.n_layers, stream=stream,
                                          ws=self.rows_ws)
                if rows.dim() == 2:
                    rows = rows.unsqueeze(0)
        n_seed = min(self.window, n_new)
        surv = p.comp.surviving_seeds(n_seed, p.max_new) if seed_rows else 0
        for l in range(sh.n_layers):
            qb = store.q[l, :, row_offset:n_total]
            kl, vl = store.k[l], store.v[l]
            if p.mode == "dense":
                outs.append(dense_attention_layer(qb, kl, vl, n_new, n_total, sh.n_kv, out_dtype=self.out_dtype,
                                                  q_head_stride=store.q.stride(1), stream=stream))
                plans_all.append(None)
                cells_all.append(None)
                continue
            plans: LayerPlans = sparsify_layer(qb, kl, rows[l], p.alpha, n_new, n_total, sh.n_kv,
                                               q_head_stride=store.q.stride(1), ws=self.ws, stream=stream)
            out, cells = attention_layer(qb, kl, vl, plans.slash_ids, plans.vert_ids, plans.counts, n_new,
                                         n_total, sh.n_kv, out_dtype=self.out_dtype,
                                         q_head_stride=store.q.stride(1), ws=self.ws, stream=stream)
            outs.append(out)
            plans_all.append(plans)
            cells_all.append(cells)
            self.cell_log.append(cells)
            self.score_log.append(plans.score_count)
            dl = self.decode_layers[l]
            dl.reset()
            slots = dl.seed_slots(n_seed)
            if surv > 0:
                # the surviving seeds are the last `surv` rows of the block
                first = slots[n_seed - surv]
                assert slots[n_seed - surv:] == list(range(first, first + surv))
                plan_rows(qb, kl, plans.slash_ids, plans.vert_ids, plans.counts, n_new, n_total, sh.n_kv, surv,
                          out=dl.ring_w[:, first:], out_row_stride=dl.row_cap,
                          out_head_stride=dl.window * dl.row_cap, q_head_stride=store.q.stride(1),
                          stream=stream)
                dl.ring_n[:, first:first + surv] = n_total
                dl.ring_dense[:, first:first + surv] = 1
        return PrefillOut(outs, plans_all, cells_all, rows, n_new, n_total)

    # -------------------------------------------------------------- decode
    def decode(self, store: QKVStore, L0: int, max_new: int, record=False, stream=None):
        """max_new decode steps (kvcompress.py:200-239) from cache length L0.
        Returns per step a list of per-layer outputs [n_q, d]."""
        p, sh = self.params, self.shape
        comp = p.comp if p.mode == "loopserve" else CompressionConfig(budget=None)
        if p.mode == "dense":
            for dl in self.decode_layers:
                dl.reset()
        length = L0
        compressed = False
        outs = []
        events = []
        for n_o in range(1, max_new + 1):
            if comp.event_at(n_o):
                for l, dl in enumerate(self.decode_layers):
                    dl.event(length, comp.budget, stream=stream)
                    dl.compact(store.k[l], store.v[l], stream=stream)
                    if record:
                        events.append((n_o, l, dl.working_ids(length, True), dl.score_cov.cpu().numpy()))
                compressed = True
            q_step = store.q[:, :, length].contiguous()  # [L, n_q, d]
            step = []
            for l, dl in enumerate(self.decode_layers):
                step.append(dl.step(q_step[l], store.k[l], store.v[l], length, compressed, stream=stream))
            # algorithmic columns per q-head (upper bound |keep| <= B + W after an event)
            cols = min(length, comp.budget + self.window) + 1 if compressed else length + 1
            self.decode_cols += cols * sh.n_q * sh.n_layers
            self.decode_launches += sh.n_layers
            outs.append(step)
            length += 1
        return outs, events

    def turn_blocks(self, input_len: int, n_turns: int, max_new: int):
        """(row_offset, n_new) of each turn: block = previous answer + input
        (session.py:122), decode rows rolled back (session.py:180)."""
        out, hist = [], 0
        for t in range(n_turns):
            n_new = input_len + (max_new if t > 0 else 0)
            out.append((hist - (max_new if t > 0 else 0), n_new))
            hist += input_len + max_new
        return out


def dialogue_cap(input_len: int, n_turns: int, max_new: int) -> int:
    return n_turns * (input_len + max_new)


__all__ = ["SessionParams", "AttnShape", "QKVStore", "SessionEngine", "PrefillOut", "dialogue_cap",
           "sample_size", "math"]
