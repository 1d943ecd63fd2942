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
  decode (per token): CUDA graphs over all layers with the step counters in
  device memory (kvcompress.py:200-239):
    event graph           K7 + K8 for every layer   (kvcompress.py:205-225)
    step graph            q gather + K6 per layer + counter advance
                          (dense-step and compressed-step variants)
  rollback                session.py:180 (the archive only grows; positions past the
                          block are simply not read by the next turn's prefill)

Layouts in HBM (bf16): Q [L, n_q, cap, d], K/V [L, n_kv, cap, d]; a q-head
h reads kv-head h // (n_q / n_kv). Outputs are token-major [n_new, n_q, d].
"""

from __future__ import annotations

import math
from contextlib import nullcontext as _nullcontext
from dataclasses import dataclass, field

import torch

from . import _lib
from .errors import CacheCorrupt, DimensionMismatch, EmptyPlan, SequenceTooLong
from .kvcompress import CompressionConfig, DecodeStack
from .prefill import LayerPlans, Workspace, sample_rows_device, sample_size, sparsify_layer
from .tensor_ops import attention_layer, dense_attention_layer, plan_rows

MODES = ("dense", "loopserve", "obswindow")  # session.py:40
GRAPH_BUCKET = 1024  # column-bound bucket of the captured decode graphs


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
    """Q/K/V of every position of a dialogue, per layer, resident in HBM: the
    append-only archive of the reference's KVCache (model.py:139-175; Q kept
    too, since the attention-only path takes the projections as inputs).
    `length` marks the filled prefix. A store built with `length=None` (the
    default, e.g. QKVStore.synthetic) is preloaded: every position is present;
    QKVStore.empty() starts at length 0 and grows with append()."""

    def __init__(self, shape: AttnShape, cap: int, device="cuda", q=None, k=None, v=None, length: int | None = None):
        self.shape, self.cap = shape, cap
        L, d = shape.n_layers, shape.d
        self.q = q if q is not None else torch.empty((L, shape.n_q, cap, d), dtype=torch.bfloat16, device=device)
        self.k = k if k is not None else torch.empty((L, shape.n_kv, cap, d), dtype=torch.bfloat16, device=device)
        self.v = v if v is not None else torch.empty((L, shape.n_kv, cap, d), dtype=torch.bfloat16, device=device)
        self.length = cap if length is None else int(length)
        self.validate()

    @staticmethod
    def empty(shape: AttnShape, cap: int, device="cuda") -> "QKVStore":
        return QKVStore(shape, cap, device=device, length=0)

    def validate(self) -> None:
        """KVCache.validate (model.py:157-168): length in range, layer/head shapes."""
        sh = self.shape
        if not (0 <= self.length <= self.cap):
            raise CacheCorrupt(f"store length {self.length} outside [0, {self.cap}]")
        want = {"q": (sh.n_layers, sh.n_q, self.cap, sh.d), "k": (sh.n_layers, sh.n_kv, self.cap, sh.d),
                "v": (sh.n_layers, sh.n_kv, self.cap, sh.d)}
        for name, shp in want.items():
            if tuple(getattr(self, name).shape) != shp:
                raise CacheCorrupt(f"{name} archive has a foreign shape {tuple(getattr(self, name).shape)} != {shp}")

    def append(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> int:
        """Write n new positions at [length, length + n) (forward_extend's cache
        write, model.py:228-231): q [L, n_q, n, d], k / v [L, n_kv, n, d].
        Returns the new length; SequenceTooLong past the capacity."""
        n = int(k.shape[2])
        if q.shape[2] != n or v.shape[2] != n:
            raise DimensionMismatch("q, k, v must add the same number of positions")
        if self.length + n > self.cap:
            raise SequenceTooLong(f"{self.length + n} positions exceed the store capacity {self.cap}")
        lo, hi = self.length, self.length + n
        self.q[:, :, lo:hi].copy_(q, non_blocking=True)
        self.k[:, :, lo:hi].copy_(k, non_blocking=True)
        self.v[:, :, lo:hi].copy_(v, non_blocking=True)
        self.length = hi
        return hi

    def truncate(self, length: int) -> None:
        """KVCache.truncate (model.py:171-174): roll back to `length`, e.g. the
        decode rows at the end of a turn (session.py:180)."""
        if not (0 <= length <= self.length):
            raise CacheCorrupt(f"cannot truncate length {self.length} to {length}")
        self.length = int(length)

    @staticmethod
    def synthetic(shape: AttnShape, cap: int, n_ref: int | None = None, seed: int = 0, device="cuda",
                  kv_offset: int = 0):
        from .synth import SynthSpec, layer_qkv_torch

        st = QKVStore(shape, cap, device)
        spec = SynthSpec(shape.n_q, shape.n_kv, shape.d, cap, n_ref=n_ref, seed=seed, kv_offset=kv_offset)
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
    n_seed: int = 0


class SessionEngine:
    """head_groups: the q-heads of a layer are processed as this many groups
    of whole kv-head groups, each on its own stream, with the line scoring
    (K1) of group g + 1 started only when group g's is done, so that group g's
    selection (K2-K4: a latency-bound chain on one SM per head) and sparse
    attention overlap the next groups' scoring. Layers stay sequential: all
    groups of layer l finish before layer l + 1 starts."""

    def __init__(self, shape: AttnShape, params: SessionParams, cap: int, device="cuda",
                 out_dtype=torch.bfloat16, head_groups: int | None = None, keep_plans: bool = True,
                 session_seeds=None):
        """session_seeds: run len(session_seeds) independent dialogue sessions
        of identical turn geometry as ONE batch (config C4, session.py:71-86 /
        cli.py:213-226): `shape` then counts the heads of all sessions, session
        s owning q-heads [s*H_s, (s+1)*H_s) and kv-heads [s*KV_s, (s+1)*KV_s);
        each session samples its rows with its own seed and head ids 0..H_s-1
        (Session.head_seed), and every kernel launch covers all sessions'
        heads (the decode moves n_sessions x the bytes per launch)."""
        params.validate()
        self.session_seeds = list(session_seeds) if session_seeds is not None else None
        if self.session_seeds is not None:
            S = len(self.session_seeds)
            if S < 1 or shape.n_q % S or shape.n_kv % S:
                raise ValueError(f"{S} sessions do not divide {shape.n_q} q-heads / {shape.n_kv} kv-heads")
        # the session's plan ledger (turn, layer) -> LayerPlans (session.py:153-154)
        self.plan_ledger = {} if keep_plans else None
        self.shape, self.params, self.cap = shape, params, cap
        self.device = device
        self.out_dtype = out_dtype
        comp = params.comp
        self.window = comp.window()
        budget_cap = comp.budget if comp.budget is not None else 1
        self.stack = DecodeStack(shape.n_layers, shape.n_q, shape.n_kv, shape.d, self.window, budget_cap, cap + 1,
                                 shape.n_kv * cap * shape.d, cap * shape.d, device=device)
        self.ws = Workspace()
        self.rows_ws = Workspace()
        self.stack.event_workspace(self.stack.row_cap)  # fixed before any graph captures it
        # observation rows of compressed steps carry (n_a, lo) instead of their ids when
        # each row is consumed by one event only (interval >= window, kvcompress.py:196)
        import os as _os
        self.stack.derived_ids = (comp.budget is not None and comp.interval >= self.window
                                  and _os.environ.get("LS_DERIVED_IDS", "1") != "0")
        self._q_buf = torch.empty((shape.n_layers, shape.n_q, 1, shape.d), dtype=torch.bfloat16, device=device)
        self._out_buf = torch.empty((shape.n_layers, shape.n_q, shape.d), dtype=out_dtype, device=device)
        self._graphs = {}
        self._ring = None
        self._obs = None  # obswindow baseline: (compact store, full-cache decode engine)
        self._obs_nb = None
        if head_groups is None:
            import os
            head_groups = int(os.environ.get("LS_HEAD_GROUPS", "1"))
        grp = shape.n_q // shape.n_kv
        if head_groups < 1 or (shape.n_kv % head_groups and (head_groups % shape.n_kv or grp % (head_groups // shape.n_kv))):
            raise ValueError(f"head_groups={head_groups} must divide n_kv={shape.n_kv}, or split each KV head's "
                             f"{grp} q-heads evenly")
        self.head_groups = head_groups
        if shape.n_kv % head_groups == 0:  # whole KV-head groups
            kv_per = shape.n_kv // head_groups
            self._groups = [(g * kv_per * grp, (g + 1) * kv_per * grp, g * kv_per, (g + 1) * kv_per)
                            for g in range(head_groups)]
        else:  # q-heads of one KV head split across groups (e.g. one C5 shard: 8 q-heads, 1 KV head)
            q_per = shape.n_q // head_groups
            self._groups = [(g * q_per, (g + 1) * q_per, (g * q_per) // grp, (g * q_per) // grp + 1)
                            for g in range(head_groups)]
        if head_groups > 1 and str(device).startswith("cuda") and torch.cuda.is_available():
            # K1 / K5 on normal-priority streams; the selection chains (few CTAs,
            # latency-bound) on high-priority streams so their CTAs are
            # dispatched ahead of the other groups' pending K1 / K5 CTAs
            self._streams = [torch.cuda.Stream(device=device) for _ in range(head_groups)]
            self._streams_hi = [torch.cuda.Stream(device=device, priority=-1) for _ in range(head_groups)]
            self._gws = [Workspace() for _ in range(head_groups)]
            self._ev_scored = [torch.cuda.Event() for _ in range(head_groups)]
            self._ev_done = [torch.cuda.Event() for _ in range(head_groups)]
            self._ev_start = torch.cuda.Event()
        # K5 overlapped with K3 (head_groups == 1): each head's K3 CTA publishes its plan
        # with a device flag (ls_select_lines_ready); the sparse attention of a group of
        # heads runs on its own stream as soon as the group's flags are set, while slower
        # heads are still selecting. Groups are whole KV-head groups (or q-heads of one
        # KV head), about LS_K5_GROUPS (8) of them. LS_K5_OVERLAP=0 turns it off.
        import os as _os
        self._overlap = (head_groups == 1 and str(device).startswith("cuda") and torch.cuda.is_available()
                         and _os.environ.get("LS_K5_OVERLAP", "1") != "0")
        if self._overlap:
            gh = max(1, shape.n_q // int(_os.environ.get("LS_K5_GROUPS", "8")))  # ~8 groups
            if gh >= grp:
                gh -= gh % grp  # whole KV-head groups
                while shape.n_q % gh:
                    gh -= grp
            else:
                while grp % gh:  # q-heads of one KV head
                    gh -= 1
            self._k5_groups = [(h0, h0 + gh) for h0 in range(0, shape.n_q, gh)]
            self._k5_streams = [torch.cuda.Stream(device=device) for _ in self._k5_groups]
            self._k5_ws = [Workspace() for _ in self._k5_groups]
            self._k5_done = [torch.cuda.Event() for _ in self._k5_groups]
            self._k5_start = torch.cuda.Event()
            self._ready = torch.zeros(shape.n_q, dtype=torch.int32, device=device)
            self._epoch = 0
            # below this context the layer's GPU work is too short to pay for the groups'
            # extra launches (measured: C2 turn 1 at 5K keys 16 -> 36 ms, turn 2 at 10K
            # neutral, turn 3 at 15K 49.5 -> 47.0 ms; C3 turn 2 at 16.6K 71.2 -> 66.6 ms;
            # C5 turn 10 at 101K keys 19 % faster)
            # (public: contexts of at least this many keys use the head-group overlap)
            self.overlap_min = int(_os.environ.get("LS_K5_OVERLAP_MIN", "12000"))
        self.clear_logs()

    def clear_logs(self):
        """Work logs (device tensors / host counts) used by bench.py's roofline."""
        self.cell_log, self.score_log, self.decode_log, self.tile_log = [], [], [], []

    # ------------------------------------------------------------- prefill
    def prefill(self, store: QKVStore, turn: int, row_offset: int, n_new: int, seed_rows: bool = True,
                stream=None, turn_offset_heads: int = 0, layer_ready=None, layer_done=None) -> PrefillOut:
        """Sparse prefill of one turn block for every layer. `turn_offset_heads`
        is the global index of local q-head 0 (head-sharded runs): sampling
        seeds use global head ids (session.py:84-86).
        layer_ready(l, stream): called before layer l's work is enqueued (a
        caller streaming the block's Q/K/V in from the host makes `stream`
        wait for layer l's rows there); layer_done(l, out, stream): called once
        layer l's output is enqueued (e.g. to start its copy-out while the
        next layer computes)."""
        p, sh = self.params, self.shape
        n_total = row_offset + n_new
        if n_total > store.length:
            raise CacheCorrupt(f"prefill of positions [{row_offset}, {n_total}) but the store holds {store.length}")
        outs, plans_all, cells_all = [], [], []
        rows = None
        if p.mode == "loopserve" and p.alpha <= 0.0:
            # alpha = 0 selects no line for any head (prefill.py:188-195), and
            # masked_sparse_attention rejects the empty plan (tensor_ops.py:165-166)
            raise EmptyPlan("alpha = 0 selects no line: the sparse prefill has an empty plan")
        if p.mode == "loopserve":
            if p.alpha >= 1.0:  # session.py:136-137: every row
                rows = torch.arange(n_new, dtype=torch.int32, device=self.device).expand(
                    sh.n_layers, sh.n_q, n_new).contiguous()
            elif self.session_seeds is not None:  # per-session seeds, per-session head ids
                hs = sh.n_q // len(self.session_seeds)
                parts = []
                for sd in self.session_seeds:
                    r_ = sample_rows_device(n_new, p.sample_rate, p.sample_floor, sd, turn, 0, 0, hs,
                                            n_layers=sh.n_layers, stream=stream, ws=self.rows_ws)
                    parts.append(r_.unsqueeze(0) if r_.dim() == 2 else r_.clone())
                rows = torch.cat(parts, dim=1)
            else:
                rows = sample_rows_device(n_new, p.sample_rate, p.sample_floor, p.seed, turn, 0,
                                          turn_offset_heads, sh.n_q, n_layers=sh.n_layers, stream=stream,
                                          ws=self.rows_ws)
                if rows.dim() == 2:
                    rows = rows.unsqueeze(0)
        n_seed = min(self.window, n_new)
        surv = p.comp.surviving_seeds(n_seed, p.max_new) if (seed_rows and p.mode == "loopserve") else 0
        st = self.stack
        main = stream if stream is not None else torch.cuda.current_stream()
        for l in range(sh.n_layers):
            if layer_ready is not None:
                layer_ready(l, main)
            qb = store.q[l, :, row_offset:n_total]
            kl, vl = store.k[l], store.v[l]
            if p.mode in ("dense", "obswindow"):
                outs.append(dense_attention_layer(qb, kl, vl, n_new, n_total, sh.n_kv, out_dtype=self.out_dtype,
                                                  q_head_stride=store.q.stride(1), stream=stream))
                plans_all.append(None)
                cells_all.append(None)
                if p.mode == "obswindow" and p.comp.budget is not None:
                    # the baseline's observation rows: the last W rows of every head's
                    # dense block (session.py:163, 89-95), into ring slots [0, n_seed)
                    sl, vt, cn = self._all_lines(n_total)
                    hr = slice(l * sh.n_q, (l + 1) * sh.n_q)
                    plan_rows(qb, kl, sl, vt, cn, n_new, n_total, sh.n_kv, n_seed, out=self.stack.ring_s[hr, 0:],
                              out_row_stride=self.stack.row_cap,
                              out_head_stride=self.stack.window * self.stack.row_cap,
                              q_head_stride=store.q.stride(1), stream=stream)
                if layer_done is not None:
                    layer_done(l, outs[-1], main)
                continue
            if self.head_groups > 1:
                plans, out, cells, tiles = self._layer_groups(l, qb, kl, vl, rows[l], n_new, n_total, surv, n_seed,
                                                              store.q.stride(1), stream)
            elif self._overlap and n_total >= self.overlap_min and (layer_ready is None or n_total >= 2 * self.overlap_min):
                # (with per-layer host inputs streaming in, layer_ready, the head groups'
                # streams contend with the copies: kept for the longest contexts only --
                # measured C2 turn 3 end to end 54 -> 63 ms with them)
                plans, out, cells, tiles = self._layer_overlap(l, qb, kl, vl, rows[l], n_new, n_total, surv, n_seed,
                                                               store.q.stride(1), stream)
            else:
                plans, out, cells, tiles = self._layer_group(l, 0, sh.n_q, 0, sh.n_kv, qb, kl, vl, rows[l], n_new,
                                                             n_total, surv, n_seed, store.q.stride(1), None,
                                                             self.ws, stream)
            self.tile_log.append(tiles)
            outs.append(out)
            if layer_done is not None:
                layer_done(l, out, main)
            plans_all.append(plans)
            cells_all.append(cells)
            if self.plan_ledger is not None:
                self.plan_ledger[(turn, l)] = plans  # session.py:153-154 (device plans, head order)
            self.cell_log.append(cells)
            self.score_log.append(plans.score_count)
        if surv > 0 and p.mode != "dense":
            # seed slots [n_seed - surv, n_seed) of every (layer, head): stored
            # probabilities (sum 0 marks them), dense rows of n_total columns
            first = n_seed - surv
            with torch.cuda.stream(stream) if stream is not None else _nullcontext():
                st.ring_ml[:, first:n_seed] = 0.0
                st.ring_n[:, first:n_seed] = n_total
                st.ring_dense[:, first:n_seed] = 1
        st.set_step(n_total, n_seed)
        return PrefillOut(outs, plans_all, cells_all, rows, n_new, n_total, n_seed)

    def _all_lines(self, n_total: int):
        """Every slash of every head: the plan whose cells are the whole causal block."""
        key = ("all_lines", n_total)
        if key not in self._graphs:
            H = self.shape.n_q
            sl = torch.arange(n_total, dtype=torch.int32, device=self.device).expand(H, n_total).contiguous()
            cn = torch.tensor([[n_total, 0]] * H, dtype=torch.int32, device=self.device)
            self._graphs[key] = (sl, torch.zeros_like(sl), cn)
        return self._graphs[key]

    def _decode_obswindow(self, store: QKVStore, L0: int, max_new: int, events, out_sink, run_sink):
        """The observation-window baseline's decode (session.py:204-257): one
        shared top-B over the prefill observation rows summed over every layer
        and head (K7-style fp64 accumulation + radix select, all on the
        device), base = retained_union(picked, W, L0) for every head, then
        append-only decoding against base + the new positions: the base rows
        are gathered once into a compact per-(layer, kv-head) store after which
        the new tokens' rows follow, and the full-cache decode (K6 dense steps)
        runs over it -- the same cells as the reference's working set."""
        import ctypes

        p, sh, st = self.params, self.shape, self.stack
        W, B = self.window, p.comp.budget
        dev = self.device
        n_rows = min(st.appended, W)
        scores = torch.empty(L0, dtype=torch.float64, device=dev)
        _lib.call("ls_obs_window_scores", sh.n_layers * sh.n_q, n_rows, st.ring_s.data_ptr(), W * st.row_cap,
                  st.row_cap, L0, scores.data_ptr(), _lib.stream_ptr())
        b = min(B, L0)
        ids = torch.arange(L0, dtype=torch.int32, device=dev)
        picked = torch.empty(b, dtype=torch.int32, device=dev)
        n_out = torch.empty(2, dtype=torch.int32, device=dev)
        ws = torch.empty(int(_lib.lib().ls_top_by_score_workspace(L0)) + (L0 + 31) // 32 * 4 + 256,
                         dtype=torch.uint8, device=dev)
        _lib.call("ls_top_by_score", L0, ids.data_ptr(), scores.data_ptr(), b, 0, L0, picked.data_ptr(),
                  n_out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr())
        base = torch.empty(b + W + 1, dtype=torch.int32, device=dev)
        _lib.call("ls_retained_union", b, picked.data_ptr(), W, L0, L0, base.data_ptr(), n_out[1:].data_ptr(),
                  ws.data_ptr(), ws.numel(), _lib.stream_ptr())
        nb = int(n_out[1].item())  # the compact store's length (one sync per turn)
        base = base[:nb]
        if events is not None:
            events.append({"step": 0, "length": L0, "base": base})
        cap_c = (B + W + 1) + max_new + 1
        if self._obs is None or self._obs[0].cap < cap_c:
            comp = CompressionConfig(budget=None, interval=p.comp.interval, warmup=p.comp.warmup,
                                     obs_window=p.comp.obs_window)
            inner = SessionEngine(sh, SessionParams(mode="dense", comp=comp, max_new=max_new), cap_c, device=dev,
                                  out_dtype=self.out_dtype)
            self._obs = (QKVStore(sh, cap_c, device=dev), inner)
        sc, inner = self._obs
        rows = torch.cat([base, torch.arange(L0, L0 + max_new, dtype=torch.int32, device=dev)])
        d2 = sh.d * 2
        for src, dst in ((store.k, sc.k), (store.v, sc.v)):
            _lib.call("ls_gather_rows", sh.n_layers * sh.n_kv, rows.numel(), rows.data_ptr(), src.data_ptr(),
                      store.cap * d2, dst.data_ptr(), sc.cap * d2, d2, _lib.stream_ptr())
        qrows = rows[nb:]
        _lib.call("ls_gather_rows", sh.n_layers * sh.n_q, max_new, qrows.data_ptr(), store.q.data_ptr(),
                  store.cap * d2, sc.q.data_ptr() + nb * d2, sc.cap * d2, d2, _lib.stream_ptr())
        inner.stack.set_step(nb, 0)
        self._last_decode = (L0, max_new, events)
        self._obs_nb = nb
        del ctypes
        return inner.decode(sc, nb, max_new, out_sink=out_sink, run_sink=run_sink)

    def _layer_group(self, l, h0, h1, kv0, kv1, qb, kl, vl, rows_l, n_new, n_total, surv, n_seed, qhs, out, ws,
                     stream, on_scored=None, select_stream=None):
        """K1-K5 (+ seed rows) of q-heads [h0, h1) of layer l, on `stream`."""
        p, sh, st = self.params, self.shape, self.stack
        n_kv = kv1 - kv0
        qg, kg, vg = qb[h0:h1], kl[kv0:kv1], vl[kv0:kv1]
        plans: LayerPlans = sparsify_layer(qg, kg, rows_l[h0:h1], p.alpha, n_new, n_total, n_kv, q_head_stride=qhs,
                                           ws=ws, stream=stream, on_scored=on_scored, select_stream=select_stream)
        tiles = torch.empty(h1 - h0, dtype=torch.int64, device=self.device)
        out, cells = attention_layer(qg, kg, vg, plans.slash_ids, plans.vert_ids, plans.counts, n_new, n_total, n_kv,
                                     out=out, out_dtype=self.out_dtype, q_head_stride=qhs, ws=ws, stream=stream,
                                     tiles=tiles)
        if surv > 0:
            # the seeds that are still in the deque at the first event are the
            # last `surv` block rows; they sit in slots [n_seed - surv, n_seed)
            first = n_seed - surv
            hr = slice(l * sh.n_q + h0, l * sh.n_q + h1)
            plan_rows(qg, kg, plans.slash_ids, plans.vert_ids, plans.counts, n_new, n_total, n_kv, surv,
                      out=st.ring_s[hr, first:], out_row_stride=st.row_cap, out_head_stride=st.window * st.row_cap,
                      q_head_stride=qhs, stream=stream)
            # (the seed slots' metadata is set once for every layer after the loop)
        return plans, out, cells, tiles

    def _layer_overlap(self, l, qb, kl, vl, rows_l, n_new, n_total, surv, n_seed, qhs, stream):
        """One layer with K5 overlapped with K3: K1 + K2/K3 on the caller's stream
        (each head's K3 CTA writes its plan and sets its ready flag), then per head
        group, on its own stream: a device wait on the group's flags, K5 and the
        seed rows; joined on the caller's stream."""
        p, sh, st = self.params, self.shape, self.stack
        main = stream if stream is not None else torch.cuda.current_stream()
        grp = sh.n_q // sh.n_kv
        self._epoch += 1
        self._k5_start.record(main)  # the layer's inputs are in place
        plans: LayerPlans = sparsify_layer(qb, kl, rows_l, p.alpha, n_new, n_total, sh.n_kv, q_head_stride=qhs,
                                           ws=self.ws, stream=stream, plan_ready=self._ready, epoch=self._epoch)
        out = torch.empty((n_new, sh.n_q, sh.d), dtype=self.out_dtype, device=self.device)
        cells = torch.empty(sh.n_q, dtype=torch.int64, device=self.device)
        tiles = torch.empty(sh.n_q, dtype=torch.int64, device=self.device)
        for g, (h0, h1) in enumerate(self._k5_groups):
            s = self._k5_streams[g]
            s.wait_event(self._k5_start)
            sp = _lib.stream_ptr(s)
            for h in range(h0, h1):
                _lib.call("ls_stream_wait_value", sp, self._ready[h:h + 1].data_ptr(), self._epoch)
            kv0, kv1 = h0 // grp, (h1 - 1) // grp + 1
            qg, kg, vg = qb[h0:h1], kl[kv0:kv1], vl[kv0:kv1]
            sl, vt, cn = plans.slash_ids[h0:h1], plans.vert_ids[h0:h1], plans.counts[h0:h1]
            with torch.cuda.stream(s):
                attention_layer(qg, kg, vg, sl, vt, cn, n_new, n_total, kv1 - kv0, out=out[:, h0:h1],
                                out_dtype=self.out_dtype, q_head_stride=qhs, ws=self._k5_ws[g], stream=s,
                                tiles=tiles[h0:h1], cells=cells[h0:h1])
                if surv > 0:
                    first = n_seed - surv
                    hr = slice(l * sh.n_q + h0, l * sh.n_q + h1)
                    plan_rows(qg, kg, sl, vt, cn, n_new, n_total, kv1 - kv0, surv, out=st.ring_s[hr, first:],
                              out_row_stride=st.row_cap, out_head_stride=st.window * st.row_cap, q_head_stride=qhs,
                              stream=s)
            self._k5_done[g].record(s)
        for g in range(len(self._k5_groups)):
            main.wait_event(self._k5_done[g])
        # (the tensors made on the caller's stream and read on the group streams stay
        # referenced by the returned plans / outputs until after this join)
        return plans, out, cells, tiles

    def _layer_groups(self, l, qb, kl, vl, rows_l, n_new, n_total, surv, n_seed, qhs, stream):
        """One layer as head groups on their own streams, K1 of group g + 1
        after K1 of group g; joined on the caller's stream."""
        main = stream if stream is not None else torch.cuda.current_stream()
        sh = self.shape
        out = torch.empty((n_new, sh.n_q, sh.d), dtype=self.out_dtype, device=self.device)
        self._ev_start.record(main)
        parts = []
        for g, (h0, h1, kv0, kv1) in enumerate(self._groups):
            s = self._streams[g]
            s.wait_event(self._ev_start)
            if g > 0:
                s.wait_event(self._ev_scored[g - 1])
            ev = self._ev_scored[g]
            with torch.cuda.stream(s):
                res = self._layer_group(l, h0, h1, kv0, kv1, qb, kl, vl, rows_l, n_new, n_total, surv, n_seed, qhs,
                                        out[:, h0:h1], self._gws[g], s, on_scored=lambda s=s, ev=ev: ev.record(s),
                                        select_stream=self._streams_hi[g])
            self._ev_done[g].record(s)
            parts.append(res)
        for g in range(len(self._groups)):
            main.wait_event(self._ev_done[g])
        plans = LayerPlans.cat([r[0] for r in parts])
        cells = torch.cat([r[2] for r in parts])
        tiles = torch.cat([r[3] for r in parts])
        for r in parts:  # group-stream tensors now read on the caller's stream
            pl = r[0]
            ts = [v for v in vars(pl).values() if isinstance(v, torch.Tensor)]
            ts += list(getattr(pl, "line_arrays", ())) + [r[2], r[3]]
            for t in ts:
                t.record_stream(main)
        return plans, out, cells, tiles

    # -------------------------------------------------------------- decode
    def _step(self, store: QKVStore, q_buf, out_buf, compressed: bool, max_cols: int, stream=None):
        """One decode step of every layer: K6 per layer reading q from the Q
        archive at the device cache length, each launched as a programmatic
        dependent of the previous layer's kernel, then the counter advance."""
        st = self.stack
        for l in range(self.shape.n_layers):
            # layer 0 follows the counter advance (or an event) in full: its tile
            # prefetch reads the step counters those kernels write
            st.step_archive(l, store.q[l], store.k[l], store.v[l], compressed, max_cols, out_buf[l], pdl=l > 0,
                            stream=stream)
        st.advance(stream=stream)

    def _graph(self, key, name, fn):
        """CUDA graph of a fixed launch sequence, captured once per key (the
        kernels read the cache length and deque position from the device step
        counters, so a graph serves every step and turn of its shape bucket)."""
        g = self._graphs.get(key)
        if g is None:
            st = self.stack
            host = (st.length, st.appended)
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                g = _lib.Captured(name, s, fn)
            torch.cuda.current_stream().wait_stream(s)
            st.length, st.appended = host  # capture does not execute; restore the host mirror
            self._graphs[key] = g
        return g

    def decode(self, store: QKVStore, L0: int, max_new: int, use_graphs: bool = True, out_sink=None,
               events: list | None = None, run_sink=None):
        """max_new decode steps (kvcompress.py:200-239) from cache length L0,
        after prefill() set the counters. Returns the last step's outputs
        [L, n_q, d]; out_sink(step, out_buf) is called after every step.
        events: if a list, every compression event appends a device snapshot
        (step n_o, cache length, selected ids, score coverage) -- no host sync;
        event_log() turns them into the reference's event records and
        decode_op_counts() into its decode op counts.
        run_sink(step0, outs): with multi-step graphs, called after each run of
        steps between two events with that run's outputs [n, L, n_q, d] (one
        call per run instead of one host round trip per step: e.g. the
        head-sharded output all-gather)."""
        p, sh = self.params, self.shape
        st = self.stack
        if L0 + max_new > store.length:
            raise CacheCorrupt(f"decode of positions [{L0}, {L0 + max_new}) but the store holds {store.length} "
                               "(append the decoded tokens' q / k / v first)")
        self._last_decode = (L0, max_new, events)
        self._obs_nb = None
        if p.mode == "obswindow" and p.comp.budget is not None:
            return self._decode_obswindow(store, L0, max_new, events, out_sink, run_sink)

        def snap(n_o):
            if events is not None:
                events.append({"step": n_o, "length": st.length, "sel": st.sel_ids.clone(),
                               "n_sel": st.n_sel.clone(), "cov": st.score_cov.clone()})
        comp = p.comp if p.mode == "loopserve" else CompressionConfig(budget=None)
        if p.mode == "dense":
            st.set_step(L0, 0)
        n_dense = max_new if comp.budget is None else min(max_new, comp.warmup - 1)
        # grid sizes come from column bounds; bucket them so graphs are reused
        dense_cols = min(st.row_cap, -(-(L0 + n_dense + 1) // GRAPH_BUCKET) * GRAPH_BUCKET)
        comp_cols = min((comp.budget or 0) + self.window + 1, L0 + max_new + 1)
        ev_len = min(st.row_cap, -(-(L0 + max_new) // GRAPH_BUCKET) * GRAPH_BUCKET)
        q_buf, out_buf = self._q_buf, self._out_buf
        # K/V rows each step reads (all layers), 4*d bytes each (bf16 K + V):
        # dense steps read each archive row once per KV head (the q-group
        # shares it); compressed steps read each q-head's own compacted cache
        # (per-q-head kept sets) plus the recent window
        for t in range(max_new):
            if t < n_dense:
                self.decode_log.append(("dense", (L0 + t + 1) * sh.n_kv * sh.n_layers))
            else:
                self.decode_log.append(("comp", min(comp_cols, L0 + t + 1) * sh.n_q * sh.n_layers))
        if not use_graphs:
            compressed = False
            for n_o in range(1, max_new + 1):
                if comp.event_at(n_o):
                    st.event(comp.budget, store.k, store.v, max_len=ev_len)
                    snap(n_o)
                    compressed = True
                self._step(store, q_buf, out_buf, compressed, comp_cols if compressed else dense_cols)
                if out_sink is not None:
                    out_sink(n_o - 1, out_buf)
            return out_buf
        # graphs bake in the store's K/V/Q pointers: key them on those, not on
        # id(store) (a recycled id would replay a graph bound to freed memory)
        sk = (store.q.data_ptr(), store.k.data_ptr(), store.v.data_ptr(), tuple(store.k.shape))
        graphs = {}
        if n_dense > 0:
            graphs["dense"] = self._graph(("dense", sk, dense_cols), "decode_graph_dense",
                                          lambda: self._step(store, q_buf, out_buf, False, dense_cols))
        if n_dense < max_new:
            graphs["comp"] = self._graph(("comp", sk, comp_cols), "decode_graph_comp",
                                         lambda: self._step(store, q_buf, out_buf, True, comp_cols))
            graphs["event"] = self._graph(("event", sk, comp.budget, ev_len), "decode_graph_event",
                                          lambda: st.event(comp.budget, store.k, store.v, max_len=ev_len))
        compressed = False
        if out_sink is None:
            # no per-step host work: every run of steps between two events is one
            # graph of that many steps (the kernels read the device counters, so
            # a multi-step graph is the same launch sequence back to back)
            ring = None
            if run_sink is not None:
                if self._ring is None or self._ring.shape[0] < max_new:
                    self._ring = torch.empty((max_new,) + tuple(out_buf.shape), dtype=out_buf.dtype,
                                             device=out_buf.device)
                    self._graphs = {k: v for k, v in self._graphs.items() if k[-1] != "ring"}
                ring = self._ring
            n_o = 1
            while n_o <= max_new:
                if comp.event_at(n_o):
                    graphs["event"].replay()
                    snap(n_o)
                    compressed = True
                nxt = n_o + 1
                while nxt <= max_new and not comp.event_at(nxt):
                    nxt += 1
                n = nxt - n_o
                kind, cols = ("comp", comp_cols) if compressed else ("dense", dense_cols)
                if ring is None:
                    g = self._graph((kind, sk, cols, n), f"decode_graph_{kind}",
                                    lambda n=n, c=compressed, cols=cols: [self._step(store, q_buf, out_buf, c, cols)
                                                                          for _ in range(n)])
                else:  # step k of the run writes ring[k]
                    g = self._graph((kind, sk, cols, n, "ring"), f"decode_graph_{kind}",
                                    lambda n=n, c=compressed, cols=cols: [self._step(store, q_buf, ring[k], c, cols)
                                                                          for k in range(n)])
                g.replay()
                st.length += n
                st.appended += n
                if ring is not None:
                    run_sink(n_o - 1, ring[:n])
                n_o = nxt
            return ring[n - 1] if ring is not None else out_buf
        for n_o in range(1, max_new + 1):
            if comp.event_at(n_o):
                graphs["event"].replay()
                snap(n_o)
                compressed = True
            graphs["comp" if compressed else "dense"].replay()
            st.length += 1
            st.appended += 1
            out_sink(n_o - 1, out_buf)
        return out_buf

    def check(self, stream=None) -> None:
        """Synchronise and raise the reference exception any kernel of this
        process recorded on the device since the last check (NonFiniteInput /
        AllMaskedRow from the sampled-row softmax, EmptyPlan from the sparse
        attention). prefill()/decode() stay asynchronous; call this where the
        caller would read results anyway."""
        _lib.device_status(stream, what="SessionEngine")

    # ------------------------------------------------------- session records
    def event_log(self, events: list, head_offset: int = 0) -> list[dict]:
        """kvcompress.py:217-224 records {step, head "L{l}H{h}", retained_ids,
        score_coverage} from decode(events=...) snapshots: retained_ids =
        retained_union(selected, window, length) (kvcompress.py:214)."""
        import numpy as np

        sh, W = self.shape, self.window
        out = []
        for ev in events:
            if "base" in ev:  # the obswindow baseline's one selection (session.py:226-234)
                keep = [int(g) for g in ev["base"].cpu().numpy()]
                out += [{"step": 0, "head": f"L{l}H{h + head_offset}", "retained_ids": list(keep),
                         "score_coverage": 1.0} for l in range(sh.n_layers) for h in range(sh.n_q)]
                continue
            sel, n_sel, cov = ev["sel"].cpu().numpy(), ev["n_sel"].cpu().numpy(), ev["cov"].cpu().numpy()
            L = ev["length"]
            recent = np.arange(max(0, L - W), L)
            for l in range(sh.n_layers):
                for h in range(sh.n_q):
                    hr = l * sh.n_q + h
                    keep = np.union1d(sel[hr, :n_sel[hr]], recent)
                    out.append({"step": ev["step"], "head": f"L{l}H{h + head_offset}",
                                "retained_ids": [int(g) for g in keep], "score_coverage": float(cov[hr])})
        return out

    def decode_op_counts(self, events: list) -> dict:
        """decode_scores / decode_steps of session.py:186-191 for the last
        decode(): every step scores |working| + 1 cells per (layer, head)
        (model.py:236-237), working = all positions before the first event,
        retained_union(selected, W, length) after it (kvcompress.py:234-237)."""
        import numpy as np

        L0, max_new, _ = self._last_decode
        sh, W = self.shape, self.window
        if self._obs_nb is not None:  # obswindow: base + the appended positions (session.py:243-253)
            nb = self._obs_nb
            return {"decode_scores": sh.n_layers * sh.n_q * sum(nb + t + 1 for t in range(max_new)),
                    "decode_steps": max(0, max_new - 1)}
        by_step = {ev["step"]: ev for ev in events}
        cur = None
        total = 0
        for n_o in range(1, max_new + 1):
            length = L0 + n_o - 1  # cache length when token n_o is appended
            if n_o in by_step:
                ev = by_step[n_o]
                cur = (ev["sel"].cpu().numpy(), ev["n_sel"].cpu().numpy())
            if cur is None:
                total += sh.n_layers * sh.n_q * (length + 1)
            else:
                sel, n_sel = cur
                lo = max(0, length - W)
                for hr in range(sh.n_layers * sh.n_q):
                    s = sel[hr, :n_sel[hr]]
                    total += int(n_sel[hr]) + (length - lo) - int(np.count_nonzero(s >= lo)) + 1
        return {"decode_scores": total, "decode_steps": max(0, max_new - 1)}

    def prefill_op_counts(self, res: "PrefillOut") -> dict:
        """prefill_scores / prefill_dense_cells of session.py:186-189: sampled
        scoring cells (prefill.py:388-389) + sparse attention cells
        (tensor_ops.py:172-174), all layers and heads."""
        sh = self.shape
        scores = 0
        for l in range(sh.n_layers):
            if res.cells[l] is not None:
                scores += int(res.cells[l].sum().item()) + int(res.plans[l].score_count.sum().item())
            else:
                scores += sh.n_q * sum(min(res.n_total, res.n_total - res.n_new + r + 1) for r in range(res.n_new))
        return {"prefill_scores": scores, "prefill_dense_cells": sh.n_layers * sh.n_q * res.n_new * res.n_total}

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
