"""Switch a reference LoopServe installation onto the B200 path.

The reference binds its hot-path functions by name at import time
(SURVEY.md section 8b): session.py:19-37 imports `sparsify_head`,
`decode_step`, `retained_union`, `select_topB_obs`, `token_scores`;
model.py:20 imports `masked_sparse_attention` / `scaled_dot_attention`;
kvcompress.py:18 imports `decode_step`, and `progressive_decode`
(kvcompress.py:167-240) calls `accumulate_scores`, `_top_by_score` and
`retained_union` through its module globals. A drop-in therefore rebinds the
names in the CALLING modules, not only the defining ones:

    import loopserve.session
    from paper_2507_13681_b200 import dropin
    dropin.install()          # every later run_turn / progressive_decode uses the CUDA kernels
    ...
    dropin.uninstall()

Prefill: `sparsify_head` (K0-K4), `masked_sparse_attention` (K5),
`scaled_dot_attention`. Decode: `decode_step` -- the reference's one-token
forward (model.py:289-311) with its working-set attention (model.py:232-241)
on the device for every head of a layer in one launch (ls_gather_attention,
K/V mirrored in HBM as bf16, appended row by row), while the toy model's own
embedding / RMSNorm / projections / FFN / logits stay the reference's
functions, called from the patched module -- plus `accumulate_scores`,
`_top_by_score`, `select_topB_obs`, `token_scores`, `retained_union`,
`compact_cache`, `ground_truth_topB`, `overlap_rate` (kvcompress.py:58-147).

The replacements keep the reference signatures and return types and raise
the reference's own exception classes (errors.py:4-65); they need a CUDA
device and the built library (no CPU fallback).
"""

from __future__ import annotations

import functools
import importlib
import sys
import weakref

import numpy as np

# (module, attribute) -> (our module, our attribute); "@decode_step" entries are
# built per installation around the reference's model module
PATCHES = {
    ("loopserve.session", "sparsify_head"): ("prefill", "sparsify_head"),
    ("loopserve.prefill", "sparsify_head"): ("prefill", "sparsify_head"),
    ("loopserve.model", "masked_sparse_attention"): ("tensor_ops", "masked_sparse_attention"),
    ("loopserve.tensor_ops", "masked_sparse_attention"): ("tensor_ops", "masked_sparse_attention"),
    ("loopserve.model", "scaled_dot_attention"): ("tensor_ops", "scaled_dot_attention"),
    ("loopserve.tensor_ops", "scaled_dot_attention"): ("tensor_ops", "scaled_dot_attention"),
    ("loopserve.kvcompress", "accumulate_scores"): ("kvcompress", "accumulate_scores"),
    ("loopserve.kvcompress", "_top_by_score"): ("kvcompress", "_top_by_score"),
    ("loopserve.kvcompress", "select_topB_obs"): ("kvcompress", "select_topB_obs"),
    ("loopserve.kvcompress", "token_scores"): ("kvcompress", "token_scores"),
    ("loopserve.kvcompress", "retained_union"): ("kvcompress", "retained_union"),
    ("loopserve.kvcompress", "compact_cache"): ("kvcompress", "compact_cache"),
    ("loopserve.kvcompress", "ground_truth_topB"): ("kvcompress", "ground_truth_topB"),
    ("loopserve.kvcompress", "overlap_rate"): ("kvcompress", "overlap_rate"),
    ("loopserve.session", "retained_union"): ("kvcompress", "retained_union"),
    ("loopserve.session", "select_topB_obs"): ("kvcompress", "select_topB_obs"),
    ("loopserve.session", "token_scores"): ("kvcompress", "token_scores"),
    ("loopserve.model", "decode_step"): ("@decode_step", None),
    ("loopserve.kvcompress", "decode_step"): ("@decode_step", None),
    ("loopserve.session", "decode_step"): ("@decode_step", None),
}

_saved: dict = {}


def _module(name: str, modules: dict | None):
    mod = (modules or {}).get(name) or sys.modules.get(name)
    if mod is None:
        try:
            mod = importlib.import_module(name)
        except ImportError:
            return None
    return mod


def _reference_errors(fn, errors_mod):
    """Re-raise our LoopServeError subclasses as the reference's class of the
    same name, so callers catching loopserve.errors.* keep working."""
    from .errors import LoopServeError

    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        try:
            return fn(*args, **kwargs)
        except LoopServeError as exc:
            cls = getattr(errors_mod, type(exc).__name__, None) if errors_mod is not None else None
            if cls is None or not isinstance(cls, type):
                raise
            raise cls(str(exc)) from exc

    wrapped.__b200__ = True
    return wrapped


# ------------------------------------------------------------ decode_step
class _ArchiveMirror:
    """bf16 copy in HBM of a reference KVCache (model.py:139-175): K/V rows
    [0, synced) are current. Rows are uploaded lazily before each decode step;
    KVCache.truncate (patched by install) lowers `synced`, so the rolled-back
    rows that the next turn re-prefills are uploaded again."""

    def __init__(self, cache):
        import torch

        c = cache.config
        self.k = torch.zeros((c.n_layers, c.n_heads, c.max_seq_len, c.d_k), dtype=torch.bfloat16, device="cuda")
        self.v = torch.zeros((c.n_layers, c.n_heads, c.max_seq_len, c.d_v), dtype=torch.bfloat16, device="cuda")
        self.synced = 0

    def sync(self, cache, upto: int) -> None:
        import torch

        if upto <= self.synced:
            self.synced = min(self.synced, upto)
            return
        lo = self.synced
        for l in range(len(cache.k)):
            self.k[l, :, lo:upto].copy_(torch.from_numpy(np.asarray(cache.k[l][:, lo:upto], np.float32)))
            self.v[l, :, lo:upto].copy_(torch.from_numpy(np.asarray(cache.v[l][:, lo:upto], np.float32)))
        self.synced = upto


_mirrors: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _mirror(cache) -> _ArchiveMirror:
    m = _mirrors.get(cache)
    if m is None:
        m = _ArchiveMirror(cache)
        _mirrors[cache] = m
    return m


def working_set_attention(q, k_layer, v_layer, cols_per_head):
    """model.py:232-241 for every head of one layer on the device:
    q [H, d] bf16, k_layer / v_layer [H, T, d] bf16, cols_per_head: H int
    arrays (the working set + the new position). Returns (out [H, d] fp64
    numpy, [w_h] fp64 numpy per head)."""
    import torch

    from . import _lib

    H, d = q.shape
    lens = np.array([len(c) for c in cols_per_head], dtype=np.int64)
    col_ptr = np.zeros(H + 1, dtype=np.int64)
    col_ptr[1:] = np.cumsum(lens)
    cols = np.concatenate([np.asarray(c, dtype=np.int32) for c in cols_per_head])
    dev = q.device
    cols_t = torch.as_tensor(cols, device=dev)
    ptr_t = torch.as_tensor(col_ptr, device=dev)
    out = torch.empty((H, d), dtype=torch.float64, device=dev)
    w = torch.empty(max(1, int(col_ptr[-1])), dtype=torch.float64, device=dev)
    _lib.call("ls_gather_attention", H, k_layer.shape[0], d, q.data_ptr(), int(q.stride(0)), k_layer.data_ptr(),
              v_layer.data_ptr(), int(k_layer.stride(0)), ptr_t.data_ptr(), cols_t.data_ptr(), out.data_ptr(),
              w.data_ptr(), _lib.stream_ptr())
    w_h = w.cpu().numpy()
    return out.cpu().numpy(), [w_h[col_ptr[h]:col_ptr[h + 1]] for h in range(H)]


def make_decode_step(model_mod):
    """decode_step (model.py:289-311) for the reference model module
    `model_mod`: one token through every layer, the working-set attention of
    all heads of a layer in one ls_gather_attention launch, the rest of the
    toy model through model_mod's own functions."""
    import torch

    errs = sys.modules.get(model_mod.__name__.rsplit(".", 1)[0] + ".errors")

    def decode_step(weights, cache, last_token, working_sets=None, counter=None):
        c = weights.config
        if working_sets is None:  # model.py:301-306: the full cache
            working_sets = {(l, h): np.arange(cache.length) for l in range(c.n_layers) for h in range(c.n_heads)}
        cache.validate()
        start = cache.length
        if start + 1 > c.max_seq_len:
            raise getattr(errs, "SequenceTooLong", ValueError)(
                f"{start + 1} tokens exceed max_seq_len={c.max_seq_len}")
        tok = int(last_token)
        if tok < 0 or tok >= c.vocab_size:
            raise getattr(errs, "DimensionMismatch", ValueError)("token id outside the vocabulary")
        if c.d_k != c.d_v:
            raise getattr(errs, "DimensionMismatch", ValueError)("the B200 decode step requires d_k == d_v")
        mirror = _mirror(cache)
        mirror.sync(cache, start)
        x = weights.token_embedding[[tok]] + weights.pos_embedding[[start]]
        obs_rows = {}
        for l, layer in enumerate(weights.layers):
            normed = model_mod.rms_norm(x, layer.attn_gain)
            qs, ks, vs = [], [], []
            for h, head in enumerate(layer.heads):
                Q, K_new, V_new = model_mod.qkv_project(normed, head)
                cache.k[l][h][start] = K_new[0]
                cache.v[l][h][start] = V_new[0]
                qs.append(Q[0])
                ks.append(K_new[0])
                vs.append(V_new[0])
            mirror.k[l, :, start].copy_(torch.from_numpy(np.asarray(ks, np.float32)))
            mirror.v[l, :, start].copy_(torch.from_numpy(np.asarray(vs, np.float32)))
            q = torch.from_numpy(np.asarray(qs, np.float32)).to("cuda").to(torch.bfloat16)
            cols = [np.append(np.asarray(working_sets[(l, h)], dtype=np.intp), start) for h in range(c.n_heads)]
            if counter is not None:
                for cl in cols:
                    counter.add(len(cl))
            out, w = working_set_attention(q, mirror.k[l], mirror.v[l], cols)
            for h in range(c.n_heads):
                obs_rows[(l, h)] = (cols[h], w[h])
            x = x + out.reshape(1, -1) @ layer.w_o
            hh = model_mod.rms_norm(x, layer.ffn_gain)
            x = x + np.maximum(hh @ layer.w1 + layer.b1, 0.0) @ layer.w2 + layer.b2
        cache.length = start + 1
        mirror.synced = start + 1
        logits = model_mod.logits_from_hidden(weights, x[-1])[0]
        return logits, model_mod.argmax_token(logits), obs_rows

    decode_step.__b200__ = True
    return decode_step


def _patch_truncate(model_mod):
    kv_cls = getattr(model_mod, "KVCache", None)
    if kv_cls is None or getattr(kv_cls.truncate, "__b200__", False):
        return
    orig = kv_cls.truncate

    def truncate(self, length):
        orig(self, length)
        m = _mirrors.get(self)
        if m is not None:
            m.synced = min(m.synced, int(length))

    truncate.__b200__ = True
    _saved[(id(kv_cls), "truncate")] = (kv_cls, orig)
    kv_cls.truncate = truncate


def install(modules: dict | None = None) -> list[str]:
    """Rebind every reference name in PATCHES that is importable (or present
    in `modules`, a {name: module} map used by tests). Returns the patched
    'module.attr' names. The CUDA library is loaded first so a missing build
    fails here, loudly, instead of at the first call."""
    from . import _lib

    _lib.lib()
    done = []
    model_mod = _module("loopserve.model", modules)
    errors_mod = _module("loopserve.errors", modules)
    decode_fn = make_decode_step(model_mod) if model_mod is not None else None
    if model_mod is not None:
        _patch_truncate(model_mod)
    for (mod_name, attr), (ours, our_attr) in PATCHES.items():
        mod = _module(mod_name, modules)
        if mod is None or not hasattr(mod, attr):
            continue
        if ours == "@decode_step":
            if decode_fn is None:
                continue
            fn = decode_fn
        else:
            fn = _reference_errors(getattr(importlib.import_module(f"{__package__}.{ours}"), our_attr), errors_mod)
        key = (id(mod), attr)
        if key not in _saved:
            _saved[key] = (mod, getattr(mod, attr))
        setattr(mod, attr, fn)
        done.append(f"{mod_name}.{attr}")
    return done


def uninstall() -> None:
    for (_, attr), (mod, fn) in list(_saved.items()):
        setattr(mod, attr, fn)
    _saved.clear()


__all__ = ["install", "uninstall", "PATCHES", "make_decode_step", "working_set_attention"]
