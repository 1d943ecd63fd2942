"""B200-native LoopServe hot paths (arxiv 2507.13681).

Drop-in for the reference package's prefill-sparsify and decode-compress
calls (same names, config fields and exceptions), computed by hand-written
sm_100a CUDA kernels behind the C ABI in include/loopserve_b200.h.
There is no CPU fallback: without the built library or a CUDA device the
compute functions raise NativeLibraryMissing.
"""

from .errors import (  # noqa: F401
    AllMaskedRow, CacheCorrupt, DimensionMismatch, EmptyBlock, EmptyPlan, EmptyWindow, InstanceTooLarge,
    InvalidAlpha, InvalidConfig, InvalidIds, LoopServeError, NativeError, NativeLibraryMissing, NonFiniteInput,
    SequenceTooLong, SizeMismatch)
from .opcount import OpCounter  # noqa: F401

__version__ = "0.1.0"


_EXPORTS = {
    "SparsePlan": "prefill", "Line": "prefill", "sample_rows": "prefill", "sparsify_head": "prefill",
    "sparsify_layer": "prefill", "greedy_select_lines": "prefill", "vertical_length": "prefill",
    "slash_length": "prefill", "masked_sparse_attention": "tensor_ops", "scaled_dot_attention": "tensor_ops",
    "AttentionBlock": "tensor_ops", "attention_layer": "tensor_ops", "CompressionConfig": "kvcompress",
    "DecodeStats": "kvcompress", "KVCacheHead": "kvcompress", "DecodeStack": "kvcompress",
    "accumulate_scores": "kvcompress", "select_topB_obs": "kvcompress", "retained_union": "kvcompress",
    "compact_cache": "kvcompress", "progressive_decode": "kvcompress", "token_scores": "kvcompress",
    "SessionParams": "engine", "SessionEngine": "engine", "AttnShape": "engine", "QKVStore": "engine",
}


def __getattr__(name):  # lazy: importing the package must not need torch/CUDA
    import importlib

    mod = _EXPORTS.get(name)
    if mod is None:
        raise AttributeError(name)
    return getattr(importlib.import_module(f".{mod}", __name__), name)
