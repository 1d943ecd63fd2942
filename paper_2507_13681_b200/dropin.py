"""Switch a reference LoopServe installation onto the B200 path.

The reference binds its hot-path functions by name at import time
(SURVEY.md section 8b): session.py:19-37 imports `sparsify_head`, model.py:20
imports `masked_sparse_attention` / `scaled_dot_attention`. A drop-in therefore
rebinds the names in the CALLING modules, not only the defining ones:

    import loopserve.session, loopserve.model, loopserve.prefill, loopserve.tensor_ops
    from paper_2507_13681_b200 import dropin
    dropin.install()          # every later run_turn / forward_extend uses the CUDA kernels
    ...
    dropin.uninstall()

The replacements keep the reference signatures, return types (SparsePlan /
numpy Z / AttentionBlock-compatible objects) and exception classes; they need
a CUDA device and the built library (no CPU fallback).
"""

from __future__ import annotations

import importlib
import sys

# (module, attribute) -> (our module, our attribute)
PATCHES = {
    ("loopserve.session", "sparsify_head"): ("prefill", "sparsify_head"),
    ("loopserve.prefill", "sparsify_head"): ("prefill", "sparsify_head"),
    ("loopserve.model", "masked_sparse_attention"): ("tensor_ops", "masked_sparse_attention"),
    ("loopserve.tensor_ops", "masked_sparse_attention"): ("tensor_ops", "masked_sparse_attention"),
    ("loopserve.model", "scaled_dot_attention"): ("tensor_ops", "scaled_dot_attention"),
    ("loopserve.tensor_ops", "scaled_dot_attention"): ("tensor_ops", "scaled_dot_attention"),
}

_saved: dict = {}


def install(modules: dict | None = None) -> list[str]:
    """Rebind every reference name in PATCHES that is importable (or present
    in `modules`, a {name: module} map used by tests). Returns the patched
    'module.attr' names. The CUDA library is loaded first so a missing build
    fails here, loudly, instead of at the first call."""
    from . import _lib

    _lib.lib()
    done = []
    for (mod_name, attr), (ours, our_attr) in PATCHES.items():
        mod = (modules or {}).get(mod_name) or sys.modules.get(mod_name)
        if mod is None:
            try:
                mod = importlib.import_module(mod_name)
            except ImportError:
                continue
        if not hasattr(mod, attr):
            continue
        key = (id(mod), attr)
        if key not in _saved:
            _saved[key] = (mod, getattr(mod, attr))
        fn = getattr(importlib.import_module(f"{__package__}.{ours}"), our_attr)
        setattr(mod, attr, fn)
        done.append(f"{mod_name}.{attr}")
    return done


def uninstall() -> None:
    for (_, attr), (mod, fn) in list(_saved.items()):
        setattr(mod, attr, fn)
    _saved.clear()


__all__ = ["install", "uninstall", "PATCHES"]
