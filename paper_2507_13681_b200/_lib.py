"""ctypes binding of libloopserve_b200.so (the C ABI in include/loopserve_b200.h).

The library is built in-tree by `__graft_entry__.build()` (nvcc, sm_100a).
Loading never falls back to anything: a missing library raises
NativeLibraryMissing, a failing call raises the mapped LoopServeError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import STATUS, NativeError, NativeLibraryMissing

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LS_LIB_PATH") or os.path.join(HERE, "libloopserve_b200.so")  # override: A/B builds

_lock = threading.Lock()
_lib = None

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
U64 = C.c_uint64
F64 = C.c_double
SZ = C.c_size_t


class LayerDesc(C.Structure):
    _fields_ = [("n_heads", I32), ("n_kv_heads", I32), ("head_dim", I32), ("n_new", I32),
                ("n_total", I32), ("row_offset", I32), ("q_head_stride", I64),
                ("kv_head_stride", I64), ("out_row_stride", I64)]


class DecodeStackDesc(C.Structure):
    _fields_ = [("n_layers", I32), ("n_heads", I32), ("n_kv_heads", I32), ("head_dim", I32), ("window", I32),
                ("row_cap", I32), ("sparse_cap", I32), ("budget_cap", I32), ("kv_layer_stride", I64),
                ("kv_head_stride", I64), ("ring_s", P), ("ring_ml", P), ("ring_ids", P), ("ring_n", P),
                ("ring_dense", P), ("sel_ids", P), ("n_sel", P), ("ck", P), ("cv", P), ("partials", P),
                ("counters", P), ("step", P), ("n_a", P)]


LD = C.POINTER(LayerDesc)
DS = C.POINTER(DecodeStackDesc)

# name -> (restype, argtypes)
SIGNATURES = {
    "ls_last_error": (C.c_char_p, []),
    "ls_version": (C.c_int, []),
    "ls_device_status": (C.c_int, [C.POINTER(I32), P]),
    "ls_debug_set_buffer": (C.c_int, [P]),
    "ls_device_info": (C.c_int, [C.POINTER(C.c_int), C.c_char_p, C.c_int]),
    "ls_sample_size": (C.c_int, [I32, F64, I32, C.POINTER(I32)]),
    "ls_sample_rows_workspace": (SZ, [I32, I32]),
    "ls_sample_rows": (C.c_int, [U64, I32, I32, I32, I32, I32, I32, F64, I32, P, P, SZ, P]),
    "ls_sample_rows_host": (C.c_int, [U64, I32, I32, I32, I32, F64, I32, P]),
    "ls_head_seed_host": (U64, [U64, I32, I32, I32]),
    "ls_score_lines_workspace": (SZ, [LD, I32]),
    "ls_score_lines": (C.c_int, [LD, I32, P, P, P, P, P, P, P, P, P, P, P, SZ, P]),
    "ls_score_lines_simt": (C.c_int, [LD, I32, P, P, P, P, P, P, P, P, P, P, P, SZ, P]),
    "ls_select_lines_workspace": (SZ, [LD, I32]),
    "ls_select_lines": (C.c_int, [LD, I32, F64, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P,
                                  SZ, P]),
    "ls_select_lines_ready": (C.c_int, [LD, I32, F64, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, I32, P,
                                        SZ, P]),
    "ls_stream_wait_value": (C.c_int, [P, P, I32]),
    "ls_greedy_dense": (C.c_int, [I32, P, P, P, P, I32, P, P, P, P, F64, F64, P, P, I32, I32, P, P,
                                  P, P, P, P, SZ, P]),
    "ls_vs_attention_workspace": (SZ, [LD]),
    "ls_vs_attention": (C.c_int, [LD, P, P, P, P, P, P, P, I32, P, P, SZ, P]),
    "ls_vs_attention_simt": (C.c_int, [LD, P, P, P, P, P, P, P, I32, P, P, SZ, P]),
    "ls_vs_attention_ex": (C.c_int, [LD, P, P, P, P, P, P, P, I32, P, P, P, SZ, P]),
    "ls_plan_rows": (C.c_int, [LD, I32, P, P, P, P, P, P, I64, I64, P]),
    "ls_dense_attention": (C.c_int, [LD, P, P, P, P, I32, P]),
    "ls_plan_coverage_workspace": (SZ, [LD]),
    "ls_plan_coverage": (C.c_int, [LD, P, P, P, P, P, P, P, P, SZ, P]),
    "ls_decode_partials_size": (SZ, [DS, I32]),
    "ls_decode_step": (C.c_int, [DS, I32, P, P, P, I32, I32, P, I32, P]),
    "ls_decode_step_archive": (C.c_int, [DS, I32, P, I64, P, P, I32, I32, P, I32, I32, P]),
    "ls_decode_advance": (C.c_int, [DS, P]),
    "ls_decode_select_workspace": (SZ, [DS]),
    "ls_decode_event": (C.c_int, [DS, I32, I32, P, P, P, P, P, SZ, P]),
    "ls_accumulate_scores": (C.c_int, [I32, P, P, P, I32, P, P, P]),
    "ls_top_by_score_workspace": (SZ, [I32]),
    "ls_top_by_score": (C.c_int, [I32, P, P, I32, I32, I32, P, P, P, SZ, P]),
    "ls_retained_union": (C.c_int, [I32, P, I32, I32, I32, P, P, P, SZ, P]),
    "ls_kv_compact": (C.c_int, [I32, P, P, P, I32, P, I32, I32, P, P, P, P]),
    "ls_gather_attention": (C.c_int, [I32, I32, I32, P, I64, P, P, I64, P, P, P, P, P]),
    "ls_obs_window_scores": (C.c_int, [I32, I32, P, I64, I64, I32, P, P]),
    "ls_gather_rows": (C.c_int, [I32, I32, P, P, I64, P, I64, I32, P]),
}


def lib():
    """Load (once) and return the ctypes library, or raise NativeLibraryMissing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    msg = lib().ls_last_error().decode(errors="replace")
    exc = STATUS.get(int(status), NativeError)
    raise exc(f"{what}: {msg}" if what else msg)


# CUDA kernels each C-ABI entry launches (memsets/memcpys not counted);
# bench.py reports the sum over its timed region as `gpu_launches`.
KERNELS_PER_CALL = {
    "ls_sample_rows": 1, "ls_score_lines": 3, "ls_select_lines": 6, "ls_select_lines_ready": 4,
    "ls_greedy_dense": 5,
    "ls_vs_attention": 3, "ls_vs_attention_ex": 3, "ls_vs_attention_simt": 3, "ls_plan_rows": 4, "ls_dense_attention": 1,
    "ls_plan_coverage": 7,
    "ls_decode_step": 1, "ls_decode_step_archive": 1, "ls_decode_advance": 1, "ls_decode_event": 3,
    "ls_accumulate_scores": 1, "ls_top_by_score": 1, "ls_retained_union": 1, "ls_kv_compact": 1,
    "ls_gather_attention": 1, "ls_obs_window_scores": 1, "ls_gather_rows": 1,
}
launch_count = 0
entry_hook = None  # optional callable(name, phase) used by bench.py to time entries


_capture = None  # list collecting kernel counts while a CUDA graph is being captured


def call(name: str, *args):
    global launch_count
    if _capture is not None:  # captured, not executed: no timing, count at replay
        check(getattr(lib(), name)(*args), name)
        _capture.append(KERNELS_PER_CALL.get(name, 0))
        return
    if entry_hook is not None:
        entry_hook(name, "begin")
    check(getattr(lib(), name)(*args), name)
    if entry_hook is not None:
        entry_hook(name, "end")
    launch_count += KERNELS_PER_CALL.get(name, 0)


class Captured:
    """A CUDA graph of C-ABI calls; replay() counts its kernels and reports
    it to entry_hook under `name` like a single entry."""

    def __init__(self, name: str, stream, fn):
        import torch

        global _capture
        self.name = name
        self.graph = torch.cuda.CUDAGraph()
        _capture = []
        try:
            with torch.cuda.graph(self.graph, stream=stream):
                fn()
            self.kernels = sum(_capture)
        finally:
            _capture = None

    def replay(self):
        global launch_count
        if entry_hook is not None:
            entry_hook(self.name, "begin")
        self.graph.replay()
        if entry_hook is not None:
            entry_hook(self.name, "end")
        launch_count += self.kernels


def device_status(stream=None, what: str = "device") -> None:
    """Raise the reference exception a kernel recorded on the device since the
    last check (ls_device_status: synchronises the stream)."""
    st = C.c_int32(0)
    check(lib().ls_device_status(C.byref(st), stream_ptr(stream)), "ls_device_status")
    if st.value:
        exc = STATUS.get(int(st.value), NativeError)
        raise exc(f"{what}: reported by the device (status {st.value})")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
