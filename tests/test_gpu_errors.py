"""Reference error semantics on the device path (errors.py:4-65):
NonFiniteInput from the sampled-row softmax (tensor_ops.py:34-38) detected by
K1 on the device, EmptyPlan for alpha = 0 in the engine and for an empty plan
in K5 (tensor_ops.py:165-166), and the C-ABI status mapping."""

import numpy as np
import pytest
import torch

from paper_2507_13681_b200 import _lib
from paper_2507_13681_b200 import prefill as pf
from paper_2507_13681_b200 import tensor_ops as tops
from paper_2507_13681_b200.errors import EmptyPlan, InvalidAlpha, NonFiniteInput

pytestmark = pytest.mark.gpu


def test_sparsify_head_non_finite_input(cuda_lib):
    rng = np.random.Generator(np.random.PCG64(1))
    K = rng.normal(size=(300, 64))
    Q = rng.normal(size=(40, 64))
    pos = np.sort(rng.choice(np.arange(100, 300), 40, replace=False))
    pf.sparsify_head(Q, K, 0.9, pos)  # clean input: no error
    K[5, 3] = np.nan
    with pytest.raises(NonFiniteInput):
        pf.sparsify_head(Q, K, 0.9, pos)
    K[5, 3] = np.inf
    with pytest.raises(NonFiniteInput):
        pf.sparsify_head(Q, K, 0.9, pos)
    _lib.device_status()  # cleared by the raise: nothing pending
    with pytest.raises(InvalidAlpha):
        pf.sparsify_head(Q, K, 1.5, pos)


def test_engine_alpha_zero_empty_plan(cuda_lib):
    from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams

    shape = AttnShape(1, 2, 1, 64)
    store = QKVStore.synthetic(shape, 400, seed=2)
    eng = SessionEngine(shape, SessionParams(alpha=0.0, max_new=4), 400)
    with pytest.raises(EmptyPlan):
        eng.prefill(store, 0, 0, 300)


def test_k5_empty_plan_reported_by_device(cuda_lib):
    from paper_2507_13681_b200.synth import SynthSpec, layer_qkv_torch

    spec = SynthSpec(2, 1, 128, 512, seed=3)
    Q, K, V = layer_qkv_torch(spec, 0)
    sl = torch.zeros((2, 512), dtype=torch.int32, device="cuda")
    vt = torch.zeros((2, 512), dtype=torch.int32, device="cuda")
    counts = torch.tensor([[1, 0], [0, 0]], dtype=torch.int32, device="cuda")  # head 1: no line
    _lib.device_status()
    tops.attention_layer(Q, K, V, sl, vt, counts, 512, 512, 1)
    with pytest.raises(EmptyPlan):
        _lib.device_status(what="attention_layer")
    counts[1, 0] = 1
    tops.attention_layer(Q, K, V, sl, vt, counts, 512, 512, 1)
    _lib.device_status()  # a plan with a line on every head: no error
