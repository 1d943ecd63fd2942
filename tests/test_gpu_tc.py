"""Tensor-core kernels cross-checked at C2-like sizes: K1 (tcgen05 scoring +
line sums) against the CUDA-core path and the fp64 oracle, and the resulting
plans against the oracle's (identical or near-tie)."""

import ctypes

import numpy as np
import pytest
import torch

from oracle import attention as oatt
from oracle import prefill as opf
from paper_2507_13681_b200 import _lib
from paper_2507_13681_b200 import prefill as pf
from paper_2507_13681_b200.synth import SynthSpec, layer_qkv_torch
from parity import check_plan

pytestmark = pytest.mark.gpu


def _score(entry, qb, K, rows, n_new, n_total, n_kv):
    H, n_s = rows.shape
    d = qb.shape[-1]
    L = pf.layer_desc(H, n_kv, d, n_new, n_total, qb.stride(0), K.stride(0))
    dev = qb.device
    out = dict(v_w=torch.empty((H, n_total), dtype=torch.float64, device=dev),
               v_max=torch.empty((H, n_total), dtype=torch.float32, device=dev),
               s_w=torch.empty((H, n_total), dtype=torch.float64, device=dev),
               s_max=torch.empty((H, n_total), dtype=torch.float32, device=dev),
               rs=torch.empty((H, n_s, 2), dtype=torch.float32, device=dev),
               total=torch.empty(H, dtype=torch.float64, device=dev),
               cnt=torch.empty(H, dtype=torch.int64, device=dev))
    n = _lib.lib().ls_score_lines_workspace(ctypes.byref(L), n_s)
    ws = torch.empty(n, dtype=torch.uint8, device=dev)
    _lib.call(entry, ctypes.byref(L), n_s, qb.data_ptr(), K.data_ptr(), rows.data_ptr(), out["v_w"].data_ptr(),
              out["v_max"].data_ptr(), out["s_w"].data_ptr(), out["s_max"].data_ptr(), out["rs"].data_ptr(),
              out["total"].data_ptr(), out["cnt"].data_ptr(), ws.data_ptr(), n, _lib.stream_ptr())
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("d,n_q,n_kv,ro,n_new,rate", [(128, 4, 1, 5000, 5128, 0.1), (64, 4, 2, 300, 700, 0.1),
                                                      (128, 2, 1, 0, 1000, 1.0), (128, 2, 2, 10128, 5128, 0.1)])
def test_score_lines_tc_vs_simt_vs_oracle(cuda_lib, d, n_q, n_kv, ro, n_new, rate):
    n_total = ro + n_new
    spec = SynthSpec(n_q, n_kv, d, n_total, seed=11)
    Q, K, V = layer_qkv_torch(spec, 0)
    qb = Q[:, ro:].contiguous()
    rows = pf.sample_rows_device(n_new, rate, 32, 5, 2, 1, 0, n_q)
    tc = _score("ls_score_lines", qb, K, rows, n_new, n_total, n_kv)
    si = _score("ls_score_lines_simt", qb, K, rows, n_new, n_total, n_kv)
    assert torch.equal(tc["cnt"], si["cnt"])
    for key in ("v_w", "s_w"):
        scale = si[key].abs().max().item()
        assert (tc[key] - si[key]).abs().max().item() <= 1e-5 * max(1.0, scale), key
    # max cells: one fp32 probability each; tcgen05 and FFMA accumulate the
    # 128-term logit in different orders (|s| up to ~20 -> ~1e-6 logit error,
    # a few 1e-5 relative in exp)
    for key in ("v_max", "s_max"):
        assert (tc[key] - si[key]).abs().max().item() <= 5e-5 * max(1.0, si[key].abs().max().item()), key
    # oracle on one head
    group = n_q // n_kv
    h = n_q - 1
    r = rows[h].cpu().numpy()
    pos = ro + r
    Qd = qb[h].double().cpu().numpy()[r]
    Kd = K[h // group, :n_total].double().cpu().numpy()
    W = oatt.softmax_rows(opf.sampled_logits(Qd, Kd, pos))
    a = opf.line_arrays(W, pos)
    assert np.abs(tc["v_w"][h].cpu().numpy() - a["v_w"]).max() <= 1e-5 * max(1.0, a["v_w"].max())
    assert np.abs(tc["s_w"][h].cpu().numpy() - a["s_w"]).max() <= 1e-5 * max(1.0, a["s_w"].max())
    assert abs(tc["total"][h].item() - W.sum()) <= 1e-4


def test_c2_turn3_plans_match_oracle(cuda_lib):
    """Full C2 turn-3 geometry (n_new 5128, n_total 15256, d 128) on two
    q-heads: device plans equal the oracle's or differ only at a near-tie."""
    ro, n_new = 10128, 5128
    n_total = ro + n_new
    spec = SynthSpec(8, 2, 128, n_total, seed=21)
    Q, K, V = layer_qkv_torch(spec, 0)
    qb = Q[:, ro:].contiguous()
    rows = pf.sample_rows_device(n_new, 0.1, 32, 0, 2, 0, 0, 8)
    plans = pf.sparsify_layer(qb, K, rows, 0.955, n_new, n_total, 2)
    hp = plans.to_host()
    seqs = plans.pick_sequences()
    outcomes = []
    for h in (0, 5):
        r = rows[h].cpu().numpy()
        pos = ro + r
        Qd = qb[h].double().cpu().numpy()[r]
        Kd = K[h // 4].double().cpu().numpy()
        oplan = opf.sparsify_head(Qd, Kd, 0.955, pos)
        W = oatt.softmax_rows(opf.sampled_logits(Qd, Kd, pos))
        sl, vl = opf.line_sums_view(W, pos)
        outcomes.append(check_plan(oplan, hp[h], seqs[h], {x.index: x.weight for x in sl},
                                   {x.index: x.weight for x in vl}))
    print("C2 t3 plan parity:", outcomes)
