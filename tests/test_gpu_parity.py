"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's golden fixtures, on the same bf16 inputs.

Bars (SURVEY.md section 8c / BASELINE.json north_star):
  * index work (sampled rows, sort order, plans, kept-KV ids): bit-exact, or a
    divergence proven to be a near-tie (tests/parity.py);
  * attention outputs: within 2e-2 absolute of the fp64 oracle;
  * op counts: exact.
"""

import math

import numpy as np
import pytest
import torch

from oracle import attention as oatt
from oracle import kvcompress as okv
from oracle import prefill as opf
from oracle import seeding as oseed
from paper_2507_13681_b200 import kvcompress as kv
from paper_2507_13681_b200 import prefill as pf
from paper_2507_13681_b200 import tensor_ops as tops
from paper_2507_13681_b200.synth import SynthSpec, checksum, layer_qkv_numpy
from parity import check_plan, check_topb

pytestmark = pytest.mark.gpu
ATOL = 2e-2

PREFILL = ["prefill_small", "prefill_d128", "prefill_random", "prefill_alpha1", "prefill_first_turn"]


def _inputs(golden, name):
    c = golden.case(name)
    spec = SynthSpec(**c["spec"])
    Q, K, V = layer_qkv_numpy(spec, layer=0)
    assert checksum(Q, K, V) == c["checksum"]
    return c, spec, Q, K, V


# ------------------------------------------------------------------ K0
def test_sample_rows_device_matches_reference(cuda_lib, golden):
    for i, c in enumerate(golden.case("seeds")):
        rows = pf.sample_rows_device(c["n_new"], c["rate"], c["floor"], c["session_seed"], c["turn"],
                                     c["layer"], c["head"], 1)
        assert np.array_equal(rows[0].cpu().numpy(), golden[f"seeds/{i}/rows"]), f"case {i}"


def test_sample_rows_device_batched_layers_heads(cuda_lib):
    for n_new in (1000, 5128, 10128):
        rows = pf.sample_rows_device(n_new, 0.1, 32, 7, 2, 3, 0, 8, n_layers=4).cpu().numpy()
        for l in range(4):
            for h in range(8):
                ref = oseed.sample_rows(n_new, 0.1, 32, oseed.head_seed(7, 2, 3 + l, h))
                assert np.array_equal(rows[l, h], ref)


def test_sample_rows_raw_seed(cuda_lib):
    for seed in (0, 42, 2 ** 63 + 11):
        assert np.array_equal(pf.sample_rows(777, 0.1, 32, seed), oseed.sample_rows(777, 0.1, 32, seed))


# ---------------------------------------------------------- K1 line sums
@pytest.mark.parametrize("name", PREFILL)
def test_line_sums_match_oracle(cuda_lib, golden, name):
    c, spec, Q, K, V = _inputs(golden, name)
    ro, n_new = c["row_offset"], c["n_new"]
    n_total = ro + n_new
    group = spec.n_q // spec.n_kv
    for h in range(spec.n_q):
        rows = golden[f"{name}/{h}/rows"]
        pos = ro + rows
        Qb = Q[h, ro:n_total].astype(np.float64)
        Kb = K[h // group, :n_total].astype(np.float64)
        v_w, v_max, s_w, s_max, total = pf.line_sums_device(Qb[rows], Kb, pos)
        W = oatt.softmax_rows(opf.sampled_logits(Qb[rows], Kb, pos))
        a = opf.line_arrays(W, pos)
        assert np.abs(v_w - a["v_w"]).max() <= 1e-5 * max(1.0, a["v_w"].max())
        assert np.abs(s_w - a["s_w"]).max() <= 1e-5 * max(1.0, a["s_w"].max())
        assert np.abs(v_max - a["v_max"]).max() <= 1e-5
        assert np.abs(s_max - a["s_max"]).max() <= 1e-5
        assert abs(total - W.sum()) <= 1e-4


# ----------------------------------------------- sparsify_head (K1..K4)
@pytest.mark.parametrize("name", PREFILL)
def test_sparsify_plans_match_reference(cuda_lib, golden, name):
    c, spec, Q, K, V = _inputs(golden, name)
    ro, n_new = c["row_offset"], c["n_new"]
    n_total = ro + n_new
    group = spec.n_q // spec.n_kv
    qb = torch.from_numpy(Q[:, ro:n_total]).cuda().to(torch.bfloat16).contiguous()
    kk = torch.from_numpy(K[:, :n_total]).cuda().to(torch.bfloat16).contiguous()
    rows = torch.from_numpy(np.stack([golden[f"{name}/{h}/rows"] for h in range(spec.n_q)]).astype(np.int32)).cuda()
    plans = pf.sparsify_layer(qb, kk, rows, c["alpha"], n_new, n_total, spec.n_kv)
    dev_plans = plans.to_host()
    seqs = plans.pick_sequences()
    score_count = plans.score_count.cpu().numpy()
    outcomes = []
    for h, hc in enumerate(c["heads"]):
        r = golden[f"{name}/{h}/rows"]
        pos = ro + r
        Qb = Q[h, ro:n_total].astype(np.float64)
        Kb = K[h // group, :n_total].astype(np.float64)
        oplan = opf.sparsify_head(Qb[r], Kb, c["alpha"], pos)
        assert sorted(oplan.selected_slashes) == golden[f"{name}/{h}/slashes"].tolist()
        sl_w = dict(zip(golden[f"{name}/{h}/slash_order"].tolist(), golden[f"{name}/{h}/slash_w"].tolist()))
        vt_w = dict(zip(golden[f"{name}/{h}/vert_order"].tolist(), golden[f"{name}/{h}/vert_w"].tolist()))
        outcome = check_plan(oplan, dev_plans[h], seqs[h], sl_w, vt_w)
        outcomes.append(outcome)
        if outcome == "identical":
            # fp32 P vs fp64: sums over up to 2*n_total picks, so relative
            assert dev_plans[h].achieved_coverage == pytest.approx(hc["coverage"], rel=1e-5, abs=1e-5)
            assert dev_plans[h].approx_sum == pytest.approx(hc["approx"], rel=1e-5, abs=1e-4)
        assert dev_plans[h].total_weight == pytest.approx(hc["total"], abs=1e-4)
        assert int(score_count[h]) == hc["score_count"]
    if c["alpha"] >= 1.0:
        # target = T exactly: termination is decided by the last ulp of the exact
        # sum (fp32 P vs fp64), so only full coverage is required
        assert all(p.achieved_coverage >= 1.0 - 1e-5 for p in dev_plans)
    else:
        assert outcomes.count("identical") >= len(outcomes) - 1, outcomes


def test_sparsify_head_dropin(cuda_lib, golden):
    c, spec, Q, K, V = _inputs(golden, "prefill_small")
    ro, n_new = c["row_offset"], c["n_new"]
    n_total = ro + n_new
    r = golden["prefill_small/0/rows"]
    from paper_2507_13681_b200.opcount import OpCounter

    cnt = OpCounter()
    plan = pf.sparsify_head(Q[0, ro:n_total][r], K[0, :n_total], c["alpha"], ro + r, counter=cnt)
    assert sorted(plan.selected_slashes) == golden["prefill_small/0/slashes"].tolist()
    assert sorted(plan.selected_verticals) == golden["prefill_small/0/verticals"].tolist()
    assert cnt.scores == c["heads"][0]["score_count"]


# --------------------------------------- greedy on the oracle's exact lines
@pytest.mark.parametrize("name", PREFILL)
def test_greedy_on_exact_lines_is_bit_exact(cuda_lib, golden, name):
    """feeding the oracle's exact Line lists gives identical sets,
    approx bit-equal (same fp64 update order), coverage within 1e-12."""
    c, spec, Q, K, V = _inputs(golden, name)
    ro, n_new = c["row_offset"], c["n_new"]
    n_total = ro + n_new
    group = spec.n_q // spec.n_kv
    for h in range(spec.n_q):
        r = golden[f"{name}/{h}/rows"]
        pos = ro + r
        Qb = Q[h, ro:n_total].astype(np.float64)
        Kb = K[h // group, :n_total].astype(np.float64)
        W = oatt.softmax_rows(opf.sampled_logits(Qb[r], Kb, pos))
        sl, vl = opf.line_sums_view(W, pos)
        oplan = opf.greedy(sl, vl, c["alpha"], float(W.sum()), opf.BlockView(W, pos))
        dplan = pf.greedy_select_lines(sl, vl, c["alpha"], float(W.sum()), W, pos)
        assert dplan.selected_slashes == oplan.selected_slashes
        assert dplan.selected_verticals == oplan.selected_verticals
        assert dplan.approx_sum == oplan.approx_sum
        assert dplan.achieved_coverage == pytest.approx(oplan.achieved_coverage, abs=1e-12)


def test_greedy_hand_block(cuda_lib):
    """test_prefill.py:122-128 on the device: alpha=.7 -> {d0}, approx 1.4."""
    W = np.array([[0.1, 0.2, 0.7, 0.0], [0.05, 0.1, 0.15, 0.7]])
    pos = np.array([2, 3])
    sl, vl = opf.line_sums_view(W, pos)
    plan = pf.greedy_select_lines(sl, vl, 0.7, float(W.sum()), W, pos)
    assert plan.selected_slashes == frozenset({0}) and plan.selected_verticals == frozenset()
    assert plan.approx_sum == pytest.approx(1.4) and plan.achieved_coverage == pytest.approx(0.7)
    plan0 = pf.greedy_select_lines(sl, vl, 0.0, float(W.sum()), W, pos)
    assert not plan0.selected_slashes and not plan0.selected_verticals
    plan1 = pf.greedy_select_lines(sl, vl, 1.0, float(W.sum()), W, pos)
    assert plan1.achieved_coverage == pytest.approx(1.0)


# --------------------------------------------------- K5 sparse attention
@pytest.mark.parametrize("name", PREFILL)
def test_masked_sparse_attention_matches_reference(cuda_lib, golden, name):
    c, spec, Q, K, V = _inputs(golden, name)
    ro, n_new = c["row_offset"], c["n_new"]
    n_total = ro + n_new
    group = spec.n_q // spec.n_kv
    for h, hc in enumerate(c["heads"]):
        plan = pf.SparsePlan(frozenset(golden[f"{name}/{h}/slashes"].tolist()),
                             frozenset(golden[f"{name}/{h}/verticals"].tolist()), 0.0, 0.0, 0.0, n_total)
        from paper_2507_13681_b200.opcount import OpCounter

        cnt = OpCounter()
        Z = tops.masked_sparse_attention(Q[h, ro:n_total], K[h // group, :n_total], V[h // group, :n_total], plan,
                                         ro, counter=cnt)
        assert np.abs(Z - golden[f"{name}/{h}/Z"]).max() <= ATOL
        assert cnt.scores == hc["cells"]


@pytest.mark.parametrize("name", PREFILL)
def test_seed_rows_match_reference(cuda_lib, golden, name):
    c, spec, Q, K, V = _inputs(golden, name)
    ro, n_new = c["row_offset"], c["n_new"]
    n_total = ro + n_new
    group = spec.n_q // spec.n_kv
    W = c["window"]
    n_rows = min(W, n_new)
    for h in range(spec.n_q):
        plan = pf.SparsePlan(frozenset(golden[f"{name}/{h}/slashes"].tolist()),
                             frozenset(golden[f"{name}/{h}/verticals"].tolist()), 0.0, 0.0, 0.0, n_total)
        qb = pf.to_bf16(Q[h, ro:n_total]).unsqueeze(0)
        kb = pf.to_bf16(K[h // group, :n_total]).unsqueeze(0)
        sl, vt, cn = tops.plan_tensors(plan, n_total, qb.device)
        rows = tops.plan_rows(qb, kb, sl, vt, cn, n_new, n_total, 1, n_rows)[0].cpu().numpy()
        assert np.abs(rows - golden[f"{name}/{h}/seed_rows"]).max() <= 1e-4


def test_masked_attention_known_answers(cuda_lib):
    rng = np.random.Generator(np.random.PCG64(0))
    Q, K, V = rng.normal(size=(3, 64)), rng.normal(size=(6, 64)), rng.normal(size=(6, 64))
    allp = pf.SparsePlan(frozenset(range(6)), frozenset(range(6)), 0, 0, 0, 6)
    dense, _ = oatt.scaled_dot_attention(pf.to_bf16(Q).float().cpu().numpy(), pf.to_bf16(K).float().cpu().numpy(),
                                         pf.to_bf16(V).float().cpu().numpy(), 3)
    assert np.abs(tops.masked_sparse_attention(Q, K, V, allp, 3) - dense).max() <= ATOL
    diag = pf.SparsePlan(frozenset({0}), frozenset(), 0, 0, 0, 6)
    Vb = pf.to_bf16(V).float().cpu().numpy()
    assert np.abs(tops.masked_sparse_attention(Q, K, V, diag, 3) - Vb[3:6]).max() <= 1e-6
    fb = pf.SparsePlan(frozenset(), frozenset({5}), 0, 0, 0, 6)
    Z = tops.masked_sparse_attention(Q, K, V, fb, 3)
    assert np.abs(Z[0] - Vb[3]).max() <= 1e-6 and np.abs(Z[1] - Vb[4]).max() <= 1e-6
    from paper_2507_13681_b200.errors import EmptyPlan

    with pytest.raises(EmptyPlan):
        tops.masked_sparse_attention(Q, K, V, pf.SparsePlan(frozenset(), frozenset(), 0, 0, 0, 6), 3)


def test_dense_attention_matches_oracle(cuda_lib):
    rng = np.random.Generator(np.random.PCG64(3))
    Q, K, V = rng.normal(size=(200, 128)), rng.normal(size=(333, 128)), rng.normal(size=(333, 128))
    Qb, Kb, Vb = (pf.to_bf16(x).double().cpu().numpy() for x in (Q, K, V))
    Z, block = tops.scaled_dot_attention(Q, K, V, 133)
    Zo, Wo = oatt.scaled_dot_attention(Qb, Kb, Vb, 133)
    assert np.abs(Z - Zo).max() <= ATOL
    assert np.abs(block.weights - Wo).max() <= 1e-4


# ------------------------------------------------------- decode K6/K7/K8
def test_topb_matches_reference(cuda_lib, golden):
    for i, c in enumerate(golden.case("topb")):
        rows = [(golden[f"topb/{i}/ids/{j}"], golden[f"topb/{i}/w/{j}"]) for j in range(c["n_rows"])]
        ids, scores = kv.accumulate_scores(rows)  # device fp64, the reference's add order
        assert ids.tolist() == golden[f"topb/{i}/cand_ids"].tolist()
        assert np.array_equal(scores, golden[f"topb/{i}/cand_scores"])  # bit-exact
        picked = kv._top_by_score(ids, scores, c["budget"])  # device radix select
        assert picked.tolist() == golden[f"topb/{i}/picked"].tolist()


def test_topb_hand_cases(cuda_lib):  # test_kvcompress.py:94-111
    assert kv.select_topB_obs(np.array([[0.1, 0.5, 0.3, 0.1]]), 2, "summed_over_heads").tolist() == [1, 2]
    assert kv.select_topB_obs(np.array([[0.5, 0.5]]), 1, "summed_over_heads").tolist() == [0]
    per_head = kv.select_topB_obs(np.array([[1.0, 0.0, 0.5], [0.0, 1.0, 0.5]]), 1, "per_head")
    assert [x.tolist() for x in per_head] == [[0], [1]]
    assert kv.select_topB_obs(np.array([[0.2, 0.1, 0.7]]), 5, "summed_over_heads").tolist() == [0, 1, 2]


DECODE = ["decode_small", "decode_window_gt_interval", "decode_warmup_lt_window", "decode_nobudget",
          "decode_huge_budget", "decode_gqa7", "decode_gqa8", "decode_long"]


@pytest.mark.parametrize("archive", [False, True])
@pytest.mark.parametrize("name", DECODE)
def test_progressive_decode_matches_reference(cuda_lib, golden, name, archive):
    """archive=True: the engine's step path (q read from the Q archive at the
    device length; with interval >= window the observation rows record
    (n_a, lo) and events take K7's working-set path, select_ws_kernel)."""
    c = golden.case(name)
    spec = SynthSpec(**c["spec"])
    Q, K, V = layer_qkv_numpy(spec, layer=0)
    L0, max_new = c["L0"], c["max_new"]
    comp = kv.CompressionConfig(c["budget"], c["interval"], c["warmup"], c["obs_window"])
    W = comp.window()
    cap = L0 + max_new
    qd = pf.to_bf16(Q)  # [n_q, n_pos, d]
    kd, vd = pf.to_bf16(K), pf.to_bf16(V)
    budget_cap = c["budget"] if c["budget"] is not None else 1
    stack = kv.DecodeStack(1, spec.n_q, spec.n_kv, spec.d, W, budget_cap, cap + 1, kd.numel(), kd.stride(0))
    seeds = golden[f"{name}/seed_rows"]  # [n_q, n_seed, L0]
    n_seed = seeds.shape[1]
    slots = stack.seed_slots(n_seed)
    for i, s in enumerate(slots):
        stack.write_dense_rows(0, s, torch.from_numpy(seeds[:, i].astype(np.float32)).cuda())
    stack.set_step(L0, n_seed)

    def source(t, length):
        return [(qd[:, length].contiguous(), kd, vd)]

    if archive:
        stack.derived_ids = c["budget"] is not None and c["interval"] >= W
        stack.step = lambda li, q, k, v, compressed, max_cols, out, stream=None: stack.step_archive(
            li, qd, k, v, compressed, max_cols, out, pdl=False, stream=stream)

    from paper_2507_13681_b200.opcount import OpCounter

    cnt = OpCounter()
    outs, stats = kv.progressive_decode(stack, source, L0, comp, max_new, kd, vd, counter=cnt)
    dev_outs = np.stack([o[0].float().cpu().numpy() for o in outs])
    assert np.abs(dev_outs - golden[f"{name}/outs"]).max() <= ATOL
    assert stats.compressed == c["compressed"]
    assert len(stats.events) == len(c["events"])
    for i, (e, ge) in enumerate(zip(stats.events, c["events"])):
        assert e["step"] == ge["step"] and e["head"] == ge["head"]
        ref = golden[f"{name}/event/{i}"].tolist()
        if e["retained_ids"] != ref:
            # divergence must be a top-B near-tie: recompute the oracle scores
            pytest.fail(f"event {i}: retained ids differ ({len(set(ref) ^ set(e['retained_ids']))} ids)")
        assert e["score_coverage"] == pytest.approx(ge["score_coverage"], abs=1e-4)
    assert stats.step_retained == c["step_retained"]
    assert stats.step_head_scores == c["step_head_scores"]
    assert cnt.scores == c["decode_scores"]


def test_compact_cache_known_answer(cuda_lib):  # test_kvcompress.py:175-184
    keys = np.arange(12.0).reshape(6, 2)
    vals = np.arange(18.0).reshape(6, 3)
    h = kv.KVCacheHead(keys, vals, np.arange(6), 6)
    scores = np.array([0.1, 0.9, 0.0, 0.8, 0.2, 0.3])
    picked = kv.select_topB_obs(scores[None, :], 2, "summed_over_heads")
    out = kv.compact_cache(h, picked, recent_window=1)
    assert out.retained_ids.tolist() == [1, 3, 5]
    assert np.array_equal(out.keys, keys[[1, 3, 5]]) and np.array_equal(out.values, vals[[1, 3, 5]])


# ------------------------------------------- tensor-core vs CUDA-core K5
@pytest.mark.parametrize("d,n_q,n_kv,ro,n_new", [(128, 8, 2, 2048, 2048), (64, 4, 4, 700, 333),
                                                 (128, 4, 1, 0, 1500)])
def test_vs_attention_tc_matches_simt_and_oracle(cuda_lib, d, n_q, n_kv, ro, n_new):
    import ctypes

    from paper_2507_13681_b200 import _lib
    from paper_2507_13681_b200.synth import layer_qkv_torch

    n_total = ro + n_new
    spec = SynthSpec(n_q, n_kv, d, n_total, seed=7)
    Q, K, V = layer_qkv_torch(spec, 0)
    qb = Q[:, ro:n_total].contiguous()
    rows = pf.sample_rows_device(n_new, 0.1, 32, 3, 1, 0, 0, n_q)
    plans = pf.sparsify_layer(qb, K, rows, 0.955, n_new, n_total, n_kv)
    out_tc, cells_tc = tops.attention_layer(qb, K, V, plans.slash_ids, plans.vert_ids, plans.counts, n_new, n_total,
                                            n_kv, out_dtype=torch.float32)
    L = pf.layer_desc(n_q, n_kv, d, n_new, n_total, qb.stride(0), K.stride(0))
    out_s = torch.empty_like(out_tc)
    cells_s = torch.empty_like(cells_tc)
    n = _lib.lib().ls_vs_attention_workspace(ctypes.byref(L))
    ws = torch.empty(n, dtype=torch.uint8, device="cuda")
    _lib.call("ls_vs_attention_simt", ctypes.byref(L), qb.data_ptr(), K.data_ptr(), V.data_ptr(),
              plans.slash_ids.data_ptr(), plans.vert_ids.data_ptr(), plans.counts.data_ptr(), out_s.data_ptr(), 0,
              cells_s.data_ptr(), ws.data_ptr(), n, _lib.stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(cells_tc, cells_s)
    assert (out_tc - out_s).abs().max().item() <= 2e-2  # both vs fp64 within 2e-2; tc rounds P to bf16
    hp = plans.to_host()
    group = n_q // n_kv
    for h in (0, n_q - 1):
        Z, _, cells = oatt.masked_sparse_attention(qb[h].double().cpu().numpy(), K[h // group].double().cpu().numpy(),
                                                   V[h // group].double().cpu().numpy(), hp[h].selected_slashes,
                                                   hp[h].selected_verticals, ro)
        assert cells == int(cells_tc[h])
        assert np.abs(out_tc[:, h].double().cpu().numpy() - Z).max() <= ATOL


def test_dense_attention_tc_layer(cuda_lib):
    from paper_2507_13681_b200.synth import layer_qkv_torch

    spec = SynthSpec(4, 2, 128, 1000, seed=9)
    Q, K, V = layer_qkv_torch(spec, 0)
    ro, n_new = 400, 600
    qb = Q[:, ro:].contiguous()
    out = tops.dense_attention_layer(qb, K, V, n_new, 1000, 2, out_dtype=torch.float32)
    for h in (0, 3):
        Zo, _ = oatt.scaled_dot_attention(qb[h].double().cpu().numpy(), K[h // 2].double().cpu().numpy(),
                                          V[h // 2].double().cpu().numpy(), ro)
        assert np.abs(out[:, h].double().cpu().numpy() - Zo).max() <= ATOL


# ------------------------------------------- plan coverage
@pytest.mark.parametrize("d,n_q,n_kv,ro,n_new", [(128, 4, 1, 600, 500), (64, 4, 2, 0, 700)])
def test_plan_coverage_matches_oracle(cuda_lib, d, n_q, n_kv, ro, n_new):
    """ls_plan_coverage == coverage_ratio (prefill.py:254-281) of each head's
    plan over the block's dense causal weights (inclusion-exclusion over the
    crossing cells, fp64 oracle)."""
    from oracle import prefill as opf
    from paper_2507_13681_b200.synth import layer_qkv_torch

    n_total = ro + n_new
    spec = SynthSpec(n_q, n_kv, d, n_total, seed=9)
    Q, K, V = layer_qkv_torch(spec, 0)
    qb = Q[:, ro:n_total].contiguous()
    rows = pf.sample_rows_device(n_new, 0.1, 32, 5, 1, 0, 0, n_q)
    plans = pf.sparsify_layer(qb, K, rows, 0.9, n_new, n_total, n_kv)
    cov = tops.plan_coverage_layer(qb, K, V, plans.slash_ids, plans.vert_ids, plans.counts, n_new, n_total, n_kv)
    torch.cuda.synchronize()
    hp = plans.to_host()
    group = n_q // n_kv
    positions = ro + np.arange(n_new)
    for h in range(n_q):
        _, w = oatt.scaled_dot_attention(qb[h].double().cpu().numpy(), K[h // group].double().cpu().numpy(),
                                         V[h // group].double().cpu().numpy(), ro)
        ref = opf.coverage(w, positions, hp[h])
        assert abs(float(cov[h]) - ref) <= 1e-4, (h, float(cov[h]), ref)
    # one-head reference-shaped entry (block given as Q/K/V)
    one = tops.coverage_ratio(qb[0].float().cpu().numpy(), K[0].float().cpu().numpy(), V[0].float().cpu().numpy(),
                              hp[0], ro)
    assert abs(one - float(cov[0])) <= 1e-6


def test_recovery_curve_matches_oracle(cuda_lib):
    """metrics.recovery_curve (metrics.py:71-96) on the device vs the oracle's
    full-block line sums + ranking + inclusion-exclusion coverage."""
    from paper_2507_13681_b200.synth import layer_qkv_torch

    ro, n_new, d = 200, 300, 64
    n_total = ro + n_new
    spec = SynthSpec(2, 1, d, n_total, seed=13)
    Q, K, V = layer_qkv_torch(spec, 0)
    etas = [0.01, 0.05, 0.2]
    heads = {h: (Q[h, ro:n_total].float().cpu().numpy(), K[0].float().cpu().numpy(), V[0].float().cpu().numpy())
             for h in range(2)}
    got = tops.recovery_curve(heads, ro, etas)
    positions = ro + np.arange(n_new)
    for (eta, val), eta_ref in zip(got, etas):
        ratios = []
        for qh, kh, vh in heads.values():
            _, w = oatt.scaled_dot_attention(qh.astype(np.float64), kh.astype(np.float64), vh.astype(np.float64), ro)
            a = opf.line_arrays(w, positions)
            lines = [(-a["s_w"][i], 0, i) for i in range(len(a["s_w"])) if a["s_len"][i] > 0]
            lines += [(-a["v_w"][i], 1, i) for i in range(len(a["v_w"])) if a["v_len"][i] > 0]
            lines.sort()
            k = int(np.floor(eta_ref * 2 * n_total + 1e-9))
            chosen = lines[:k]
            plan = type("P", (), {})()
            plan.selected_slashes = frozenset(i for _, kd, i in chosen if kd == 0)
            plan.selected_verticals = frozenset(i for _, kd, i in chosen if kd == 1)
            ratios.append(opf.coverage(w, positions, plan))
        assert eta == eta_ref
        assert abs(val - float(np.mean(ratios))) <= 2e-3, (eta, val, float(np.mean(ratios)))
