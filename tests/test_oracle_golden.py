"""Pin the CPU oracle to the reference: golden fixtures produced by running the
reference (tests/golden/make_golden.py) and the hand-computed known answers of
the reference's own tests. CPU only."""

import math

import numpy as np
import pytest

from oracle import attention as oatt
from oracle import kvcompress as okv
from oracle import prefill as opf
from oracle import seeding as oseed
from oracle.session import OpCounter, seed_rows_for_plan
from paper_2507_13681_b200.synth import SynthSpec, checksum, layer_qkv_numpy

# reference pkg/tests/test_prefill.py:29-32
HAND_W = np.array([[0.1, 0.2, 0.7, 0.0], [0.05, 0.1, 0.15, 0.7]])
HAND_POS = np.array([2, 3])


class TestHandBlock:
    def test_line_sums(self):  # test_prefill.py:73-80
        sl, vl = opf.line_sums_view(HAND_W, HAND_POS)
        v = {ln.index: ln.weight for ln in vl}
        s = {ln.index: ln.weight for ln in sl}
        assert v == pytest.approx({0: 0.15, 1: 0.3, 2: 0.85, 3: 0.7})
        assert s == pytest.approx({0: 1.4, 1: 0.35, 2: 0.2, 3: 0.05})
        assert [ln.index for ln in sl] == [0, 1, 2, 3]
        assert [ln.index for ln in vl] == [2, 3, 1, 0]

    def test_lengths(self):  # test_prefill.py:107-109
        sl, vl = opf.line_sums_view(HAND_W, HAND_POS)
        assert {ln.index: ln.length for ln in vl} == {0: 2, 1: 2, 2: 2, 3: 1}
        assert {ln.index: ln.length for ln in sl} == {0: 2, 1: 2, 2: 2, 3: 1}

    def test_greedy_point_seven(self):  # test_prefill.py:122-128
        plan = opf.plan_for_block(HAND_W, 2, 0.7)
        assert plan.selected_slashes == frozenset({0})
        assert plan.selected_verticals == frozenset()
        assert plan.approx_sum == pytest.approx(1.4)
        assert plan.achieved_coverage == pytest.approx(0.7)

    def test_alpha_zero(self):  # test_prefill.py:114-117
        plan = opf.plan_for_block(HAND_W, 2, 0.0)
        assert not plan.selected_slashes and not plan.selected_verticals

    def test_invalid_alpha(self):
        with pytest.raises(opf.InvalidAlpha):
            opf.plan_for_block(HAND_W, 2, 1.5)

    def test_coverage_inclusion_exclusion(self):  # test_prefill.py:157-166
        plan = opf.Plan(frozenset({0}), frozenset({2}), 0.0, 0.0, 2.0, 4)
        assert opf.coverage(HAND_W, HAND_POS, plan) == pytest.approx((0.85 + 1.4 - 0.7) / 2.0)


class TestAttentionKnownAnswers:
    def qkv(self, seed, n_new=3, n_total=6, d=4):  # test_tensor_ops.py:123-128
        rng = np.random.Generator(np.random.PCG64(seed))
        return rng.normal(size=(n_new, d)), rng.normal(size=(n_total, d)), rng.normal(size=(n_total, 2))

    def test_all_lines_equals_dense(self):  # test_tensor_ops.py:130-134
        Q, K, V = self.qkv(0)
        dense, _ = oatt.scaled_dot_attention(Q, K, V, 3)
        Z, _, _ = oatt.masked_sparse_attention(Q, K, V, set(range(6)), set(range(6)), 3)
        assert np.abs(Z - dense).max() <= 1e-12

    def test_diagonal_only(self):  # test_tensor_ops.py:136-140
        Q, K, V = self.qkv(1)
        Z, _, _ = oatt.masked_sparse_attention(Q, K, V, {0}, set(), 3)
        assert np.allclose(Z, V[3:6])

    def test_fallback(self):  # test_tensor_ops.py:160-166
        Q, K, V = self.qkv(4)
        Z, _, cells = oatt.masked_sparse_attention(Q, K, V, set(), {5}, 3)
        assert np.allclose(Z[0], V[3]) and np.allclose(Z[1], V[4])
        assert cells == 3

    def test_empty_plan(self):  # test_tensor_ops.py:155-158
        Q, K, V = self.qkv(3)
        with pytest.raises(oatt.EmptyPlan):
            oatt.masked_sparse_attention(Q, K, V, set(), set(), 3)

    @pytest.mark.parametrize("seed", range(20))
    def test_matches_row_loop(self, seed):  # restated tensor_ops.py:141-183 per-row loop
        rng = np.random.Generator(np.random.PCG64(seed))
        n_new, n_total, d = 5, 11, 4
        Q, K, V = rng.normal(size=(n_new, d)), rng.normal(size=(n_total, d)), rng.normal(size=(n_total, 3))
        S = set(int(x) for x in rng.choice(n_total, size=2, replace=False))
        Vs = set(int(x) for x in rng.choice(n_total, size=2, replace=False))
        Z, W, cells = oatt.masked_sparse_attention(Q, K, V, S, Vs, n_total - n_new, return_weights=True)
        count = 0
        for r in range(n_new):
            cols = oatt.row_columns(S, Vs, n_total - n_new + r)
            count += len(cols)
            sc = (K[cols] @ Q[r]) / math.sqrt(d)
            w = np.exp(sc - sc.max())
            w /= w.sum()
            assert np.abs(Z[r] - w @ V[cols]).max() <= 1e-12
        assert cells == count


class TestSeeds:
    def test_rows_match_reference(self, golden):
        for i, c in enumerate(golden.case("seeds")):
            hs = oseed.head_seed(c["session_seed"], c["turn"], c["layer"], c["head"])
            assert str(hs) == c["head_seed"]
            rows = oseed.sample_rows(c["n_new"], c["rate"], c["floor"], hs)
            assert np.array_equal(rows, golden[f"seeds/{i}/rows"])

    def test_properties(self):  # test_prefill.py:46-69
        rows = oseed.sample_rows(100, 0.1, 32, seed=42)
        assert len(rows) == 32 and 99 in rows and list(rows) == sorted(rows)
        assert list(oseed.sample_rows(10, 1.0, 1, seed=0)) == list(range(10))
        with pytest.raises(oseed.EmptyBlock):
            oseed.sample_rows(0, 0.5, 1, seed=0)


def _prefill_inputs(golden, name):
    c = golden.case(name)
    spec = SynthSpec(**c["spec"])
    Q, K, V = layer_qkv_numpy(spec, layer=0)
    assert checksum(Q, K, V) == c["checksum"], "synthetic input regeneration drifted"
    return c, spec, Q, K, V


PREFILL = ["prefill_small", "prefill_d128", "prefill_random", "prefill_alpha1", "prefill_first_turn"]


@pytest.mark.parametrize("name", PREFILL)
def test_prefill_oracle_matches_reference(golden, name):
    c, spec, Q, K, V = _prefill_inputs(golden, name)
    ro, n_new = c["row_offset"], c["n_new"]
    n_total = ro + n_new
    group = spec.n_q // spec.n_kv
    for h, hc in enumerate(c["heads"]):
        kv = h // group
        Qb = Q[h, ro:n_total].astype(np.float64)
        Kb = K[kv, :n_total].astype(np.float64)
        Vb = V[kv, :n_total].astype(np.float64)
        rows = oseed.turn_rows(n_new, c["alpha"], c["rate"], c["floor"], c["session_seed"],
                               c["turn"], c["layer"], h)
        p = f"{name}/{h}"
        assert np.array_equal(rows, golden[p + "/rows"])
        pos = ro + rows
        cnt = OpCounter()
        plan = opf.sparsify_head(Qb[rows], Kb, c["alpha"], pos, counter=cnt)
        assert sorted(plan.selected_slashes) == golden[p + "/slashes"].tolist()
        assert sorted(plan.selected_verticals) == golden[p + "/verticals"].tolist()
        assert plan.achieved_coverage == pytest.approx(hc["coverage"], abs=1e-12)
        assert plan.approx_sum == pytest.approx(hc["approx"], abs=1e-12)
        assert plan.total_weight == pytest.approx(hc["total"], abs=1e-12)
        assert cnt.scores == hc["score_count"]
        # sorted line lists (order and sums) -- bit-identical restatement
        W = oatt.softmax_rows(opf.sampled_logits(Qb[rows], Kb, pos))
        sl, vl = opf.line_sums_view(W, pos)
        assert [ln.index for ln in sl] == golden[p + "/slash_order"].tolist()
        assert [ln.index for ln in vl] == golden[p + "/vert_order"].tolist()
        assert np.abs(np.array([ln.weight for ln in sl]) - golden[p + "/slash_w"]).max() <= 1e-13
        assert np.abs(np.array([ln.weight for ln in vl]) - golden[p + "/vert_w"]).max() <= 1e-13
        Z, _, cells = oatt.masked_sparse_attention(Qb, Kb, Vb, plan.selected_slashes,
                                                   plan.selected_verticals, ro)
        assert np.abs(Z - golden[p + "/Z"]).max() <= 1e-12
        assert cells == hc["cells"]
        seeds = seed_rows_for_plan(Qb, Kb, plan.selected_slashes, plan.selected_verticals,
                                   ro, c["window"])
        assert np.abs(np.stack([w for _, w in seeds]) - golden[p + "/seed_rows"]).max() <= 1e-12


DECODE = ["decode_small", "decode_window_gt_interval", "decode_warmup_lt_window",
          "decode_nobudget", "decode_huge_budget", "decode_gqa7", "decode_gqa8", "decode_long"]


@pytest.mark.parametrize("name", DECODE)
def test_decode_oracle_matches_reference(golden, name):
    c = golden.case(name)
    spec = SynthSpec(**c["spec"])
    Q, K, V = layer_qkv_numpy(spec, layer=0)
    assert checksum(Q, K, V) == c["checksum"]
    group = spec.n_q // spec.n_kv
    L0, max_new = c["L0"], c["max_new"]
    seeds = golden[f"{name}/seed_rows"]
    obs_seed = [[(np.arange(L0), seeds[h, r]) for r in range(seeds.shape[1])] for h in range(spec.n_q)]
    comp = okv.CompressionConfig(c["budget"], c["interval"], c["warmup"], c["obs_window"])
    q_steps = np.stack([Q[:, L0 + t].astype(np.float64) for t in range(max_new)])
    cnt = OpCounter()
    outs, stats = okv.progressive_decode_attn(K.astype(np.float64), V.astype(np.float64),
                                              [h // group for h in range(spec.n_q)], L0, obs_seed,
                                              comp, max_new, q_steps, counter=cnt)
    assert np.abs(outs - golden[f"{name}/outs"]).max() <= 1e-12
    assert len(stats.events) == len(c["events"])
    for i, (e, ge) in enumerate(zip(stats.events, c["events"])):
        assert e["step"] == ge["step"] and f"L0H{e['head']}" == ge["head"]
        assert e["retained_ids"] == golden[f"{name}/event/{i}"].tolist()
        assert e["score_coverage"] == pytest.approx(ge["score_coverage"], abs=1e-12)
    assert stats.step_retained == c["step_retained"]
    assert stats.step_head_scores == c["step_head_scores"]
    assert stats.compressed == c["compressed"]
    assert cnt.scores == c["decode_scores"]


def test_topb_oracle_matches_reference(golden):
    for i, c in enumerate(golden.case("topb")):
        rows = [(golden[f"topb/{i}/ids/{j}"], golden[f"topb/{i}/w/{j}"]) for j in range(c["n_rows"])]
        ids, scores = okv.accumulate_scores(rows)
        assert ids.tolist() == golden[f"topb/{i}/cand_ids"].tolist()
        assert np.array_equal(scores, golden[f"topb/{i}/cand_scores"])  # same fp64 order
        picked = okv.top_by_score(ids, scores, c["budget"])
        assert picked.tolist() == golden[f"topb/{i}/picked"].tolist()
        keep = okv.retained_union(picked, c["window"], c["full_len"])
        assert keep.tolist() == golden[f"topb/{i}/keep"].tolist()


class TestKVKnownAnswers:
    def test_accumulate_aligns_by_id(self):  # test_kvcompress.py:83-90
        rows = [(np.array([0, 1, 5]), np.array([0.1, 0.2, 0.7])),
                (np.array([1, 5, 6]), np.array([0.3, 0.3, 0.4]))]
        ids, scores = okv.accumulate_scores(rows)
        assert ids.tolist() == [0, 1, 5, 6]
        assert np.allclose(scores, [0.1, 0.5, 1.0, 0.4])

    def test_topb_cases(self):  # test_kvcompress.py:94-111
        assert okv.select_topB_obs(np.array([[0.1, 0.5, 0.3, 0.1]]), 2, "summed_over_heads").tolist() == [1, 2]
        assert okv.select_topB_obs(np.array([[0.5, 0.5]]), 1, "summed_over_heads").tolist() == [0]
        per_head = okv.select_topB_obs(np.array([[1.0, 0.0, 0.5], [0.0, 1.0, 0.5]]), 1, "per_head")
        assert [x.tolist() for x in per_head] == [[0], [1]]

    def test_compaction(self):  # test_kvcompress.py:175-184
        keys = np.arange(12.0).reshape(6, 2)
        vals = np.arange(18.0).reshape(6, 3)
        scores = np.array([0.1, 0.9, 0.0, 0.8, 0.2, 0.3])
        picked = okv.select_topB_obs(scores[None, :], 2, "summed_over_heads")
        k, v, keep = okv.compact_cache(keys, vals, np.arange(6), 6, picked, 1)
        assert keep.tolist() == [1, 3, 5]
        assert np.array_equal(k, keys[[1, 3, 5]]) and np.array_equal(v, vals[[1, 3, 5]])

    def test_missing_rows(self):  # test_kvcompress.py:186-190
        with pytest.raises(okv.InvalidIds):
            okv.compact_cache(np.zeros((2, 2)), np.zeros((2, 2)), np.array([4, 5]), 6, np.array([0]), 1)

    def test_config(self):  # test_kvcompress.py:258-262
        with pytest.raises(okv.InvalidConfig):
            okv.CompressionConfig(budget=0).validate()
        with pytest.raises(okv.InvalidConfig):
            okv.CompressionConfig(interval=0).validate()
