"""Generate golden parity fixtures by running the REFERENCE implementation.

Run in the build container only (it imports the read-only reference from
/root/reference/pkg/src); the outputs (golden.npz + golden.json) are
committed and travel to the GPU box, the reference does not:

    python tests/golden/make_golden.py

Inputs are regenerated in the tests from `paper_2507_13681_b200.synth`
(numpy PCG64, bf16-rounded); their checksums are stored so a test fails
loudly if regeneration ever differs. Everything the reference is fed is the
bf16 value upcast to fp64, exactly what the CUDA path sees.

Cases (reference call sites in parentheses):
  seeds     -- Session.head_seed + sample_rows      (session.py:84-86, prefill.py:125-135)
  prefill_* -- sparsify_head, _line_sums order, masked_sparse_attention with
               counter, observation seeds             (prefill.py:363, 138; tensor_ops.py:141;
                                                        session.py:89-95)
  decode_*  -- progressive_decode itself with decode_step replaced by an
               attention-only step over synthetic q/k/v (kvcompress.py:167-240;
               the replacement follows model.py:232-241)
  topb      -- accumulate_scores + _top_by_score + retained_union on random rows
"""

from __future__ import annotations

import json
import os
import sys
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import loopserve.kvcompress as ref_kv  # noqa: E402
from loopserve.opcount import OpCounter  # noqa: E402
from loopserve.prefill import _BlockView, _line_sums, sample_rows, sparsify_head  # noqa: E402
from loopserve.session import Session, _obs_seed_from_blocks  # noqa: E402
from loopserve.tensor_ops import masked_sparse_attention  # noqa: E402

from paper_2507_13681_b200.synth import SynthSpec, checksum, layer_qkv_numpy  # noqa: E402

OUT: dict[str, np.ndarray] = {}
META: dict = {"numpy": np.__version__, "reference": "/root/reference/pkg/src/loopserve",
              "cases": {}}


def put(name, arr):
    OUT[name] = np.asarray(arr)


def head_seed(seed, turn, layer, head):
    return Session(_Dummy(), seed=seed).head_seed(turn, layer, head)


class _Dummy:
    class config:  # noqa: N801 - Session only stores the object
        n_layers = n_heads = d_model = d_k = d_v = vocab_size = max_seq_len = 1


def make_seeds():
    cases = []
    # (session_seed, turn, layer, head, n_new, rate, floor)
    grid = [(0, 0, 0, 0, 1000, 0.1, 32), (0, 1, 0, 7, 1032, 0.1, 32), (0, 2, 0, 3, 1032, 0.1, 32),
            (0, 0, 31, 31, 5000, 0.1, 32), (0, 2, 5, 17, 5128, 0.1, 32), (7, 3, 2, 1, 8448, 0.1, 32),
            (0, 9, 79, 63, 10128, 0.1, 32), (3, 9, 0, 0, 10128, 0.1, 32), (1, 0, 0, 0, 1, 0.1, 32),
            (1, 0, 0, 1, 2, 0.1, 32), (1, 0, 0, 2, 31, 0.1, 32), (1, 0, 0, 3, 33, 0.1, 32),
            (1, 0, 0, 4, 100, 0.25, 8), (2, 4, 4, 4, 600, 0.5, 1), (2 ** 40 + 5, 1, 2, 3, 777, 0.1, 32),
            (0, 0, 0, 0, 20000, 0.1, 32), (0, 0, 0, 1, 12000, 0.01, 32)]
    for i, (s, t, l, h, n, rate, floor) in enumerate(grid):
        hs = head_seed(s, t, l, h)
        rows = sample_rows(n, rate, floor, hs)
        put(f"seeds/{i}/rows", rows.astype(np.int64))
        cases.append(dict(session_seed=s, turn=t, layer=l, head=h, n_new=n, rate=rate,
                          floor=floor, head_seed=str(hs)))
    META["cases"]["seeds"] = cases


PREFILL_CASES = [
    # name, spec kwargs, row_offset, n_new, alpha, rate, floor, window
    ("prefill_small", dict(n_q=4, n_kv=2, d=64, n_pos=384, seed=11), 256, 128, 0.9, 0.1, 32, 16),
    ("prefill_d128", dict(n_q=4, n_kv=1, d=128, n_pos=700, seed=12), 400, 300, 0.955, 0.1, 32, 16),
    ("prefill_random", dict(n_q=2, n_kv=2, d=64, n_pos=200, seed=13, structured=False), 100, 100, 0.5, 0.2, 16, 8),
    ("prefill_alpha1", dict(n_q=2, n_kv=1, d=64, n_pos=96, seed=14), 48, 48, 1.0, 0.1, 32, 4),
    ("prefill_first_turn", dict(n_q=2, n_kv=1, d=64, n_pos=256, seed=15), 0, 256, 0.9, 0.1, 32, 16),
]


def make_prefill():
    for name, skw, row_offset, n_new, alpha, rate, floor, window in PREFILL_CASES:
        spec = SynthSpec(**skw)
        Q, K, V = layer_qkv_numpy(spec, layer=0)
        n_total = row_offset + n_new
        group = spec.n_q // spec.n_kv
        info = dict(spec=skw, row_offset=row_offset, n_new=n_new, alpha=alpha, rate=rate,
                    floor=floor, window=window, session_seed=5, turn=1, layer=0,
                    checksum=checksum(Q, K, V), heads=[])
        for h in range(spec.n_q):
            kv = h // group
            Qb = Q[h, row_offset:n_total].astype(np.float64)
            Kb = K[kv, :n_total].astype(np.float64)
            Vb = V[kv, :n_total].astype(np.float64)
            positions = row_offset + np.arange(n_new)
            if alpha >= 1.0:
                rows = np.arange(n_new)
            else:
                rows = sample_rows(n_new, rate, floor, head_seed(5, 1, 0, h))
            c1 = OpCounter()
            plan = sparsify_head(Qb[rows], Kb, alpha, positions[rows], counter=c1)
            # line-sum order of the sampled block (pins the sort keys)
            import math as _m
            logits = np.full((len(rows), n_total), -np.inf)
            for r, g in enumerate(positions[rows]):
                logits[r, :g + 1] = (Kb[:g + 1] @ Qb[rows][r]) / _m.sqrt(spec.d)
            from loopserve.tensor_ops import softmax_rows
            wts = softmax_rows(logits)
            sl, vl = _line_sums(_BlockView(wts, positions[rows]))
            c2 = OpCounter()
            Z, block = masked_sparse_attention(Qb, Kb, Vb, plan, row_offset, counter=c2,
                                               return_weights=True)
            seed_rows = _obs_seed_from_blocks({(0, h): block}, window)[(0, h)]
            p = f"{name}/{h}"
            put(p + "/rows", rows.astype(np.int64))
            put(p + "/slashes", np.array(sorted(plan.selected_slashes), dtype=np.int64))
            put(p + "/verticals", np.array(sorted(plan.selected_verticals), dtype=np.int64))
            put(p + "/slash_order", np.array([ln.index for ln in sl], dtype=np.int64))
            put(p + "/slash_w", np.array([ln.weight for ln in sl]))
            put(p + "/vert_order", np.array([ln.index for ln in vl], dtype=np.int64))
            put(p + "/vert_w", np.array([ln.weight for ln in vl]))
            put(p + "/Z", Z)
            put(p + "/seed_rows", np.stack([w for _, w in seed_rows]))
            info["heads"].append(dict(coverage=plan.achieved_coverage, approx=plan.approx_sum,
                                      total=plan.total_weight, score_count=c1.scores,
                                      cells=c2.scores))
        META["cases"][name] = info


DECODE_CASES = [
    # name, spec, L0, max_new, budget, interval, warmup, obs_window, n_seed_rows
    ("decode_small", dict(n_q=4, n_kv=2, d=64, n_pos=200 + 40, seed=21), 200, 40, 24, 8, 8, None, 8),
    ("decode_window_gt_interval", dict(n_q=2, n_kv=1, d=64, n_pos=150 + 33, seed=22), 150, 33, 16, 5, 7, 9, 9),
    ("decode_warmup_lt_window", dict(n_q=2, n_kv=2, d=128, n_pos=300 + 30, seed=23), 300, 30, 40, 6, 3, 12, 12),
    ("decode_nobudget", dict(n_q=2, n_kv=1, d=64, n_pos=64 + 20, seed=24), 64, 20, None, 4, 4, None, 4),
    ("decode_huge_budget", dict(n_q=2, n_kv=1, d=64, n_pos=64 + 20, seed=25), 64, 20, 10_000, 4, 4, None, 4),
    # GQA groups 7 (Qwen2.5-7B) and 8 (Llama-70B) and a longer cache (several tiles per split)
    ("decode_gqa7", dict(n_q=7, n_kv=1, d=128, n_pos=400 + 40, seed=26), 400, 40, 64, 8, 8, None, 8),
    ("decode_gqa8", dict(n_q=8, n_kv=1, d=128, n_pos=700 + 48, seed=27), 700, 48, 96, 16, 16, None, 16),
    ("decode_long", dict(n_q=4, n_kv=1, d=128, n_pos=1500 + 40, seed=28), 1500, 40, 300, 8, 8, None, 8),
]


def make_decode():
    for name, skw, L0, max_new, budget, interval, warmup, obs_window, n_seed in DECODE_CASES:
        spec = SynthSpec(**skw)
        Q, K, V = layer_qkv_numpy(spec, layer=0)
        group = spec.n_q // spec.n_kv
        comp = ref_kv.CompressionConfig(budget=budget, interval=interval, warmup=warmup,
                                        obs_window=obs_window)
        # seed rows: dense causal softmax rows of the last n_seed prefill positions
        rng = np.random.Generator(np.random.PCG64(99))
        obs_seed = {}
        seed_store = []
        for h in range(spec.n_q):
            rows = []
            for r in range(n_seed):
                g = L0 - n_seed + r
                w = np.zeros(L0)
                raw = rng.random(g + 1) ** 3
                w[:g + 1] = raw / raw.sum()
                rows.append((np.arange(L0), w))
            obs_seed[(0, h)] = rows
            seed_store.append(np.stack([w for _, w in rows]))
        kk = K.astype(np.float64)
        vv = V.astype(np.float64)
        qq = Q.astype(np.float64)
        outs = np.zeros((max_new, spec.n_q, spec.d))

        cache = SimpleNamespace(length=L0)

        def fake_decode_step(weights, cache, last_token, working_sets=None, counter=None):
            pos = cache.length
            t = pos - L0
            obs = {}
            for (l, h), ws in working_sets.items():
                kv = h // group
                cols = np.append(np.asarray(ws, dtype=np.intp), pos)
                scores = (kk[kv][cols] @ qq[h][pos]) / np.sqrt(spec.d)
                if counter is not None:
                    counter.add(len(cols))
                w = np.exp(scores - scores.max())
                w /= w.sum()
                outs[t, h] = w @ vv[kv][cols]
                obs[(l, h)] = (cols, w)
            cache.length = pos + 1
            return None, 0, obs

        weights = SimpleNamespace(config=SimpleNamespace(n_layers=1, n_heads=spec.n_q))
        state = ref_kv.DecodeState(cache=cache, first_logits=np.zeros(3), obs_seed=obs_seed)
        orig = ref_kv.decode_step
        ref_kv.decode_step = fake_decode_step
        try:
            counter = OpCounter()
            answer, stats = ref_kv.progressive_decode(weights, state, comp, max_new, counter=counter)
        finally:
            ref_kv.decode_step = orig
        assert len(answer) == max_new and cache.length == L0 + max_new
        put(f"{name}/outs", outs)
        put(f"{name}/seed_rows", np.stack(seed_store))
        ev = []
        for i, e in enumerate(stats.events):
            put(f"{name}/event/{i}", np.array(e["retained_ids"], dtype=np.int64))
            ev.append(dict(step=e["step"], head=e["head"], score_coverage=e["score_coverage"]))
        META["cases"][name] = dict(spec=skw, L0=L0, max_new=max_new, budget=budget,
                                   interval=interval, warmup=warmup, obs_window=obs_window,
                                   n_seed=n_seed, checksum=checksum(Q, K, V), events=ev,
                                   step_retained=stats.step_retained,
                                   step_head_scores=stats.step_head_scores,
                                   compressed=stats.compressed, decode_scores=counter.scores)


def make_topb():
    rng = np.random.Generator(np.random.PCG64(7))
    cases = []
    for i in range(12):
        n_rows = int(rng.integers(1, 6))
        rows = []
        for _ in range(n_rows):
            ids = np.sort(rng.choice(300, size=int(rng.integers(1, 120)), replace=False))
            w = np.round(rng.random(len(ids)), 2 if i % 2 else 6)  # rounding provokes ties
            rows.append((ids, w))
            put(f"topb/{i}/ids/{len(rows) - 1}", ids.astype(np.int64))
            put(f"topb/{i}/w/{len(rows) - 1}", w)
        budget = int(rng.integers(1, 80))
        window = int(rng.integers(1, 10))
        ids, scores = ref_kv.accumulate_scores(rows)
        picked = ref_kv._top_by_score(ids, scores, budget)
        keep = ref_kv.retained_union(picked, window, 320)
        put(f"topb/{i}/cand_ids", ids.astype(np.int64))
        put(f"topb/{i}/cand_scores", scores)
        put(f"topb/{i}/picked", picked.astype(np.int64))
        put(f"topb/{i}/keep", keep.astype(np.int64))
        cases.append(dict(n_rows=n_rows, budget=budget, window=window, full_len=320))
    META["cases"]["topb"] = cases


if __name__ == "__main__":
    make_seeds()
    make_topb()
    make_prefill()
    make_decode()
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **OUT)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(META, fh, indent=1, sort_keys=True)
    print("wrote", len(OUT), "arrays")
