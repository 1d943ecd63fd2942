"""C1 end-to-end harness (test infrastructure only).

Config C1 of BASELINE.json, exactly the reference toy run:
ModelConfig(1 layer, 8 heads, d_model 512, d_k = d_v = 64, vocab 1000,
max_seq_len 3*1000 + 3*32 + 8), weights seed 0, three 1000-token inputs from
PCG64(123), SessionParams(alpha=0.9, comp=CompressionConfig(budget=256,
interval=16, warmup=16), sample 0.1 / 32, max_new=32), run through the
reference's own `run_turn` (session.py:113-201).

The B200 kernels take bf16 Q/K/V (BASELINE.json north_star: bf16 kernels vs
an fp32/fp64 oracle), so both runs -- the pure reference (golden capture) and
the reference with `dropin.install()` -- round the toy model's per-head Q/K/V
projections (model.py:121-127, `qkv_project`) to bf16; everything else in the
reference stays fp64. The same rounding is what SURVEY.md 8d prescribes for
the synthetic inputs ("the oracle gets the same bf16 values upcast").

The reference is imported from oracle/_ref (its byte-compiled form, built by
oracle/build_ref.py) so this runs on the GPU box, where /root/reference does
not exist.
"""

from __future__ import annotations

import importlib
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden", "c1_run.json")
GOLDEN_OBS = os.path.join(REPO, "tests", "golden", "c1_obswindow.json")  # mode="obswindow" (session.py:204-257)

N_TURNS, INPUT_LEN, MAX_NEW = 3, 1000, 32


def reference_modules():
    """Import the compiled reference (`loopserve.*`) or return None."""
    sys.path.insert(0, REPO)
    from oracle.build_ref import install_import

    if not install_import():
        return None
    names = ("errors", "opcount", "tensor_ops", "prefill", "model", "kvcompress", "session")
    return {n: importlib.import_module(f"loopserve.{n}") for n in names}


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp64 -> fp32 -> bf16 (round to nearest even) -> fp64: the values the
    CUDA path sees after its own fp32 -> bf16 conversion (lossless on these)."""
    f = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    b = f.view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


def install_bf16_projection(model_mod):
    """Round qkv_project's outputs to bf16 (model.py:121-127; forward_extend
    calls it through the module global). Returns an undo callable."""
    orig = model_mod.qkv_project

    def qkv_project_bf16(X, head):
        return tuple(bf16_round(a) for a in orig(X, head))

    model_mod.qkv_project = qkv_project_bf16
    return lambda: setattr(model_mod, "qkv_project", orig)


def c1_inputs(mods, mode: str = "loopserve"):
    m, kv, se = mods["model"], mods["kvcompress"], mods["session"]
    cfg = m.ModelConfig(1, 8, 512, 64, 64, 1000, max_seq_len=N_TURNS * INPUT_LEN + N_TURNS * MAX_NEW + 8)
    weights = m.init_weights(cfg, 0)
    rng = np.random.Generator(np.random.PCG64(123))
    turns = [rng.integers(0, cfg.vocab_size, size=INPUT_LEN).tolist() for _ in range(N_TURNS)]
    params = se.SessionParams(mode=mode, alpha=0.9, comp=kv.CompressionConfig(budget=256, interval=16, warmup=16),
                              sample_rate=0.1, sample_floor=32, max_new=MAX_NEW, seed=0)
    return weights, turns, params


def run_c1(mods, record_argmax: bool = True, capture_sparsifier: list | None = None, mode: str = "loopserve"):
    """Three run_turn calls; returns a JSON-able record of everything the
    parity test compares. record_argmax logs, for every greedy choice, the
    gap between the two largest logits (to classify an answer divergence as
    a near-tie). capture_sparsifier collects (turn, layer, head, Q_s, K, pos)."""
    m, se = mods["model"], mods["session"]
    weights, turns, params = c1_inputs(mods, mode)
    undo = install_bf16_projection(m)
    gaps = []
    orig_argmax = m.argmax_token
    kv_mod = mods["kvcompress"]
    orig_kv_argmax = kv_mod.argmax_token
    orig_se_argmax = se.argmax_token

    def argmax_logged(logits):
        lg = np.asarray(logits, dtype=np.float64)
        top = np.sort(lg)[-2:]
        gaps.append(float(top[1] - top[0]))
        return orig_argmax(logits)

    if record_argmax:
        m.argmax_token = argmax_logged
        kv_mod.argmax_token = argmax_logged
        se.argmax_token = argmax_logged
    orig_sp = se.sparsify_head
    turn_box = [0]
    if capture_sparsifier is not None:
        def sp_capture(Q_s, K_all, alpha, pos, counter=None):
            plan = se_sparsify(Q_s, K_all, alpha, pos, counter=counter)
            capture_sparsifier.append((turn_box[0], np.array(Q_s), np.array(K_all), np.array(pos), plan))
            return plan

        se_sparsify = orig_sp
        se.sparsify_head = sp_capture
    try:
        sess = se.Session(weights, seed=params.seed)
        out = []
        for t, toks in enumerate(turns):
            turn_box[0] = t
            g0 = len(gaps)
            res = se.run_turn(sess, toks, params)
            plans = {}
            for (tt, l, h), p in sess.plans.items():
                if tt == t:
                    plans[f"L{l}H{h}"] = {"slashes": sorted(int(x) for x in p.selected_slashes),
                                          "verticals": sorted(int(x) for x in p.selected_verticals),
                                          "coverage": float(p.achieved_coverage), "approx_sum": float(p.approx_sum),
                                          "total_weight": float(p.total_weight), "n_total": int(p.n_total)}
            out.append({"answer": [int(x) for x in res.answer], "plans": plans,
                        "events": [{"step": int(e["step"]), "head": e["head"],
                                    "retained_ids": [int(g) for g in e["retained_ids"]],
                                    "score_coverage": float(e["score_coverage"])} for e in res.events],
                        "op_counts": {k: int(v) for k, v in res.op_counts.items()},
                        "argmax_gaps": gaps[g0:]})
        return out
    finally:
        undo()
        m.argmax_token = orig_argmax
        kv_mod.argmax_token = orig_kv_argmax
        se.argmax_token = orig_se_argmax
        se.sparsify_head = orig_sp


if __name__ == "__main__":
    import json
    import time

    sys.path.insert(0, REPO)
    from oracle.build_ref import build

    build()
    mods = reference_modules()
    for mode, path in (("loopserve", GOLDEN), ("obswindow", GOLDEN_OBS)):
        if len(sys.argv) > 1 and mode not in sys.argv[1:]:
            continue
        t0 = time.time()
        rec = run_c1(mods, mode=mode)
        meta = {"numpy": np.__version__, "seconds": round(time.time() - t0, 1), "mode": mode,
                "generator": "tests/c1_harness.py (pure reference, bf16-rounded projections)"}
        with open(path, "w") as fh:
            json.dump({"meta": meta, "turns": rec}, fh, separators=(",", ":"))
        print(f"wrote {path} in {meta['seconds']} s:", [(len(r["answer"]), len(r["events"]), r["op_counts"]) for r in rec])
