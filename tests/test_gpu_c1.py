"""C1 end to end through the reference's own run_turn with the B200 drop-in
installed ("C1 end-to-end: run run_turn itself"), against the
golden capture of the pure reference (tests/golden/c1_run.json, made by
tests/c1_harness.py). Both sides run the same toy model with bf16-rounded
Q/K/V projections (see c1_harness). Compared per turn: the answer tokens,
every (layer, head) plan, every compression event's retained_ids and
score_coverage, and op_counts. Every divergence must be a documented
near-tie (tests/parity.py); each one is written to
gpurun_out/c1_parity_report.json."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from c1_harness import GOLDEN, GOLDEN_OBS, reference_modules, run_c1
from parity import NEAR_TIE_REL, check_plan

REPORT_DIR = os.environ.get("LS_REPORT_DIR", "gpurun_out")
ARGMAX_TIE = 1e-6  # logit gap (absolute, logits ~O(1)) below which a greedy token flip is a near-tie


def _oracle_classify(q_s, k_all, pos, dev_plan, log):
    """Recompute the oracle plan (with its pick sequence and line weights) and
    the device pick sequence on the captured sparsifier inputs; check_plan
    asserts the divergence is a near-tie."""
    import torch

    from oracle import prefill as opf
    from paper_2507_13681_b200 import prefill as pf

    from oracle.attention import softmax_rows

    oplan = opf.sparsify_head(q_s, k_all, 0.9, pos)
    arr = opf.line_arrays(softmax_rows(opf.sampled_logits(q_s, k_all, pos)), pos)
    sl_w = dict(enumerate(arr["s_w"].tolist()))
    vt_w = dict(enumerate(arr["v_w"].tolist()))
    order = np.argsort(pos, kind="stable")
    p = np.asarray(pos)[order]
    ro = int(p.min())
    n_total = k_all.shape[0]
    n_new = n_total - ro
    block = torch.zeros((1, n_new, k_all.shape[1]), dtype=torch.bfloat16, device="cuda")
    block[0, torch.from_numpy(p - ro).cuda()] = pf.to_bf16(q_s[order])
    plans = pf.sparsify_layer(block, pf.to_bf16(k_all).unsqueeze(0),
                              torch.from_numpy(p - ro).to(torch.int32).cuda().unsqueeze(0), 0.9, n_new, n_total, 1)
    return check_plan(oplan, dev_plan, plans.pick_sequences()[0], sl_w, vt_w, log)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["loopserve", "obswindow"])
def test_c1_run_turn_dropin_matches_reference(cuda_lib, mode):
    """mode="loopserve": sparse prefill + progressive decode; mode="obswindow":
    the reference's observation-window baseline (dense prefill, one shared
    top-B summed over heads, session.py:204-257) through the same drop-in."""
    from paper_2507_13681_b200 import dropin

    mods = reference_modules()
    assert mods is not None, "oracle/_ref is not built (python oracle/build_ref.py in a container with /root/reference)"
    with open(GOLDEN if mode == "loopserve" else GOLDEN_OBS) as fh:
        gold = json.load(fh)["turns"]
    patched = dropin.install({f"loopserve.{k}": v for k, v in mods.items()})
    assert "loopserve.kvcompress.decode_step" in patched and "loopserve.session.sparsify_head" in patched
    captured = []
    try:
        got = run_c1(mods, capture_sparsifier=captured, mode=mode)
    finally:
        dropin.uninstall()
    report = {"mode": mode, "near_tie_rel": NEAR_TIE_REL, "turns": [], "violations": []}
    try:
        _compare(gold, got, captured, report)
    finally:
        os.makedirs(REPORT_DIR, exist_ok=True)
        name = "c1_parity_report.json" if mode == "loopserve" else "c1_obswindow_parity_report.json"
        with open(os.path.join(REPORT_DIR, name), "w") as fh:
            json.dump(report, fh, indent=1)
    assert not report["violations"], report["violations"][:6]


def _compare(gold, got, captured, report):
    diverged = False
    viol = report["violations"]

    def soft(cond, msg):
        if not cond:
            viol.append(msg)

    for t, (g, d) in enumerate(zip(gold, got)):
        rep = {"turn": t, "plans_identical": 0, "plan_near_ties": [], "events_identical": 0, "event_diffs": [],
               "answer_identical": g["answer"] == d["answer"]}
        report["turns"].append(rep)
        # plans (prefill runs before this turn's decode: compare even if the answer diverges later)
        for key, gp in g["plans"].items():
            dp = d["plans"][key]
            same = gp["slashes"] == dp["slashes"] and gp["verticals"] == dp["verticals"]
            if same:
                rep["plans_identical"] += 1
                soft(abs(dp["coverage"] - gp["coverage"]) <= 1e-5, f"turn {t} {key}: coverage {dp['coverage']} vs {gp['coverage']}")
                soft(abs(dp["approx_sum"] - gp["approx_sum"]) <= 1e-5 * abs(gp["approx_sum"]),
                     f"turn {t} {key}: approx_sum {dp['approx_sum']} vs {gp['approx_sum']}")
                soft(abs(dp["total_weight"] - gp["total_weight"]) <= 1e-6 * abs(gp["total_weight"]),
                     f"turn {t} {key}: total_weight")
                continue
            h = int(key.split("H")[1])
            cap = [c for c in captured if c[0] == t][h]
            from types import SimpleNamespace

            dev_plan = SimpleNamespace(selected_slashes=frozenset(dp["slashes"]),
                                       selected_verticals=frozenset(dp["verticals"]))
            log = []
            try:
                _oracle_classify(cap[1], cap[2], cap[3], dev_plan, log)  # asserts near-tie
            except AssertionError as exc:
                viol.append(f"turn {t} {key}: plan differs beyond a near-tie: {exc}")
            rep["plan_near_ties"].append({"head": key, "log": [list(map(str, x)) for x in log],
                                          "sym_diff": len(set(gp["slashes"]) ^ set(dp["slashes"]))
                                          + len(set(gp["verticals"]) ^ set(dp["verticals"]))})
        if not rep["answer_identical"]:
            i = next(j for j, (a, b) in enumerate(zip(g["answer"], d["answer"])) if a != b)
            gap = g["argmax_gaps"][i]
            rep["answer_divergence"] = {"token": i, "reference_logit_gap": gap}
            soft(gap < ARGMAX_TIE, f"turn {t}: answer token {i} differs with reference logit gap {gap:.3e}")
            diverged = True
        # events and op counts (decode happens after the prefill: identical inputs only until a divergence)
        n_ev = len(g["events"]) if rep["answer_identical"] else 0
        for ge, de in list(zip(g["events"], d["events"]))[:n_ev]:
            soft((ge["step"], ge["head"]) == (de["step"], de["head"]), f"turn {t}: event order differs")
            if ge["retained_ids"] == de["retained_ids"]:
                rep["events_identical"] += 1
                # the first event's buffer holds prefill seed rows: the K5 plan-row
                # probabilities (fp32 on the device vs the reference's fp64)
                dc = abs(de["score_coverage"] - ge["score_coverage"])
                rep["max_score_coverage_diff"] = max(rep.get("max_score_coverage_diff", 0.0), dc)
                soft(dc <= 1e-6, f"turn {t} event {ge['step']} {ge['head']}: score_coverage "
                                 f"{de['score_coverage']} vs {ge['score_coverage']}")
            else:
                rep["event_diffs"].append({"step": ge["step"], "head": ge["head"],
                                           "sym_diff": len(set(ge["retained_ids"]) ^ set(de["retained_ids"]))})
                viol.append(f"turn {t} event {ge['step']} {ge['head']}: retained_ids differ")
        rep["op_counts"] = {"reference": g["op_counts"], "b200": d["op_counts"]}
        if rep["answer_identical"] and not rep["plan_near_ties"]:
            soft(d["op_counts"] == g["op_counts"], f"turn {t}: op_counts differ")
        if diverged:
            break
