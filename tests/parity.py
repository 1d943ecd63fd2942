"""Parity helpers: compare CUDA-path plans / selections with the oracle and
classify any divergence as a documented near-tie (index
sets identical except at near-ties, i.e. a decision whose two candidates'
oracle values differ by less than NEAR_TIE_REL relative)."""

from __future__ import annotations

import numpy as np

NEAR_TIE_REL = 1e-4  # fp32 P (bf16 inputs, fp32 exp/accumulate) vs the fp64 oracle


def rel_gap(a: float, b: float) -> float:
    den = max(abs(a), abs(b), 1e-300)
    return abs(a - b) / den


def first_divergence(oracle_picks, dev_picks):
    n = min(len(oracle_picks), len(dev_picks))
    for t in range(n):
        if (oracle_picks[t][0], oracle_picks[t][1]) != tuple(dev_picks[t]):
            return t
    return None if len(oracle_picks) == len(dev_picks) else n


def check_plan(oplan, dev_plan, dev_picks, sl_w: dict, vt_w: dict, log: list | None = None):
    """Assert identical sets, or that the first divergence of the pick
    sequences is a near-tie. Returns 'identical' or 'near-tie'."""
    same = (oplan.selected_slashes == dev_plan.selected_slashes
            and oplan.selected_verticals == dev_plan.selected_verticals)
    if same:
        return "identical"
    t = first_divergence(oplan.picks, dev_picks)
    assert t is not None, "sets differ but pick sequences agree"
    if t >= len(oplan.picks) or t >= len(dev_picks):
        # one side stopped earlier: termination near the target (exact vs alpha*T)
        if log is not None:
            log.append(("termination", t))
        return "near-tie"
    ok, gk, gi, gs, gv = oplan.picks[t]
    dk, di = dev_picks[t]
    if ok != dk:
        gap = rel_gap(gs, gv)
        assert gap < NEAR_TIE_REL, f"pick {t}: kind differs ({ok} vs {dk}) with gain gap {gap:.3e}"
    else:
        w = sl_w if ok == "slash" else vt_w
        gap = rel_gap(w[gi], w[di])
        assert gap < NEAR_TIE_REL, f"pick {t}: {ok} {gi} vs {di}, weight gap {gap:.3e}"
    if log is not None:
        log.append(("pick", t, gap))
    return "near-tie"


def check_topb(ids, scores, picked_ref, picked_dev, budget):
    """Top-B sets equal, or the symmetric difference lies at the selection
    boundary within NEAR_TIE_REL of the B-th score."""
    a, b = set(int(x) for x in picked_ref), set(int(x) for x in picked_dev)
    if a == b:
        return "identical"
    sc = dict(zip((int(i) for i in ids), (float(s) for s in scores)))
    thr = sorted(sc.values(), reverse=True)[min(budget, len(sc)) - 1]
    for i in a ^ b:
        assert rel_gap(sc[i], thr) < NEAR_TIE_REL, f"id {i} score {sc[i]} far from threshold {thr}"
    return "near-tie"
