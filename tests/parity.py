"""Parity helpers: compare CUDA-path plans / selections with the oracle and
classify any divergence as a documented near-tie (index
sets identical except at near-ties, i.e. a decision whose two candidates'
oracle values differ by less than NEAR_TIE_REL relative). Every near-tie
found is appended to TIES; tests/conftest.py writes them to
gpurun_out/near_ties.json at the end of the session."""

from __future__ import annotations

NEAR_TIE_REL = 1e-6

TIES: list = []


def rel_gap(a: float, b: float) -> float:
    den = max(abs(a), abs(b), 1e-300)
    return abs(a - b) / den


def first_divergence(oracle_picks, dev_picks):
    n = min(len(oracle_picks), len(dev_picks))
    for t in range(n):
        if (oracle_picks[t][0], oracle_picks[t][1]) != tuple(dev_picks[t]):
            return t
    return None if len(oracle_picks) == len(dev_picks) else n


def check_plan(oplan, dev_plan, dev_picks, sl_w: dict, vt_w: dict, log: list | None = None, where: str = ""):
    """Assert identical sets, or that the first divergence of the pick
    sequences is a near-tie. Returns 'identical' or 'near-tie'.
    oplan.picks[t] = (kind, index, gain_s, gain_v, approx, exact, target)."""
    same = (oplan.selected_slashes == dev_plan.selected_slashes
            and oplan.selected_verticals == dev_plan.selected_verticals)
    if same:
        return "identical"
    t = first_divergence(oplan.picks, dev_picks)
    assert t is not None, "sets differ but pick sequences agree"
    if t >= len(oplan.picks) or t >= len(dev_picks):
        # one side stopped after t picks: the termination test (approx or exact
        # >= alpha T - eps, prefill.py:195) sits at the target
        if t == 0:
            raise AssertionError("termination divergence before the first pick")
        _, _, _, _, ap, ex, target = oplan.picks[t - 1]
        gap = rel_gap(max(ap, ex), target)
        assert gap < NEAR_TIE_REL, f"termination after pick {t}: max(approx, exact) vs target gap {gap:.3e}"
        rec = ("termination", t, gap)
    else:
        ok, oi, gs, gv = oplan.picks[t][:4]
        dk, di = dev_picks[t]
        if ok != dk:
            gap = rel_gap(gs, gv)
            assert gap < NEAR_TIE_REL, f"pick {t}: kind differs ({ok} vs {dk}) with gain gap {gap:.3e}"
        else:
            w = sl_w if ok == "slash" else vt_w
            gap = rel_gap(w[oi], w[di])
            assert gap < NEAR_TIE_REL, f"pick {t}: {ok} {oi} vs {di}, weight gap {gap:.3e}"
        rec = ("pick", t, gap)
    if log is not None:
        log.append(rec)
    TIES.append({"kind": "plan", "where": where, "record": [str(x) for x in rec]})
    return "near-tie"


def check_topb(ids, scores, picked_ref, picked_dev, budget, where: str = ""):
    """Top-B sets equal, or the symmetric difference lies at the selection
    boundary within NEAR_TIE_REL of the B-th score."""
    a, b = set(int(x) for x in picked_ref), set(int(x) for x in picked_dev)
    if a == b:
        return "identical"
    sc = dict(zip((int(i) for i in ids), (float(s) for s in scores)))
    thr = sorted(sc.values(), reverse=True)[min(budget, len(sc)) - 1]
    gaps = []
    for i in a ^ b:
        gaps.append(rel_gap(sc[i], thr))
        assert gaps[-1] < NEAR_TIE_REL, f"id {i} score {sc[i]} far from threshold {thr}"
    TIES.append({"kind": "topb", "where": where, "ids": sorted(a ^ b), "max_gap": max(gaps)})
    return "near-tie"
