"""KV-head-group sharding on one GPU: every rank of a W-way
HeadShard run one after the other must reproduce the unsharded run's heads --
plans and prefill outputs bit for bit (every kernel is per head and K1's
cross-CTA merges are chunk-aligned integer sums, so the launch's head count
does not change any value), compression events identical, decode outputs
within rounding (K6's split count follows the number of units per launch)."""

import numpy as np
import pytest
import torch

from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
from paper_2507_13681_b200.kvcompress import CompressionConfig
from paper_2507_13681_b200.parallel import HeadShard

pytestmark = pytest.mark.gpu

L, NQ, NKV, D = 2, 8, 4, 128
INPUT, MAX_NEW, TURNS = 1500, 40, 2


def _run(shape, kv_offset, q_offset, cap):
    store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=5, kv_offset=kv_offset)
    params = SessionParams(alpha=0.95, comp=CompressionConfig(256, 16, 16), max_new=MAX_NEW, seed=9)
    eng = SessionEngine(shape, params, cap)
    out = []
    for t, (ro, n_new) in enumerate(eng.turn_blocks(INPUT, TURNS, MAX_NEW)):
        res = eng.prefill(store, t, ro, n_new, turn_offset_heads=q_offset)
        steps, events = [], []
        eng.decode(store, ro + n_new, MAX_NEW, events=events,
                   run_sink=lambda s0, o: steps.append(o.float().cpu().clone()))
        torch.cuda.synchronize()
        out.append(dict(plans=[res.plans[l].to_host() for l in range(L)],
                        outs=[res.out[l].float().cpu() for l in range(L)],
                        events=eng.event_log(events, head_offset=q_offset),
                        dec=torch.cat(steps)))
    return out


@pytest.mark.parametrize("world", [2, 4])
def test_head_sharded_ranks_equal_unsharded(cuda_lib, world):
    cap = TURNS * (INPUT + MAX_NEW)
    full = _run(AttnShape(L, NQ, NKV, D), 0, 0, cap)
    for rank in range(world):
        sh = HeadShard(NQ, NKV, world, rank)
        part = _run(AttnShape(L, sh.n_q_local, sh.n_kv_local, D), sh.kv_begin, sh.q_begin, cap)
        hq = list(sh.q_heads())
        for t in range(TURNS):
            f, p = full[t], part[t]
            for l in range(L):
                for j, h in enumerate(hq):
                    a, b = f["plans"][l][h], p["plans"][l][j]
                    assert a.selected_slashes == b.selected_slashes and a.selected_verticals == b.selected_verticals
                    assert a.approx_sum == b.approx_sum and a.achieved_coverage == b.achieved_coverage
                assert torch.equal(f["outs"][l][:, hq], p["outs"][l]), (t, l)
            fe = [e for e in f["events"] if int(e["head"].split("H")[1]) in hq]
            pe = p["events"]
            assert [(e["step"], e["head"]) for e in fe] == [(e["step"], e["head"]) for e in pe]
            for a, b in zip(fe, pe):
                assert a["retained_ids"] == b["retained_ids"], (t, a["step"], a["head"])
            err = (f["dec"][:, :, hq] - p["dec"]).abs().max().item()
            assert err < 2e-2, err
