"""Session batching (config C4, cli.py:213-226 instance parallelism): S
independent dialogue sessions stacked along the head axis of ONE engine (every
launch covers all sessions) must give each session exactly what running it
alone gives: sampled rows, plans, prefill outputs, decode outputs and the
compression events' retained ids. Prefill is bit for bit; decode splits the
key range of each head by the number of KV heads in the launch (more units,
fewer splits), so its outputs agree to rounding and the retained sets except
at score near-ties."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_batched_sessions_equal_single_sessions(cuda_lib):
    from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
    from paper_2507_13681_b200.kvcompress import CompressionConfig

    S, Hs, KVs, L, d = 2, 4, 2, 2, 128
    max_new = 24
    blocks = [(0, 1200), (1200, 1224)]  # turn 2's block = turn 1's answer (24) + 1200 new tokens
    cap = blocks[-1][0] + blocks[-1][1] + max_new
    comp = CompressionConfig(budget=128, interval=8, warmup=8)
    seeds = [7, 11]
    big = AttnShape(L, S * Hs, S * KVs, d)
    store = QKVStore.synthetic(big, cap, n_ref=cap, seed=3)
    eng = SessionEngine(big, SessionParams(alpha=0.9, comp=comp, max_new=max_new), cap, session_seeds=seeds)
    one = AttnShape(L, Hs, KVs, d)
    singles = []
    for s, sd in enumerate(seeds):
        st = QKVStore(one, cap)
        st.q.copy_(store.q[:, s * Hs:(s + 1) * Hs])
        st.k.copy_(store.k[:, s * KVs:(s + 1) * KVs])
        st.v.copy_(store.v[:, s * KVs:(s + 1) * KVs])
        st.length = store.length
        singles.append((st, SessionEngine(one, SessionParams(alpha=0.9, comp=comp, max_new=max_new, seed=sd), cap)))
    for t, (ro, n_new) in enumerate(blocks):
        rb = eng.prefill(store, t, ro, n_new)
        outs_b, ev_b = [], []
        eng.decode(store, ro + n_new, max_new, out_sink=lambda k, ob: outs_b.append(ob.float().cpu().numpy().copy()),
                   events=ev_b)
        torch.cuda.synchronize()
        for s, (st, e1) in enumerate(singles):
            r1 = e1.prefill(st, t, ro, n_new)
            outs_1, ev_1 = [], []
            e1.decode(st, ro + n_new, max_new, out_sink=lambda k, ob: outs_1.append(ob.float().cpu().numpy().copy()),
                      events=ev_1)
            torch.cuda.synchronize()
            hs = slice(s * Hs, (s + 1) * Hs)
            assert torch.equal(rb.rows[:, hs], r1.rows), (t, s, "sampled rows")
            for l in range(L):
                pb, p1 = rb.plans[l], r1.plans[l]
                assert torch.equal(pb.counts[hs], p1.counts), (t, s, l, "plan sizes")
                cn = p1.counts.cpu().numpy()
                for j in range(Hs):  # the id lists up to each head's counts (the tails are scratch)
                    assert torch.equal(pb.slash_ids[s * Hs + j, :cn[j, 0]], p1.slash_ids[j, :cn[j, 0]])
                    assert torch.equal(pb.vert_ids[s * Hs + j, :cn[j, 1]], p1.vert_ids[j, :cn[j, 1]])
                assert torch.equal(rb.out[l][:, hs], r1.out[l]), (t, s, l, "prefill output")
            np.testing.assert_allclose(np.stack(outs_b)[:, :, hs], np.stack(outs_1), rtol=0, atol=5e-3)
            assert len(ev_b) == len(ev_1) > 0
            for eb, e_1 in zip(ev_b, ev_1):
                if "n_sel" not in eb:
                    continue
                nb = eb["n_sel"].view(L, S * Hs)[:, hs].reshape(-1)
                assert torch.equal(nb, e_1["n_sel"].reshape(-1)), (t, s, "retained counts")
                sb = eb["sel"].view(L, S * Hs, -1)[:, hs].reshape(L * Hs, -1).cpu().numpy()
                s1 = e_1["sel"].view(L * Hs, -1).cpu().numpy()
                for row in range(L * Hs):
                    n = int(nb[row])
                    common = len(set(sb[row, :n].tolist()) & set(s1[row, :n].tolist()))
                    assert common >= n - max(1, n // 100), (t, s, row, n, common, "retained ids")
