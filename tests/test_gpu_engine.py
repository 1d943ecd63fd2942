"""Engine decode paths agree with the oracle-checked per-step path.

The production decode (SessionEngine.decode: CUDA graphs, q read from the Q
archive at the device cache length, layers chained by programmatic dependent
launch) must produce exactly the outputs of the plain per-step path
(DecodeStack.step with a gathered q, the path tests/test_gpu_parity.py checks
against the reference's progressive_decode)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _engine(n_layers=2, n_q=8, n_kv=2, d=128, n_new=700, max_new=40, budget=64, interval=8, warmup=8):
    from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
    from paper_2507_13681_b200.kvcompress import CompressionConfig

    shape = AttnShape(n_layers, n_q, n_kv, d)
    cap = n_new + max_new
    store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=5)
    params = SessionParams(alpha=0.9, comp=CompressionConfig(budget, interval, warmup), max_new=max_new, seed=2)
    return SessionEngine(shape, params, cap), store, n_new, max_new


def _run(eng, store, n_new, max_new, mode):
    eng.prefill(store, 0, 0, n_new)
    outs = []
    if mode in ("graphs", "eager"):
        eng.decode(store, n_new, max_new, use_graphs=(mode == "graphs"),
                   out_sink=lambda t, ob: outs.append(ob.float().cpu().clone()))
    else:  # per-step path: gathered q, no graphs, no PDL
        st, comp, sh = eng.stack, eng.params.comp, eng.shape
        compressed = False
        q_buf = torch.empty((sh.n_layers, sh.n_q, sh.d), dtype=torch.bfloat16, device="cuda")
        out = torch.empty((sh.n_layers, sh.n_q, sh.d), dtype=torch.bfloat16, device="cuda")
        for n_o in range(1, max_new + 1):
            if comp.event_at(n_o):
                st.event(comp.budget, store.k, store.v, max_len=n_new + max_new)
                compressed = True
            q_buf.copy_(store.q[:, :, st.length])
            cols = n_new + max_new + 1
            for l in range(sh.n_layers):
                st.step(l, q_buf[l], store.k[l], store.v[l], compressed, cols, out[l])
            st.advance()
            outs.append(out.float().cpu().clone())
    torch.cuda.synchronize()
    return torch.stack(outs).numpy()


def test_engine_decode_paths_identical(cuda_lib):
    ref = _run(*_engine(), mode="step")
    eager = _run(*_engine(), mode="eager")
    graphs = _run(*_engine(), mode="graphs")
    assert np.isfinite(ref).all()
    # graphs vs eager: identical launches -> bit-identical
    assert np.array_equal(graphs, eager), float(np.abs(graphs - eager).max())
    # vs the per-step path: the split-K grid differs (column bounds), so the
    # combine order differs; outputs agree to bf16 rounding (parity bar 2e-2)
    assert np.abs(eager - ref).max() <= 2e-2, float(np.abs(eager - ref).max())


def test_vs_attention_tile_counter(cuda_lib):
    """ls_vs_attention_ex counts tiles and leaves outputs/cells unchanged."""
    from paper_2507_13681_b200.engine import AttnShape, QKVStore
    from paper_2507_13681_b200.prefill import sample_rows_device, sparsify_layer
    from paper_2507_13681_b200.tensor_ops import attention_layer

    shape = AttnShape(1, 4, 1, 128)
    n = 1500
    store = QKVStore.synthetic(shape, n, n_ref=n, seed=9)
    rows = sample_rows_device(n, 0.1, 32, 0, 0, 0, 0, 4)
    qb = store.q[0]
    plans = sparsify_layer(qb, store.k[0], rows, 0.9, n, n, 1)
    o1, c1 = attention_layer(qb, store.k[0], store.v[0], plans.slash_ids, plans.vert_ids, plans.counts, n, n, 1)
    tiles = torch.zeros(4, dtype=torch.int64, device="cuda")
    o2, c2 = attention_layer(qb, store.k[0], store.v[0], plans.slash_ids, plans.vert_ids, plans.counts, n, n, 1,
                             tiles=tiles)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(c1, c2)
    t = tiles.cpu().numpy()
    n_qt = -(-n // 128)
    assert (t >= n_qt).all() and (t <= n_qt * (n_qt + 2 * (n // 128 + 2))).all()
    # every executed tile holds at most 128 x 128 cells
    assert (c1.cpu().numpy() <= t * 128 * 128).all()


def test_long_context_turn_c3_shape(cuda_lib):
    """C3-sized turn block (33.5K keys, beyond the single-SM sort / table
    capacities): the whole LoopServe turn runs and stays consistent."""
    from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
    from paper_2507_13681_b200.kvcompress import CompressionConfig

    shape = AttnShape(1, 4, 1, 128)
    ro, n_new, max_new = 25088, 8448, 24
    cap = ro + n_new + max_new
    store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=11)
    eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(2048, 16, 16), max_new=max_new),
                        cap)
    res = eng.prefill(store, 3, ro, n_new)
    last = eng.decode(store, ro + n_new, max_new)
    torch.cuda.synchronize()
    plans = res.plans[0]
    cn = plans.counts.cpu().numpy()
    assert (cn.sum(axis=1) > 0).all()
    sl, vt = plans.slash_ids.cpu().numpy(), plans.vert_ids.cpu().numpy()
    for h in range(4):  # sorted, unique, in range
        s, v = sl[h, :cn[h, 0]], vt[h, :cn[h, 1]]
        assert (np.diff(s) > 0).all() and (np.diff(v) > 0).all()
        assert s.max(initial=0) < ro + n_new and v.max(initial=0) < ro + n_new
    cov = plans.coverage.cpu().numpy()
    assert ((cov >= 0.955 - 1e-6) & (cov <= 1.0)).all()
    cells = res.cells[0].cpu().numpy()
    dense_cells = n_new * ro + n_new * (n_new + 1) // 2
    assert (cells > 0).all() and (cells <= dense_cells).all()
    assert torch.isfinite(res.out[0].float()).all() and torch.isfinite(last.float()).all()


def test_head_group_pipeline_identical(cuda_lib):
    """Prefill as head groups on their own streams (each group writing its
    head columns of the shared output through out_row_stride) gives the
    one-launch-per-layer results bit for bit: every kernel is per head."""
    from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
    from paper_2507_13681_b200.kvcompress import CompressionConfig

    shape = AttnShape(2, 8, 4, 128)
    n_new = 900
    store = QKVStore.synthetic(shape, n_new + 16, n_ref=n_new + 16, seed=7)
    res = []
    for hg in (1, 2, 4):
        eng = SessionEngine(shape, SessionParams(alpha=0.9, comp=CompressionConfig(64, 8, 8), max_new=16, seed=3),
                            n_new + 16, head_groups=hg)
        r = eng.prefill(store, 0, 0, n_new)
        torch.cuda.synchronize()
        res.append((r, eng.stack.ring_s.clone()))
    (r1, ring1) = res[0]
    for r, ring in res[1:]:
        for l in range(shape.n_layers):
            assert torch.equal(r.out[l], r1.out[l])
            assert torch.equal(r.plans[l].counts, r1.plans[l].counts)
            cn = r1.plans[l].counts.cpu()
            for h in range(shape.n_q):  # id lists are valid up to their counts
                assert torch.equal(r.plans[l].slash_ids[h, :cn[h, 0]], r1.plans[l].slash_ids[h, :cn[h, 0]])
                assert torch.equal(r.plans[l].vert_ids[h, :cn[h, 1]], r1.plans[l].vert_ids[h, :cn[h, 1]])
            assert torch.equal(r.cells[l], r1.cells[l])
        assert torch.equal(ring, ring1)  # seed rows


def test_prefill_layer_hooks(cuda_lib):
    """layer_ready / layer_done bracket every layer in order and do not change
    the results (bench.py's e2e streams Q/K/V in and outputs out through them)."""
    eng, store, n_new, _ = _engine(n_layers=3)
    ref = eng.prefill(store, 0, 0, n_new)
    calls = []
    res = eng.prefill(store, 0, 0, n_new, layer_ready=lambda l, s: calls.append(("ready", l)),
                      layer_done=lambda l, o, s: calls.append(("done", l, o.data_ptr())))
    torch.cuda.synchronize()
    assert [c[:2] for c in calls] == [(k, l) for l in range(3) for k in ("ready", "done")]
    for l in range(3):
        assert calls[2 * l + 1][2] == res.out[l].data_ptr()
        assert torch.equal(res.out[l], ref.out[l])


def test_multistep_graphs_identical(cuda_lib):
    """Without a per-step sink every run of steps between events is one graph
    replay; the last step's outputs and the decode state equal the eager path."""
    outs = []
    for use_graphs in (False, True):
        eng, store, n_new, max_new = _engine()
        eng.prefill(store, 0, 0, n_new)
        last = eng.decode(store, n_new, max_new, use_graphs=use_graphs)
        torch.cuda.synchronize()
        st = eng.stack
        outs.append((last.float().cpu().clone(), st.step_t.cpu().clone(), st.sel_ids.cpu().clone(),
                     st.n_a.cpu().clone(), (st.length, st.appended)))
    (a, sa, sela, naa, ha), (b, sb, selb, nab, hb) = outs
    assert torch.equal(a, b)
    assert torch.equal(sa, sb) and torch.equal(sela, selb) and torch.equal(naa, nab) and ha == hb


def test_multi_turn_session_with_archive_append_truncate(cuda_lib):
    """A 3-turn session driven like run_turn (session.py:113-201) on an
    append-only archive: append the block (previous answer + input), prefill,
    append the decoded tokens' rows, decode, roll them back with truncate
    (session.py:180) -- identical plans and outputs to the preloaded store, and
    the plan ledger holds every (turn, layer)."""
    from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
    from paper_2507_13681_b200.kvcompress import CompressionConfig

    shape = AttnShape(2, 4, 2, 128)
    IN, MAX_NEW, T = 900, 24, 3
    cap = T * (IN + MAX_NEW)
    ref = QKVStore.synthetic(shape, cap, n_ref=cap, seed=8)
    params = SessionParams(alpha=0.95, comp=CompressionConfig(128, 8, 8), max_new=MAX_NEW, seed=3)
    e1, e2 = SessionEngine(shape, params, cap), SessionEngine(shape, params, cap)
    st = QKVStore.empty(shape, cap)
    for t, (ro, n_new) in enumerate(e1.turn_blocks(IN, T, MAX_NEW)):
        hi = ro + n_new
        st.truncate(ro)  # the previous turn's decode rows are re-prefilled as this block
        st.append(ref.q[:, :, ro:hi], ref.k[:, :, ro:hi], ref.v[:, :, ro:hi])
        a = e1.prefill(ref, t, ro, n_new)
        b = e2.prefill(st, t, ro, n_new)
        st.append(ref.q[:, :, hi:hi + MAX_NEW], ref.k[:, :, hi:hi + MAX_NEW], ref.v[:, :, hi:hi + MAX_NEW])
        oa = e1.decode(ref, hi, MAX_NEW).clone()
        ob = e2.decode(st, hi, MAX_NEW).clone()
        torch.cuda.synchronize()
        for l in range(2):
            assert torch.equal(a.out[l], b.out[l])
            assert a.plans[l].to_host() == b.plans[l].to_host()
        assert torch.equal(oa, ob)
        st.truncate(hi)
    assert sorted(e2.plan_ledger) == [(t, l) for t in range(T) for l in range(2)]
    with pytest.raises(Exception):
        e2.decode(st, st.length, MAX_NEW)  # decode rows not appended yet
