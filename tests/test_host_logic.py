"""Host-side logic on CPU: turn geometry, deque/seed bookkeeping, sharding
and the NCCL all-gather path (exercised with gloo, world_size 2)."""

import os
import socket
from collections import deque

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import seeding as oseed
from paper_2507_13681_b200.kvcompress import CompressionConfig
from paper_2507_13681_b200.parallel import HeadShard, OutputGather, session_shard


def test_turn_blocks_match_session_loop():
    """session.py:122 (block = previous answer + input) and :180 (rollback)."""
    from bench import turn_blocks

    input_len, max_new = 5000, 128
    blocks = turn_blocks(input_len, 3, max_new)
    assert blocks == [(0, 5000), (5000, 5128), (10128, 5128)]
    # n_total after prefill equals SURVEY 8 table: 5000, 10128, 15256
    assert [ro + n for ro, n in blocks] == [5000, 10128, 15256]
    # sample sizes of those blocks (prefill.py:132)
    assert [oseed.sample_size(n, 0.1, 32) for _, n in blocks] == [500, 513, 513]


@pytest.mark.parametrize("W,warmup,interval,n_seed,max_new", [(16, 16, 16, 16, 128), (9, 7, 5, 9, 33),
                                                               (12, 3, 6, 12, 30), (4, 4, 4, 4, 20),
                                                               (8, 30, 4, 8, 10)])
def test_surviving_seeds_matches_deque(W, warmup, interval, n_seed, max_new):
    """kvcompress.py:196/233: the seeds present at the first event."""
    comp = CompressionConfig(budget=8, interval=interval, warmup=warmup, obs_window=W)
    buf = deque([("seed", i) for i in range(n_seed)], maxlen=W)
    first = None
    for n_o in range(1, max_new + 1):
        if comp.event_at(n_o):
            first = sum(1 for x in buf if x[0] == "seed")
            break
        buf.append(("row", n_o))
    expect = first if first is not None else 0
    assert comp.surviving_seeds(n_seed, max_new) == expect


def test_event_schedule():  # test_kvcompress.py:245-256
    comp = CompressionConfig(budget=3, interval=5, warmup=5, obs_window=5)
    assert [n for n in range(1, 13) if comp.event_at(n)] == [5, 10]
    assert not any(CompressionConfig(budget=None).event_at(n) for n in range(1, 100))


def test_head_shard_partition():
    for world in (1, 2, 4, 8):
        owned = []
        for r in range(world):
            s = HeadShard(32, 8, world, r)
            assert s.n_q_local == 32 // world
            # every q-head of a kv group lives with its group
            for h in s.q_heads():
                assert h // 4 in s.kv_heads()
            owned += list(s.q_heads())
        assert owned == list(range(32))
    with pytest.raises(ValueError):
        HeadShard(28, 4, 8, 0)  # Qwen2.5-7B: 4 kv heads cannot split over 8 ranks
    assert sorted(sum((session_shard(64, 8, r) for r in range(8)), [])) == list(range(64))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shard = HeadShard(8, 4, world, rank)
    d = 4
    n_new = 3
    # every rank computes its heads' "outputs" as a function of the global head id
    local = torch.stack([torch.full((n_new, d), float(h)) for h in shard.q_heads()], dim=1)
    full = OutputGather(shard, d).prefill(local)
    step = [torch.full((shard.n_q_local, d), float(l * 100 + rank)) for l in range(2)]
    dec = OutputGather(shard, d).decode(step)
    # a run of 3 decode steps of 2 layers in one collective (SessionEngine.decode(run_sink=...))
    run = torch.stack([torch.stack([torch.stack([torch.full((d,), float(1000 * s + 100 * l + h))
                                                 for h in shard.q_heads()]) for l in range(2)]) for s in range(3)])
    run_full = OutputGather(shard, d).decode_run(run)
    assert run_full.shape == (3, 2, 8, d)
    for s_ in range(3):
        for l in range(2):
            for h in range(8):
                assert torch.all(run_full[s_, l, h] == 1000 * s_ + 100 * l + h)
    # per-head sampling seeds depend on the GLOBAL head id only
    rows = [oseed.sample_rows(500, 0.1, 32, oseed.head_seed(0, 1, 0, h)) for h in shard.q_heads()]
    q.put((rank, full.numpy(), [x.numpy() for x in dec], [r.tolist() for r in rows]))
    dist.destroy_process_group()


def test_output_gather_gloo_two_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=60) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    for rank, full, dec, rows in res:
        assert full.shape == (3, 8, 4)
        for h in range(8):
            assert np.all(full[:, h] == h)  # head concat order == global head order
        for l in range(2):
            assert dec[l].shape == (8, 4)
            assert np.all(dec[l][:4] == l * 100 + 0) and np.all(dec[l][4:] == l * 100 + 1)
    # sharded sampling == unsharded sampling (index sets invariant under sharding)
    all_rows = res[0][3] + res[1][3]
    for h in range(8):
        assert all_rows[h] == oseed.sample_rows(500, 0.1, 32, oseed.head_seed(0, 1, 0, h)).tolist()


def test_dropin_rebinds_reference_names():
    """dropin.install() rebinds the reference's import-time name bindings
    (session.py:19-37, model.py:20, kvcompress.py:18) in the calling modules
    -- on the compiled reference itself when oracle/_ref is built -- and
    uninstall() restores them."""
    import types

    from paper_2507_13681_b200 import dropin, kvcompress, prefill, tensor_ops
    from c1_harness import reference_modules

    ref = reference_modules()
    if ref is not None:
        mods = {f"loopserve.{k}": v for k, v in ref.items()}
        before = {(m, a): getattr(mods[m], a) for m, a in dropin.PATCHES if m in mods and hasattr(mods[m], a)}
    else:
        orig = object()
        mods = {}
        for (mod_name, attr) in dropin.PATCHES:
            m = mods.setdefault(mod_name, types.ModuleType(mod_name))
            setattr(m, attr, orig)
        before = {(m, a): orig for m, a in dropin.PATCHES}
    done = dropin.install(mods)
    try:
        assert sorted(done) == sorted(f"{m}.{a}" for m, a in before)
        assert mods["loopserve.session"].sparsify_head.__wrapped__ is prefill.sparsify_head
        assert mods["loopserve.model"].masked_sparse_attention.__wrapped__ is tensor_ops.masked_sparse_attention
        assert mods["loopserve.model"].scaled_dot_attention.__wrapped__ is tensor_ops.scaled_dot_attention
        assert mods["loopserve.kvcompress"].accumulate_scores.__wrapped__ is kvcompress.accumulate_scores
        assert mods["loopserve.kvcompress"]._top_by_score.__wrapped__ is kvcompress._top_by_score
        assert mods["loopserve.kvcompress"].retained_union.__wrapped__ is kvcompress.retained_union
        dec = mods["loopserve.kvcompress"].decode_step
        assert getattr(dec, "__b200__", False) and mods["loopserve.session"].decode_step is dec
        if ref is not None:
            assert getattr(ref["model"].KVCache.truncate, "__b200__", False)
    finally:
        dropin.uninstall()
    assert all(getattr(mods[m], a) is fn for (m, a), fn in before.items())
    if ref is not None:
        assert not getattr(ref["model"].KVCache.truncate, "__b200__", False)


def test_qkvstore_append_truncate_validate():
    """QKVStore as the reference KVCache archive (model.py:139-175): append at
    the filled prefix, roll back with truncate, CacheCorrupt / SequenceTooLong
    as the reference raises them."""
    import torch

    from paper_2507_13681_b200.engine import AttnShape, QKVStore
    from paper_2507_13681_b200.errors import CacheCorrupt, SequenceTooLong

    sh = AttnShape(2, 4, 2, 8)
    st = QKVStore.empty(sh, 10, device="cpu")
    assert st.length == 0
    blk = lambda n, h, x: torch.full((2, h, n, 8), float(x), dtype=torch.bfloat16)
    assert st.append(blk(6, 4, 1), blk(6, 2, 2), blk(6, 2, 3)) == 6
    assert torch.all(st.k[:, :, :6] == 2) and torch.all(st.v[:, :, :6] == 3)
    st.truncate(4)  # decode rows rolled back (session.py:180)
    assert st.append(blk(3, 4, 7), blk(3, 2, 8), blk(3, 2, 9)) == 7
    assert torch.all(st.k[:, :, 4:7] == 8) and torch.all(st.k[:, :, :4] == 2)
    with pytest.raises(SequenceTooLong):
        st.append(blk(4, 4, 0), blk(4, 2, 0), blk(4, 2, 0))
    with pytest.raises(CacheCorrupt):
        st.truncate(8)
    st.length = 11
    with pytest.raises(CacheCorrupt):
        st.validate()
    assert QKVStore(sh, 10, device="cpu").length == 10  # preloaded by default
