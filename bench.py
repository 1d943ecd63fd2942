"""LoopServe hot-path benchmark (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1], "C2"): Llama-3.1-8B attention shapes --
32 layers, 32 q / 8 KV heads, d = 128, bf16 -- a 3-turn dialogue of 5000-token
inputs, 128 decoded tokens per turn, LoopServe mode with the paper defaults
alpha = 0.955, sample 0.1 / floor 32, KV budget B = 1024, n_d = 16, warmup 16,
obs window 16. Synthetic structured Q/K/V generated on the
device; Q/K/V of all layers (~6 GB) exceed L2, so no flush is needed.

One step = one full dialogue: per turn the sparse prefill of every layer
(K0 sampling, K1 scoring, K2-K4 selection, K5 sparse attention, decode seeds)
and 128 compressed decode steps of every layer (K7/K8 events + K6).
  value  = TTFT: mean sparse-prefill time of one turn block over all layers, ms
  decode_tokens_per_s = decoded tokens / decode time
Multi-GPU (torchrun): KV-head groups are split across ranks (all q-heads of a
group on one rank, K/V never replicated) and each layer's attention output is
all-gathered over NCCL (the head concat before W_O, model.py:259); time is the
max over ranks ("strong" scaling: the dialogue is fixed).

--impl reference: the reference algorithm's CPU implementation (the oracle
port of oracle/, run with all host cores on a bounded sample of the same
workload, extrapolated to the full dialogue; the reference itself is pure
Python and cannot travel to the GPU box).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "prefill TTFT (ms) & decode tokens/s, Llama-3.1-8B attn shapes, 1/2/4/8 B200"

CONFIGS = {
    "c2": dict(workload="C2: Llama-3.1-8B attention (32q/8kv, d=128, bf16), 32 layers, 3 turns x 5000 tokens, "
                        "128 decoded tokens/turn, alpha=0.955, B=1024, n_d=16, sparse prefill + compressed decode",
               n_layers=32, n_q=32, n_kv=8, d=128, input_len=5000, n_turns=3, max_new=128, alpha=0.955,
               budget=1024, interval=16, warmup=16, obs_window=None, rate=0.1, floor=32),
    "c3": dict(workload="C3: Llama-3.1-8B attention (32q/8kv, d=128, bf16), 32 layers, 4 turns x 8192 tokens "
                        "(33.5K-token context), 256 decoded tokens/turn, alpha=0.955, B=2048, n_d=16, "
                        "head-sharded over the ranks",
               n_layers=32, n_q=32, n_kv=8, d=128, input_len=8192, n_turns=4, max_new=256, alpha=0.955,
               budget=2048, interval=16, warmup=16, obs_window=None, rate=0.1, floor=32),
    "c4": dict(workload="C4: Qwen2.5-7B attention (28q/4kv, d=128, bf16), 28 layers, 64 independent 3-turn x 5000-token "
                        "sessions sharded over 8 B200 (8 sessions per GPU, batched into every launch), 128 decoded "
                        "tokens/turn, alpha=0.955, B=1024, n_d=16",
               n_layers=28, n_q=28, n_kv=4, d=128, input_len=5000, n_turns=3, max_new=128, alpha=0.955,
               budget=1024, interval=16, warmup=16, obs_window=None, rate=0.1, floor=32, sessions=8),
    "c5": dict(workload="C5: Llama-3.1-70B attention (64q/8kv, d=128, bf16), 80 layers, 10 turns x 10000 tokens "
                        "(~101K-token context), 128 decoded tokens/turn, alpha=0.955, B=1024, n_d=16, one KV-head "
                        "group (8 q-heads) per GPU of 8 (each rank runs its shard; at N < 8 the first N shards)",
               n_layers=80, n_q=64, n_kv=8, d=128, input_len=10000, n_turns=10, max_new=128, alpha=0.955,
               budget=1024, interval=16, warmup=16, obs_window=None, rate=0.1, floor=32, kv_shards=8),
    "c1": dict(workload="C1: toy attention layer (8 heads MHA, d=64), 3 turns x 1000 tokens, alpha=0.9, B=256",
               n_layers=1, n_q=8, n_kv=8, d=64, input_len=1000, n_turns=3, max_new=32, alpha=0.9, budget=256,
               interval=16, warmup=16, obs_window=None, rate=0.1, floor=32),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    return ap.parse_args()


def _load_traffic():
    """profiles/ncu_traffic.json: dram bytes per launch of the timed entries,
    from one ncu --set full capture (tools/ncu_traffic.py)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh)
    return {}


NCU_TRAFFIC = _load_traffic()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return dict(hbm=d["hbm_gbs"], tensor=d["bf16_tflops"], tensor_sus=d.get("bf16_tflops_sustained"),
                    src="measured")
    return dict(hbm=6650.0, tensor=1590.0, tensor_sus=1400.0, src="fallback")


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------ CPU baseline
_CPU = {}


def _cpu_unit(args):
    """One (turn, head) of the sparse prefill on the oracle: sparsify_head +
    masked_sparse_attention (session.py:135-152 / model.py:242-251)."""
    turn, head = args
    import numpy as np

    from oracle.session import prefill_head

    d = _CPU
    ro, n_new = d["blocks"][turn]
    n_total = ro + n_new
    g = head // d["group"]
    Q = d["Q"][head, ro:n_total].astype(np.float64)
    K = d["K"][g, :n_total].astype(np.float64)
    V = d["V"][g, :n_total].astype(np.float64)
    t0 = time.perf_counter()
    prefill_head(Q, K, V, ro, d["alpha"], d["rate"], d["floor"], 0, turn, 0, head, d["window"])
    return time.perf_counter() - t0


def _cpu_decode_unit(args):
    import numpy as np

    from oracle.kvcompress import decode_head_step

    n_cols, reps = args
    d = _CPU
    k = d["K"][0].astype(np.float64)
    v = d["V"][0].astype(np.float64)
    q = d["Q"][0, n_cols - 1].astype(np.float64)
    cols = np.arange(n_cols)
    t0 = time.perf_counter()
    for _ in range(reps):
        decode_head_step(k, v, q, cols)
    return (time.perf_counter() - t0) / reps


def _cpu_event_unit(args):
    """One compression event of one head on the oracle (kvcompress.py:210-214):
    accumulate_scores over the W buffered rows, top-B, retained_union."""
    import numpy as np

    from oracle import kvcompress as okv

    n_cols, window, budget, length, reps = args
    rng = np.random.Generator(np.random.PCG64(0))
    rows = [(np.sort(rng.choice(length, n_cols, replace=False)), rng.random(n_cols)) for _ in range(window)]
    t0 = time.perf_counter()
    for _ in range(reps):
        ids, sc = okv.accumulate_scores(rows)
        sel = okv.top_by_score(ids, sc, budget)
        okv.retained_union(sel, window, length)
    return (time.perf_counter() - t0) / reps


def _cpu_worker_init():
    """One BLAS thread per worker: `cores` is then the number of threads used."""
    global _BLAS_LIMIT
    from threadpoolctl import threadpool_limits

    _BLAS_LIMIT = threadpool_limits(1)


_BLAS_LIMIT = None


def cpu_baseline(cfg, cores=None):
    """Oracle port on `cores` single-threaded host processes, bounded sample,
    extrapolated."""
    import multiprocessing as mp

    import numpy as np

    from paper_2507_13681_b200.engine import SessionEngine  # noqa: F401 (turn geometry only)
    from paper_2507_13681_b200.synth import SynthSpec, layer_qkv_numpy

    cores = cores or os.cpu_count() or 1
    group = cfg["n_q"] // cfg["n_kv"]
    blocks = turn_blocks(cfg["input_len"], cfg["n_turns"], cfg["max_new"])
    cap = cfg["n_turns"] * (cfg["input_len"] + cfg["max_new"])
    n_q_s = min(cfg["n_q"], max(group, cores))
    n_q_s = ((n_q_s + group - 1) // group) * group
    spec = SynthSpec(n_q_s, n_q_s // group, cfg["d"], cap, seed=0)
    Q, K, V = layer_qkv_numpy(spec, 0)
    _CPU.update(Q=Q, K=K, V=V, blocks=blocks, group=group, alpha=cfg["alpha"], rate=cfg["rate"],
                floor=cfg["floor"], window=cfg["obs_window"] or cfg["interval"])
    ctx = mp.get_context("fork")
    units = cfg["n_layers"] * cfg["n_q"]
    n_t = cfg["n_turns"]
    # one round: (turn, head) units spread over the turns, one per process, so
    # a round takes about one turn-3 unit of wall time (bounded sample)
    per_turn_heads = max(1, min(n_q_s, cores // n_t))
    work = [(t, h) for h in range(per_turn_heads) for t in range(n_t)]
    n_sample = len(work)
    W = cfg["obs_window"] or cfg["interval"]
    with ctx.Pool(min(cores, n_sample), initializer=_cpu_worker_init) as pool:
        times = pool.map(_cpu_unit, work)
        # decode: one head-step at the dense (pre-event) and compressed sizes, and one
        # compression event of a head (its buffered rows over the working set)
        L_end = blocks[-1][0] + blocks[-1][1]
        comp_cols = min(L_end, cfg["budget"] + W + 1)
        dense_t, comp_t = pool.map(_cpu_decode_unit, [(L_end, 3), (comp_cols, 20)])
        event_t = pool.map(_cpu_event_unit, [(comp_cols, W, cfg["budget"], L_end, 5)])[0] if cfg["budget"] else 0.0
    n_proc = min(cores, n_sample)
    # per-unit core time x units / cores in parallel = the turn's TTFT on this host
    per_turn_ms = [1e3 * statistics.mean(tt for (t, _), tt in zip(work, times) if t == turn) * units / n_proc
                   for turn in range(n_t)]
    n_dense = min(cfg["max_new"], cfg["warmup"] - 1 if cfg["budget"] is not None else cfg["max_new"])
    n_events = len(range(cfg["warmup"], cfg["max_new"] + 1, cfg["interval"])) if cfg["budget"] else 0
    step_s = (n_dense * dense_t + (cfg["max_new"] - n_dense) * comp_t + n_events * event_t) / cfg["max_new"]
    tok_s = 1.0 / (step_s * units / n_proc)
    sample = (f"oracle port (numpy fp64): {per_turn_heads} (layer 0, head) prefill units of each of the {n_t} turns "
              f"({n_sample} units in parallel on {n_proc} processes) + decode head-steps at {L_end} and "
              f"{comp_cols} columns + one compression event of a head; per-unit core time extrapolated to "
              f"{units} (layer, head) units on {n_proc} single-threaded processes (BLAS threads limited to 1)")
    return dict(ttft_ms=statistics.mean(per_turn_ms), per_turn_ms=per_turn_ms, decode_tokens_per_s=tok_s,
                cores=n_proc, sample=sample)


def turn_blocks(input_len, n_turns, max_new):
    out, hist = [], 0
    for t in range(n_turns):
        out.append((hist - (max_new if t > 0 else 0), input_len + (max_new if t > 0 else 0)))
        hist += input_len + max_new
    return out


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    for _ in range(args.warmup if args.warmup < 1 else 0):
        pass
    res = []
    for _ in range(max(1, args.steps)):
        res.append(cpu_baseline(cfg))
    v = statistics.mean(r["ttft_ms"] for r in res)
    tok = statistics.mean(r["decode_tokens_per_s"] for r in res)
    line = {"metric": METRIC, "value": round(v, 3), "unit": "ms", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(v * cfg["n_turns"], 3),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": cfg["workload"]},
            "decode_tokens_per_s": round(tok, 3),
            "cpu_baseline": {"value": round(v, 3), "unit": "ms", "cores": res[0]["cores"], "kind": "port",
                             "sample": res[0]["sample"]},
            "e2e": {"value": round(v, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ B200 arm
def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.config != "c2":  # the committed ncu captures are of the C2 workload
        NCU_TRAFFIC.clear()
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")
    from paper_2507_13681_b200 import _lib
    from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
    from paper_2507_13681_b200.kvcompress import CompressionConfig
    from paper_2507_13681_b200.parallel import HeadShard

    n_sess = cfg.get("sessions", 1)
    if n_sess > 1:  # C4: session sharding (no collective), n_sess sessions per GPU batched into every launch
        shard = HeadShard(cfg["n_q"], cfg["n_kv"], 1, 0)
        shape = AttnShape(cfg["n_layers"], n_sess * cfg["n_q"], n_sess * cfg["n_kv"], cfg["d"])
        session_seeds = [rank * n_sess + s for s in range(n_sess)]  # global session ids as Session seeds
        kv_offset = rank * n_sess * cfg["n_kv"]
    else:  # head sharding over the ranks (C5: a fixed 8-way shard, rank r runs shard r)
        shard = HeadShard(cfg["n_q"], cfg["n_kv"], cfg.get("kv_shards", world), rank % cfg.get("kv_shards", world))
        shape = AttnShape(cfg["n_layers"], shard.n_q_local, shard.n_kv_local, cfg["d"])
        session_seeds, kv_offset = None, shard.kv_begin
    comp = CompressionConfig(cfg["budget"], cfg["interval"], cfg["warmup"], cfg["obs_window"])
    params = SessionParams(alpha=cfg["alpha"], comp=comp, sample_rate=cfg["rate"], sample_floor=cfg["floor"],
                           max_new=cfg["max_new"], seed=0)
    blocks = turn_blocks(cfg["input_len"], cfg["n_turns"], cfg["max_new"])
    cap = cfg["n_turns"] * (cfg["input_len"] + cfg["max_new"])
    store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1, kv_offset=kv_offset)
    eng = SessionEngine(shape, params, cap, session_seeds=session_seeds)
    stream = torch.cuda.current_stream()

    # per-entry CUDA-event timing (on the launching stream)
    recs = []
    timing = {"on": False}

    def hook(name, phase):
        if not timing["on"]:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()  # the stream the entry runs on (head-group streams in prefill)
        if phase == "begin":
            recs.append([name, ev, None])
        else:
            for r in reversed(recs):
                if r[0] == name and r[2] is None:
                    r[2] = ev
                    break

    _lib.entry_hook = hook

    gather = shard.make_gather(cfg["d"]) if (world > 1 and n_sess == 1 and "kv_shards" not in cfg) else None

    side = torch.cuda.Stream() if gather is not None else None
    gathered = []

    def layer_done(l, out, s):
        # head-sharded prefill: layer l's output all-gather (the head concat
        # before W_O) runs on a side stream while layer l + 1 computes
        ev = torch.cuda.Event()
        ev.record(s)
        side.wait_event(ev)
        with torch.cuda.stream(side):
            gathered.append(gather.prefill(out))
            out.record_stream(side)

    def dialogue(ev_log):
        for t, (ro, n_new) in enumerate(blocks):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e2 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            gathered.clear()
            res = eng.prefill(store, t, ro, n_new, turn_offset_heads=shard.q_begin,
                              layer_done=layer_done if gather is not None else None)
            if gather is not None:
                stream.wait_stream(side)
            e1.record(stream)
            # decode: one all-gather per run of steps between events (multi-step graphs)
            run_sink = (lambda s0, outs: gather.decode_run(outs)) if gather is not None else None
            eng.decode(store, ro + n_new, cfg["max_new"], run_sink=run_sink)
            e2.record(stream)
            ev_log.append((e0, e1, e2))
            # rollback is implicit: the next block starts at ro + n_new (session.py:180)
        return res

    # warmup
    for _ in range(args.warmup):
        dialogue([])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # timed region
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ev_log = []
    recs.clear()
    eng.clear_logs()
    launches0 = _lib.launch_count
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for _ in range(args.steps):
        dialogue(ev_log)
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = _lib.launch_count - launches0
    clk = clocks.stop()
    total_ms = t_start.elapsed_time(t_end)
    # per-entry breakdown (stages_ms, the rooflines): one more dialogue outside the
    # timed region with CUDA events around every C-ABI entry on its launching
    # stream (the events' host cost stays out of the timed steps), and without the
    # K3/K5 head-group overlap so every kernel's time is its own
    recs.clear()
    eng.clear_logs()
    overlap_min = getattr(eng, "overlap_min", None)
    if overlap_min is not None:
        eng.overlap_min = 1 << 30
    timing["on"] = True
    dialogue([])
    torch.cuda.synchronize()
    timing["on"] = False
    if overlap_min is not None:
        eng.overlap_min = overlap_min
    if world > 1:
        dist.barrier()
    dialogue_ms = total_ms / args.steps  # the breakdown pass covers one dialogue
    prefill_ms = sum(e0.elapsed_time(e1) for e0, e1, _ in ev_log)
    decode_ms = sum(e1.elapsed_time(e2) for _, e1, e2 in ev_log)
    n_prefills = len(ev_log)
    vals = torch.tensor([total_ms, prefill_ms, decode_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    total_ms, prefill_ms, decode_ms = vals.tolist()
    ttft = prefill_ms / n_prefills
    # every session (C4) decodes its own tokens; head-sharded ranks decode the same tokens
    tok_s = n_sess * world ** (n_sess > 1) * args.steps * cfg["n_turns"] * cfg["max_new"] / (decode_ms / 1e3)

    # per-entry shares and the dominant kernel's roofline
    per = {}
    for name, a, b in recs:
        if b is None:
            continue
        per.setdefault(name, []).append(a.elapsed_time(b))
    stages = {k: round(sum(v), 3) for k, v in per.items()}
    peaks = load_peaks()
    roof = roofline(per, cfg, eng, store, blocks, peaks)
    if roof is not None and roof.get("kernel") in per:
        roof["share_of_timed"] = round(sum(per[roof["kernel"]]) / dialogue_ms, 4)
    pre_roof = None  # the sparse-attention kernel (K5) against the tensor pipe
    k5 = next((k for k in ("ls_vs_attention_ex", "ls_vs_attention") if k in per), None)
    if k5 is not None:
        pre_roof = roofline({k5: per[k5]}, cfg, eng, store, blocks, peaks)
        pre_roof["share_of_timed"] = round(sum(per[k5]) / dialogue_ms, 4)
    dec_roof = None  # the decode step (one graph replay, all layers) against HBM
    for k in ("decode_graph_comp", "decode_graph_dense"):
        if k in per:
            dec_roof = roofline({k: per[k]}, cfg, eng, store, blocks, peaks)
            dec_roof["share_of_timed"] = round(sum(per[k]) / dialogue_ms, 4)
            break

    ev_roof = event_roofline(per, cfg, eng, shape, blocks, peaks)
    k1_roof = k1_roofline(per, eng, cfg, clk)
    if n_sess > 1 or "kv_shards" in cfg:
        # plan quality, end-to-end and CPU legs are measured on C2; the dense
        # baseline also runs at C5 (the long-context case), not for C4's batch
        args.no_e2e = args.no_cpu_baseline = True
        if n_sess > 1:
            args.no_dense = True
    dense = None if args.no_dense else dense_baseline(cfg, store, blocks, shard, ttft)
    quality = None if args.no_dense or "kv_shards" in cfg else plan_quality(cfg, eng, store, blocks, shard)

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, cfg, eng, store, blocks, shard, gather)

    line = {"metric": METRIC, "value": round(ttft, 3), "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 3), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (structured Q/K/V, SURVEY 8d; random-init, no checkpoint)",
            "config": {"workload": cfg["workload"], "layers": cfg["n_layers"], "q_heads": cfg["n_q"],
                       "kv_heads": cfg["n_kv"], "head_dim": cfg["d"], "turn_blocks": blocks,
                       "max_new": cfg["max_new"], "parallelism": f"kv-head groups x{world}",
                       "l2": "inputs larger than L2 (Q/K/V of all layers ~%.1f GB)" % (
                           store.q.numel() * 2 * (1 + 2 * cfg["n_kv"] / cfg["n_q"]) / 1e9)},
            "decode_tokens_per_s": round(tok_s, 2),
            "prefill_ms_per_turn": round(ttft, 3), "decode_ms_per_turn": round(decode_ms / n_prefills, 3),
            "stages_ms": stages, "stages_note": "per-entry CUDA-event times of one dialogue run after the timed "
                                                  "steps (no head-group overlap); the rooflines use the same pass",
            "gpu_launches": launches, "clocks": clk, "roofline": roof,
            "decode_roofline": dec_roof, "prefill_roofline": pre_roof, "event_roofline": ev_roof,
            "k1_roofline": k1_roof, "dense_baseline": dense, "plan_quality": quality}
    if n_sess > 1:
        line["scaling"] = "weak"
        line["config"]["parallelism"] = f"sessions: {n_sess} per GPU x {world} GPU(s), batched per launch"
    if "kv_shards" in cfg:
        line["scaling"] = "weak"
        line["config"]["parallelism"] = f"kv-head group shard {rank % cfg['kv_shards']} of {cfg['kv_shards']} per GPU"
    if e2e is not None:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(cfg)
        line["cpu_baseline"] = {"value": round(cb["ttft_ms"], 1), "unit": "ms", "cores": cb["cores"], "kind": "port",
                                "sample": cb["sample"], "decode_tokens_per_s": round(cb["decode_tokens_per_s"], 4)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def event_roofline(per, cfg, eng, shape, blocks, peaks):
    """Compression events (one graph: K7 select + K8 compaction, all layers)
    against HBM. Algorithmic bytes of the turn's events:
    K7 reads every buffered row once -- dense rows (prefill seeds, pre-event
    steps) 4 B per column; compressed rows 4 B per logit over B + W + 1 columns
    plus the B picked ids once (the rows' ids derive from the selection when
    interval >= window, else 4 B more per column) -- and K8 reads and writes
    every selected K and V row: 2 * 2 * B * d * 2 B per (layer, q-head)."""
    name = "decode_graph_event"
    if name not in per or not cfg.get("budget"):
        return None
    B, W, d = cfg["budget"], cfg["obs_window"] or cfg["interval"], cfg["d"]
    units = shape.n_layers * shape.n_q
    tot, n_ev = 0.0, 0
    for ro, n_new in blocks:
        L0 = ro + n_new
        for n_o in range(cfg["warmup"], cfg["max_new"] + 1, cfg["interval"]):
            L = L0 + n_o - 1
            if n_o == cfg["warmup"]:  # seeds and dense steps: every column
                k7 = sum(4.0 * (L0 + t) for t in range(max(0, n_o - W), n_o))
            elif cfg["interval"] >= W:  # working-set rows (LS_RING_WORKING_SET)
                k7 = W * 4.0 * (B + W + 1) + 4.0 * B
            else:
                k7 = W * 8.0 * (B + W + 1)
            k8 = 2 * 2 * min(B, L) * d * 2.0
            tot += units * (k7 + k8)
            n_ev += 1
    mean_ms = statistics.mean(per[name])
    bytes_ = tot / max(1, n_ev)
    ach = bytes_ / (mean_ms * 1e-3) / 1e9
    return {"kernel": name, "bound": "hbm", "achieved": round(ach, 3), "peak": peaks["hbm"], "unit": "GB/s",
            "frac": round(ach / peaks["hbm"], 5), "mean_launch_ms": round(mean_ms, 4), "launches": len(per[name]),
            "work_per_launch": bytes_, "peak_src": peaks["src"],
            "traffic": (NCU_TRAFFIC.get(name) or {}).get("dram_bytes_per_launch"),
            "traffic_src": (NCU_TRAFFIC.get(name) or {}).get("source")}


def k1_roofline(per, eng, cfg, clk):
    """K1 (ls_score_lines: stats + lines passes over the causal sampled cells)
    against max(tensor, MUFU): per pass 2*d FLOPs of QK^T and
    one ex2 per cell, so 2 passes = 4*d FLOPs + 2 ex2 per cell. MUFU peak: 16
    ex2 / clk / SM x 148 SMs at the sampled SM clock (B200_PROFILING.md)."""
    name = "ls_score_lines"
    if name not in per or not eng.score_log:
        return None
    n = len(per[name])
    cells = float(sum(int(c.sum()) for c in eng.score_log)) / n
    mean_ms = statistics.mean(per[name])
    sm_ghz = ((clk or {}).get("sm_mhz") or 1965.0) / 1e3
    mufu_peak = 16 * 148 * sm_ghz * 1e9  # ex2 / s
    peaks = load_peaks()
    tensor_peak = (peaks["tensor_sus"] or peaks["tensor"]) * 1e12
    t_mufu = 2 * cells / mufu_peak * 1e3
    t_tensor = 2 * 2 * cfg["d"] * cells / tensor_peak * 1e3
    bound = "mufu" if t_mufu >= t_tensor else "tensor"
    nc = NCU_TRAFFIC.get(name) or {}
    return {"kernel": name, "bound": bound, "cells_per_launch": cells, "bound_ms": round(max(t_mufu, t_tensor), 4),
            "mufu_bound_ms": round(t_mufu, 4), "tensor_bound_ms": round(t_tensor, 4),
            "mean_launch_ms": round(mean_ms, 4), "frac": round(max(t_mufu, t_tensor) / mean_ms, 4),
            "achieved": round(2 * cells / (mean_ms * 1e-3) / 1e12, 4), "unit": "T ex2/s",
            "peak": round(mufu_peak / 1e12, 4), "launches": n, "traffic": nc.get("dram_bytes_per_launch"),
            "ncu_xu_pct": {"lines": nc.get("lines_xu_pct"), "stats": nc.get("stats_xu_pct")},
            "traffic_src": nc.get("source")}


def roofline(per, cfg, eng, store, blocks, peaks):
    """Dominant entry by measured time; algorithmic work per launch / mean
    launch duration. K5 (ls_vs_attention): 4*d*cells FLOPs (exact plan cells,
    the reference's OpCounter units, tensor_ops.py:172-174). K1
    (ls_score_lines): 2*d*score_count FLOPs + 1 exp per cell."""
    if not per:
        return None
    # the dominant entry among those with an algorithmic model (K3's sequential
    # greedy, dominant at C5's 101K keys, has none)
    modeled = {k: v for k, v in per.items() if k in ("ls_vs_attention", "ls_vs_attention_ex", "ls_score_lines")
               or (k.startswith("decode_graph_") and k != "decode_graph_event")}
    name = max(modeled or per, key=lambda k: sum(per[k]))
    mean_ms = statistics.mean(per[name])
    extra = {}
    d = cfg["d"]
    # algorithmic work of the last dialogue's launches of this entry
    work = None
    n = len(per[name])
    if name in ("ls_vs_attention", "ls_vs_attention_ex") and eng.cell_log:
        work = 4.0 * d * float(sum(int(c.sum()) for c in eng.cell_log)) / n
        bound, unit, peak = "tensor", "TFLOP/s", peaks["tensor_sus"] or peaks["tensor"]
        achieved = work / (mean_ms * 1e-3) / 1e12
        if eng.tile_log:  # executed 128x128 tiles: the tensor pipe's actual work
            ex = 4.0 * d * 128 * 128 * float(sum(int(t.sum()) for t in eng.tile_log)) / n
            extra = {"executed_tflops": round(ex / (mean_ms * 1e-3) / 1e12, 3),
                     "executed_frac": round(ex / (mean_ms * 1e-3) / 1e12 / peak, 5),
                     "algorithmic_over_executed": round(work / ex, 4),
                     # the same executed work against the nominal 2.25 PF dense bf16 peak, beside
                     # ncu's tensor-pipe activity of one captured launch (of nominal)
                     "executed_frac_of_nominal": round(ex / (mean_ms * 1e-3) / 1e12 / 2250.0, 5)}
            nc = NCU_TRAFFIC.get("ls_vs_attention") or {}
            if "ncu_tensor_active_pct_of_nominal" in nc:
                extra["ncu_tensor_active_of_nominal"] = round(nc["ncu_tensor_active_pct_of_nominal"] / 100.0, 5)
    elif name == "ls_score_lines" and eng.score_log:
        work = 2.0 * d * float(sum(int(c.sum()) for c in eng.score_log)) / n  # QK^T of the causal sampled cells
        bound, unit, peak = "tensor", "TFLOP/s", peaks["tensor_sus"] or peaks["tensor"]
        achieved = work / (mean_ms * 1e-3) / 1e12
    elif name.startswith("decode_graph_") and name != "decode_graph_event":
        kind = name[len("decode_graph_"):]
        cols = [c for k, c in eng.decode_log if k == kind]
        # bf16 K + V row per KV-head column, all layers, per launch (a launch is a
        # graph of one or more steps)
        bytes_ = 4.0 * d * sum(cols) / max(1, n)
        extra = {"steps_per_launch": round(len(cols) / max(1, n), 3)}
        bound, unit, peak = "hbm", "GB/s", peaks["hbm"]
        achieved = bytes_ / (mean_ms * 1e-3) / 1e9 if bytes_ else None
        work = bytes_
    else:
        return {"kernel": name, "mean_ms": round(mean_ms, 4), "note": "no algorithmic model"}
    res = {"kernel": name, "bound": bound, "achieved": round(achieved, 3) if achieved else None,
            "peak": peak, "unit": unit, "frac": round(achieved / peak, 5) if achieved else None,
            "traffic": None, "mean_launch_ms": round(mean_ms, 4), "launches": len(per[name]),
            "work_per_launch": work, "peak_src": peaks["src"] + (" sustained" if bound == "tensor" else ""),
            "share_of_timed": None}
    res.update(extra)
    tr = NCU_TRAFFIC.get("ls_vs_attention" if name.startswith("ls_vs_attention") else name)
    if tr is not None and "steps_per_launch" in extra:  # the capture is one step
        tr = dict(tr, dram_bytes_per_launch=round(tr["dram_bytes_per_launch"] * extra["steps_per_launch"]))
    if tr:  # dram bytes per launch from the committed ncu --set full capture
        res["traffic"] = tr["dram_bytes_per_launch"]
        res["traffic_src"] = tr["source"]
    return res


def dense_baseline(cfg, store, blocks, shard, sparse_ttft):
    """the same turn blocks through dense causal attention
    (scaled_dot_attention, tensor_ops.py:104-127; K5 in dense mode) -- the
    speed-up denominator of the sparse prefill. Outside the timed region, one
    pass after a warm-up, CUDA events on the launching stream."""
    import torch

    from paper_2507_13681_b200.engine import AttnShape, SessionEngine, SessionParams
    from paper_2507_13681_b200.kvcompress import CompressionConfig

    shape = AttnShape(cfg["n_layers"], shard.n_q_local, shard.n_kv_local, cfg["d"])
    cap = store.cap
    eng = SessionEngine(shape, SessionParams(mode="dense", comp=CompressionConfig(budget=None),
                                             max_new=cfg["max_new"]), cap)
    stream = torch.cuda.current_stream()
    ro, n_new = blocks[0]
    eng.prefill(store, 0, ro, n_new)  # warm-up
    per_turn = []
    for t, (ro, n_new) in enumerate(blocks):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.prefill(store, t, ro, n_new)
        e1.record(stream)
        per_turn.append((e0, e1))
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in per_turn]
    dense_cells = sum(n * ro + n * (n + 1) // 2 for ro, n in blocks) * shard.n_q_local * cfg["n_layers"]
    tflops = 4.0 * cfg["d"] * dense_cells / (sum(ms) * 1e-3) / 1e12
    # full-cache decode (decode_step without working sets, model.py:301-306): every
    # step attends to the whole archive; after the last turn's prefill
    ro, n_new = blocks[-1]
    eng.decode(store, ro + n_new, cfg["max_new"])  # graphs captured + warm
    eng.prefill(store, len(blocks) - 1, ro, n_new)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    eng.decode(store, ro + n_new, cfg["max_new"])
    e1.record(stream)
    torch.cuda.synchronize()
    dec_ms = e0.elapsed_time(e1)
    return {"ttft_ms_per_turn": [round(x, 3) for x in ms], "ttft_ms": round(statistics.mean(ms), 3),
            "sparse_speedup": round(statistics.mean(ms) / sparse_ttft, 3), "dense_tflops": round(tflops, 1),
            "decode_tokens_per_s_last_turn": round(cfg["max_new"] / (dec_ms * 1e-3), 2),
            "note": "dense causal attention of the same turn blocks (K5 dense mode, all layers), one pass; "
                    "full-cache decode (no compression) of the last turn's max_new tokens"}


def plan_quality(cfg, eng, store, blocks, shard):
    """full-block coverage (coverage_ratio, prefill.py:254-281,
    on the device) of the last turn's sampled-row plans, first and last layer,
    beside the greedy's own sampled-row coverage. Outside the timed region."""
    import torch

    from paper_2507_13681_b200.tensor_ops import plan_coverage_layer

    t = len(blocks) - 1
    ro, n_new = blocks[t]
    n_total = ro + n_new
    res = eng.prefill(store, t, ro, n_new, turn_offset_heads=shard.q_begin)
    full, sampled = [], []
    for l in (0, cfg["n_layers"] - 1):
        p = res.plans[l]
        cov = plan_coverage_layer(store.q[l, :, ro:n_total], store.k[l], store.v[l], p.slash_ids, p.vert_ids,
                                  p.counts, n_new, n_total, shard.n_kv_local, q_head_stride=store.q.stride(1))
        full.append(cov)
        sampled.append(p.coverage)
    full, sampled = torch.cat(full), torch.cat(sampled)
    torch.cuda.synchronize()
    return {"full_block_coverage_mean": round(float(full.mean()), 4),
            "full_block_coverage_min": round(float(full.min()), 4),
            "sampled_row_coverage_mean": round(float(sampled.mean()), 4),
            "alpha": cfg["alpha"], "layers": [0, cfg["n_layers"] - 1], "turn": t + 1,
            "note": "coverage_ratio of each q-head's plan over the block's dense causal attention (all rows) vs "
                    "the greedy's coverage of the sampled rows it was built from"}


def run_e2e(args, cfg, eng, store, blocks, shard, gather):
    """Same dialogue through the public API with HOST inputs: every turn copies
    its block's Q/K/V (all layers, one contiguous pinned buffer per tensor, as
    a serving front-end hands over the new tokens' projections) into the HBM
    archive and reads every layer's attention output back; the turn's decode
    inputs (q and the new K/V row of each of the max_new steps, all layers) are
    copied in before its decode loop and every step's outputs are copied out.
    Pinned buffers are allocated once, outside the timed region."""
    import torch

    stream = torch.cuda.current_stream()
    L = cfg["n_layers"]
    dev_views = (store.q, store.k, store.v)
    host_blocks = []  # per turn: (prefill q/k/v, decode q/k/v), contiguous pinned
    for ro, n_new in blocks:
        n_total = ro + n_new
        hi = n_total + cfg["max_new"]
        pre = tuple(x[:, :, ro:n_total].contiguous().cpu().pin_memory() for x in dev_views)
        dec = tuple(x[:, :, n_total:hi].contiguous().cpu().pin_memory() for x in dev_views)
        host_blocks.append((pre, dec))
    from cuda.bindings import runtime as cudart

    def h2d_2d(dst, src, stream):
        """pinned [H, n, d] -> the archive's strided [H, n, d] view in one 2-D copy
        (full PCIe rate, no staging buffer, no device-side copy)"""
        H_, n_, d_ = src.shape
        err, = cudart.cudaMemcpy2DAsync(dst.data_ptr(), dst.stride(0) * 2, src.data_ptr(), n_ * d_ * 2, n_ * d_ * 2, H_,
                                        cudart.cudaMemcpyKind.cudaMemcpyHostToDevice, stream.cuda_stream)
        assert err == cudart.cudaError_t.cudaSuccess, err

    stage_dec = tuple(torch.empty(b.shape, dtype=b.dtype, device="cuda") for b in host_blocks[-1][1])
    max_new_rows = max(n for _, n in blocks)
    host_out = [torch.empty((max_new_rows, shard.n_q_local, cfg["d"]), dtype=torch.bfloat16, pin_memory=True)
                for _ in range(L)]
    outs_host = torch.empty((cfg["max_new"], L, shard.n_q_local, cfg["d"]), dtype=torch.bfloat16, pin_memory=True)
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(L)]
    ev_out = [torch.cuda.Event() for _ in range(L)]
    h2d = d2h = 0
    ttfts, dec = [], []
    steps = max(1, args.steps)
    for it in range(steps + 1):  # first iteration warms up
        for t, (ro, n_new) in enumerate(blocks):
            n_total = ro + n_new
            hi = n_total + cfg["max_new"]
            (pq, pk, pv), (dq, dk, dv) = host_blocks[t]
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e2 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            # the block's Q/K/V stream in layer by layer on a copy stream; layer l
            # computes once its rows are in HBM, and its output is copied out on a
            # third stream while layer l + 1 computes (PCIe is full duplex)
            h2d_s.wait_stream(stream)  # the archive rows are free (previous turn done)
            for l in range(L):
                for dst, src in zip(dev_views, (pq, pk, pv)):
                    h2d_2d(dst[l, :, ro:n_total], src[l], h2d_s)
                ev_in[l].record(h2d_s)

            def ready(l, s):
                s.wait_event(ev_in[l])

            def done(l, o, s):
                ev_out[l].record(s)
                d2h_s.wait_event(ev_out[l])
                with torch.cuda.stream(d2h_s):
                    host_out[l][:n_new].copy_(o, non_blocking=True)

            res = eng.prefill(store, t, ro, n_new, turn_offset_heads=shard.q_begin, layer_ready=ready,
                              layer_done=done)
            stream.wait_stream(d2h_s)  # TTFT: every layer's output is on the host
            e1.record(stream)
            if it > 0:
                h2d += sum(x.numel() * 2 for x in (pq, pk, pv))
                d2h += sum(o.numel() * 2 for o in res.out)
            # decode with per-step host I/O
            for dst, stg, src in zip(dev_views, stage_dec, (dq, dk, dv)):
                stg.copy_(src, non_blocking=True)
                dst[:, :, n_total:hi].copy_(stg)
                if it > 0:
                    h2d += src.numel() * 2

            def run_sink(t0, outs):
                # every run's outputs (all steps, all layers) back to the host on the
                # copy stream while the next run computes (each run writes its own
                # slots of the engine's output ring; the turn waits for the copies)
                ev_run = torch.cuda.Event()
                ev_run.record(stream)
                d2h_s.wait_event(ev_run)
                with torch.cuda.stream(d2h_s):
                    outs_host[t0:t0 + outs.shape[0]].copy_(outs, non_blocking=True)

            eng.decode(store, n_total, cfg["max_new"], run_sink=run_sink)
            stream.wait_stream(d2h_s)  # every step's output is on the host
            if it > 0:
                d2h += outs_host.numel() * 2
            e2.record(stream)
            if it > 0:
                ttfts.append((e0, e1))
                dec.append((e1, e2))
    torch.cuda.synchronize()
    ttft = statistics.mean(a.elapsed_time(b) for a, b in ttfts)
    n_t = len(blocks)
    per_turn = [round(statistics.mean(a.elapsed_time(b) for a, b in ttfts[t::n_t]), 3) for t in range(n_t)]
    dec_ms = sum(a.elapsed_time(b) for a, b in dec)
    tok_s = steps * cfg["n_turns"] * cfg["max_new"] / (dec_ms / 1e3)
    return {"value": round(ttft, 3), "unit": "ms", "ttft_ms_per_turn": per_turn, "h2d_bytes_per_step": h2d // steps,
            "d2h_bytes_per_step": d2h // steps, "decode_tokens_per_s": round(tok_s, 2),
            "note": "value = TTFT incl. the turn block's Q/K/V H2D (all layers) and the attention outputs' D2H, "
                    "layer-pipelined (H2D of layer l+1 and D2H of layer l-1 overlap layer l); step = one 3-turn "
                    "dialogue; decode inputs of a turn are copied before its decode loop"}


if __name__ == "__main__":
    main()
