"""Diagnostics for one attention layer at C2 shapes: per-entry CUDA-event
times, plan sizes, chain/final pick counts. Used under ncu for launch lists:
  python tools/diag_layer.py [--turn 2] [--decode 20]
"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2507_13681_b200 import _lib  # noqa: E402
from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams  # noqa: E402
from paper_2507_13681_b200.kvcompress import CompressionConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--turn", type=int, default=2)
    ap.add_argument("--decode", type=int, default=20)
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    input_len, max_new, n_turns = 5000, 128, 3
    cap = n_turns * (input_len + max_new)
    shape = AttnShape(a.layers, 32, 8, 128)
    store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
    params = SessionParams(alpha=0.955, comp=CompressionConfig(1024, 16, 16, None), max_new=max_new)
    eng = SessionEngine(shape, params, cap)
    blocks = [(0, 5000), (5000, 5128), (10128, 5128)]
    ro, n_new = blocks[a.turn]
    stream = torch.cuda.current_stream()
    per = {}
    recs = []

    def hook(name, phase):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        if phase == "begin":
            recs.append([name, ev, None])
        else:
            recs[-1][2] = ev

    for rep in range(a.reps):
        recs.clear()
        _lib.entry_hook = hook
        res = eng.prefill(store, a.turn, ro, n_new)
        eng.decode(store, ro + n_new, a.decode)
        torch.cuda.synchronize()
        _lib.entry_hook = None
        per = {}
        for name, e0, e1 in recs:
            per.setdefault(name, []).append(e0.elapsed_time(e1))
    for k, v in per.items():
        print(f"{k:28s} n={len(v):4d} total={sum(v):9.3f} ms  mean={sum(v)/len(v):8.4f} ms")
    p = res.plans[0]
    cn = p.counts.cpu().numpy()
    npk = p.n_picks.cpu().numpy()
    print("plan sizes (S, V) per head:", [tuple(x) for x in cn[:8]], "...")
    print("final picks per head:", npk[:8].tolist())
    print("coverage:", p.coverage.cpu().numpy()[:8].round(4).tolist())
    print("cells per head:", res.cells[0].cpu().numpy()[:8].tolist(),
          "dense cells/head:", n_new * ro + n_new * (n_new + 1) // 2)


if __name__ == "__main__":
    main()
