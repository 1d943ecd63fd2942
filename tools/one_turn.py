"""One C2 turn-3 prefill + its 128-token decode (no warm-up): the workload the
committed ncu launch list is taken on (tools/gpu_round.sh launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
from paper_2507_13681_b200.kvcompress import CompressionConfig

shape = AttnShape(32, 32, 8, 128)
cap = 3 * 5128
store = QKVStore.synthetic(shape, cap, n_ref=cap, seed=1)
eng = SessionEngine(shape, SessionParams(alpha=0.955, comp=CompressionConfig(1024, 16, 16), max_new=128), cap)
eng.prefill(store, 2, 10128, 5128)
eng.decode(store, 15256, 128)
torch.cuda.synchronize()
print("ok")
