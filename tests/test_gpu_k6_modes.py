"""The decode kernel's alternative launch modes agree with the default one.

K6 chooses its split-K combine at launch (cluster DSMEM for compressed steps,
last-CTA global combine for dense steps) and keeps the CUDA-core kernel as a
cross-check; the alternatives are selected by environment variables read once
per process, so each runs in its own subprocess on the same seeded dialogue."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2507_13681_b200.engine import AttnShape, QKVStore, SessionEngine, SessionParams
from paper_2507_13681_b200.kvcompress import CompressionConfig
shape = AttnShape(2, 8, 2, 128)
n_new, max_new = 1500, 40
store = QKVStore.synthetic(shape, n_new + max_new, n_ref=n_new + max_new, seed=11)
eng = SessionEngine(shape, SessionParams(alpha=0.9, comp=CompressionConfig(256, 8, 8), max_new=max_new, seed=4),
                    n_new + max_new)
eng.prefill(store, 0, 0, n_new)
outs = []
eng.decode(store, n_new, max_new, out_sink=lambda t, ob: outs.append(ob.float().cpu().numpy().copy()))
torch.cuda.synchronize()
np.save(sys.argv[2], np.stack(outs))
np.save(sys.argv[2].replace('.npy', '_sel.npy'), eng.stack.sel_ids.cpu().numpy())
"""


def _run(tmp_path, name, env_extra):
    out = str(tmp_path / f"{name}.npy")
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, out], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out), np.load(out.replace(".npy", "_sel.npy"))


@pytest.mark.parametrize("mode", [{"LS_K6_ALL_CTA": "1"}, {"LS_K6_NO_CLUSTER": "1"}, {"LS_K6_SIMT": "1"},
                                  {"LS_K6_SPLIT_DENSE": "5", "LS_K6_SPLIT_COMP": "3"}],
                         ids=lambda m: json.dumps(m))
def test_k6_modes_agree(cuda_lib, tmp_path, mode):
    ref, ref_sel = _run(tmp_path, "default", {})
    got, sel = _run(tmp_path, "mode", mode)
    assert np.isfinite(got).all()
    # different split counts / combine orders: bf16 outputs agree to rounding
    # (the attention parity bar is 2e-2 abs)
    assert np.abs(got - ref).max() < 2e-2, float(np.abs(got - ref).max())
    # the compression events select from the same logits up to rounding: the
    # retained sets agree except at near-ties
    agree = np.mean(sel == ref_sel)
    assert agree > 0.99, agree
