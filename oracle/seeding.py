"""Row sampling and per-head seeds (oracle; test infrastructure only).

Restates:
  * `Session.head_seed`      -- reference session.py:84-86
  * `sample_rows`            -- reference prefill.py:125-135
The bits are defined by numpy's SeedSequence / PCG64 / Generator.choice, so the
restatement calls numpy exactly as the reference does (numpy version is
recorded with every golden file).
"""

from __future__ import annotations

import math

import numpy as np


class EmptyBlock(Exception):
    pass


def head_seed(session_seed: int, turn: int, layer: int, head: int) -> int:
    """session.py:84-86."""
    ss = np.random.SeedSequence(entropy=session_seed, spawn_key=(turn, layer, head))
    return int(ss.generate_state(1, dtype=np.uint64)[0])


def sample_size(n_new: int, rate: float, floor: int) -> int:
    """prefill.py:132."""
    return min(n_new, max(floor, math.ceil(rate * n_new)))


def sample_rows(n_new: int, rate: float, floor: int, seed: int) -> np.ndarray:
    """prefill.py:125-135: sorted uniform sample, last row always included."""
    if n_new <= 0:
        raise EmptyBlock("cannot sample rows of an empty block")
    if not (0.0 < rate <= 1.0) or floor < 1:
        raise ValueError("need 0 < rate <= 1 and floor >= 1")
    size = sample_size(n_new, rate, floor)
    rng = np.random.Generator(np.random.PCG64(seed))
    rest = rng.choice(n_new - 1, size=size - 1, replace=False) if size > 1 else []
    return np.sort(np.append(np.asarray(rest, dtype=np.intp), n_new - 1))


def turn_rows(n_new: int, alpha: float, rate: float, floor: int, session_seed: int,
              turn: int, layer: int, head: int) -> np.ndarray:
    """The sparsifier closure's row policy, session.py:135-144."""
    if alpha >= 1.0:
        return np.arange(n_new)
    return sample_rows(n_new, rate, floor, head_seed(session_seed, turn, layer, head))
