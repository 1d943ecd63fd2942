"""Synthetic attention inputs with planted vertical/slash structure.

The generator of SURVEY.md section 8(d), defined in logit units:
  * background q, k, v ~ N(0, 1)^d;
  * slash structure: F=16 phase features, w_k ~ U(0.5, pi),
    a = sqrt(b_loc * sqrt(d) / 16), ph(p) = a [cos(w p), sin(w p)] added to
    dims [0, 32) of q_p and k_p, so the logit gains b_loc * mean_k cos(w_k (i-j))
    (exactly b_loc on the diagonal);
  * vertical structure on u = e_{d-1}: every q gets +s_q (s_q = 4); 16 hot
    keys per KV head, drawn without replacement from [1, n_ref), get
    +b_hot sqrt(d)/s_q and key 0 (the sink) +b_sink sqrt(d)/s_q, i.e. logit
    boosts b_hot / b_sink;
  * the q-heads of a GQA group share the group's structure, noise is
    independent;
  * everything is rounded to bf16.
Boosts follow the survey calibration (b_loc, b_hot, b_sink) =
(12, 9, 12) + 1.5 ln(n_ref / 2000).

Q, K, V of a position do not depend on the turn, so a decode row and the
re-prefilled answer row at the same position are the same (session.py:122,180).

Two back ends with the same formula: numpy (PCG64; used for parity fixtures,
deterministic across machines) and torch on the device (for bench-scale
inputs). They do not produce the same numbers.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

N_FEAT = 16
S_Q = 4.0
N_HOT = 16


@dataclass(frozen=True)
class SynthSpec:
    n_q: int
    n_kv: int
    d: int
    n_pos: int            # positions generated: [0, n_pos)
    n_ref: int | None = None  # calibration length (defaults to n_pos)
    structured: bool = True
    seed: int = 0
    kv_offset: int = 0    # global index of local kv-head 0 (head-sharded runs draw the same data)

    def boosts(self):
        n_ref = self.n_ref or self.n_pos
        extra = 1.5 * math.log(max(n_ref, 1) / 2000.0)
        return 12.0 + extra, 9.0 + extra, 12.0 + extra


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as float32 values."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = ((u + 0x7FFF + lsb) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def bf16_bits(x32: np.ndarray) -> np.ndarray:
    """float32 values that are exact bf16 -> uint16 bit patterns."""
    return (np.ascontiguousarray(x32, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


def _rng(seed: int, *key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed, spawn_key=key)))


def layer_qkv_numpy(spec: SynthSpec, layer: int):
    """-> (Q [n_q, n_pos, d], K [n_kv, n_pos, d], V [n_kv, n_pos, d]) float32 bf16-exact."""
    d, n = spec.d, spec.n_pos
    group = spec.n_q // spec.n_kv
    b_loc, b_hot, b_sink = spec.boosts()
    Q = np.empty((spec.n_q, n, d), np.float32)
    K = np.empty((spec.n_kv, n, d), np.float32)
    V = np.empty((spec.n_kv, n, d), np.float32)
    p = np.arange(n, dtype=np.float64)
    n_ref = spec.n_ref or n
    for g in range(spec.n_kv):
        srng = _rng(spec.seed, layer, g, 0)
        k = srng.standard_normal((n, d))
        v = srng.standard_normal((n, d))
        if spec.structured:
            omega = srng.uniform(0.5, math.pi, size=N_FEAT)
            a = math.sqrt(b_loc * math.sqrt(d) / N_FEAT)
            ph = np.concatenate([np.cos(p[:, None] * omega[None, :]),
                                 np.sin(p[:, None] * omega[None, :])], axis=1) * a
            nf = min(2 * N_FEAT, d - 1)
            k[:, :nf] += ph[:, :nf]
            hot = srng.choice(np.arange(1, max(n_ref, 2)), size=min(N_HOT, max(n_ref - 1, 1)),
                              replace=False)
            hot = hot[hot < n]
            k[hot, d - 1] += b_hot * math.sqrt(d) / S_Q
            k[0, d - 1] += b_sink * math.sqrt(d) / S_Q
        K[g] = bf16_round(k)
        V[g] = bf16_round(v)
        for j in range(group):
            qrng = _rng(spec.seed, layer, g, 1 + j)
            q = qrng.standard_normal((n, d))
            if spec.structured:
                q[:, :nf] += ph[:, :nf]
                q[:, d - 1] += S_Q
            Q[g * group + j] = bf16_round(q)
    return Q, K, V


def layer_qkv_torch(spec: SynthSpec, layer: int, device="cuda"):
    """Device generator, same formula (different random numbers): bf16 tensors
    Q [n_q, n_pos, d], K/V [n_kv, n_pos, d]. Every (layer, global kv head)
    has its own generator, so a head-sharded rank (kv_offset = its first kv
    head) draws exactly the heads an unsharded run would."""
    import torch

    d, n = spec.d, spec.n_pos
    group = spec.n_q // spec.n_kv
    b_loc, b_hot, b_sink = spec.boosts()
    n_ref = spec.n_ref or n
    nf = min(2 * N_FEAT, d - 1)
    p = torch.arange(n, device=device, dtype=torch.float64)
    a = math.sqrt(b_loc * math.sqrt(d) / N_FEAT)
    Q = torch.empty((spec.n_q, n, d), device=device, dtype=torch.bfloat16)
    K = torch.empty((spec.n_kv, n, d), device=device, dtype=torch.bfloat16)
    V = torch.empty((spec.n_kv, n, d), device=device, dtype=torch.bfloat16)
    for g in range(spec.n_kv):
        gg = spec.kv_offset + g
        gen = torch.Generator(device=device)
        gen.manual_seed((spec.seed * 1_000_003 + layer * 7919 + gg * 104_729 + 17) & 0x7FFFFFFFFFFFFFFF)
        k = torch.randn((n, d), generator=gen, device=device, dtype=torch.float32)
        v = torch.randn((n, d), generator=gen, device=device, dtype=torch.float32)
        q = torch.randn((group, n, d), generator=gen, device=device, dtype=torch.float32)
        if spec.structured:
            omega = torch.rand(N_FEAT, generator=gen, device=device, dtype=torch.float64) * (math.pi - 0.5) + 0.5
            ang = p[:, None] * omega[None, :]
            ph = (torch.cat([torch.cos(ang), torch.sin(ang)], dim=1) * a).to(torch.float32)[:, :nf]
            k[:, :nf] += ph
            q[:, :, :nf] += ph[None]
            perm = torch.randperm(max(n_ref - 1, 1), generator=gen, device=device)[:N_HOT] + 1
            perm = perm[perm < n]
            k[perm, d - 1] += b_hot * math.sqrt(d) / S_Q
            k[0, d - 1] += b_sink * math.sqrt(d) / S_Q
            q[:, :, d - 1] += S_Q
        K[g] = k.to(torch.bfloat16)
        V[g] = v.to(torch.bfloat16)
        Q[g * group:(g + 1) * group] = q.to(torch.bfloat16)
    return Q, K, V


def checksum(*arrays) -> str:
    import hashlib

    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]
