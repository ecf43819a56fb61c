"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the FlatQuant method (no transform, no
quantizer, no GEMM).  It only draws random inputs with the shapes and value
distributions of the paper's workloads (DESIGN.md §"Input recipe"):

* activations X [T, n]: N(0,1) with 1% "channel outliers" scaled x50
  (Fig.1 "channel-wise outliers") and a "pivot token" 0 whose 4
  channels are scaled x400 ("massive outliers ... pivot tokens"),
  clamped to +-60000 and rounded to the compute dtype (fp16 by default, the
  paper's activation precision);
* transforms P1 [n1,n1], P2 [n2,n2]: U diag(exp(sigma)) V^T with Haar-random
  orthogonal U, V and sigma ~ U(-0.5, 0.5) (cond <= e), mirroring the SVD
  parameterisation of App. B.1 and the random initialisation of
  PAPER.md:363;
* weights W [N, K]: N(0, 1/K);
* special transforms for the pins: identity, scalar, permutation, Sylvester
  Hadamard (PAPER.md:177-180 uses Hadamards as the QuaRot transform).

Every stream is a counter-based Philox generator keyed by
(seed, tag, *shape) so that every rank (and the oracle and the GPU side)
regenerates identical data without communication.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

__all__ = [
    "rng", "activations", "well_conditioned", "weights", "hadamard", "permutation",
    "random_codes", "random_scales", "Linear", "CONFIGS", "config",
]


def _key(seed: int, tag: str, *extra) -> int:
    h = hashlib.sha256(repr((int(seed), str(tag)) + tuple(int(e) for e in extra)).encode()).digest()
    return int.from_bytes(h[:16], "little")


def rng(seed: int, tag: str, *extra) -> np.random.Generator:
    """Counter-based (Philox) generator keyed by (seed, tag, extra...)."""
    return np.random.Generator(np.random.Philox(key=_key(seed, tag, *extra)))


ROW_BLOCK = 256


def activations(T: int, n: int, seed: int = 0, tag: str = "x", dtype=np.float16,
                outlier_frac: float = 0.01, outlier_scale: float = 50.0,
                pivot_channels: int = 4, pivot_scale: float = 400.0,
                clamp: float = 60000.0, rows=None) -> np.ndarray:
    """Gaussian activations with channel outliers and one pivot token (token 0).

    Rows are drawn in blocks of ROW_BLOCK from streams keyed by (seed, tag, n, block), so
    row t is the same for every T and any subset `rows` can be regenerated on its own
    (the oracle re-derives sampled tokens of a large workload this way).
    """
    idx = np.arange(T) if rows is None else np.asarray(rows, dtype=np.int64)
    out = np.empty((idx.size, n), dtype=dtype)
    if n == 0 or idx.size == 0:
        return out
    go = rng(seed, tag + "/outlier_channels", n)      # fixed per layer
    k = max(1, int(round(outlier_frac * n))) if outlier_frac > 0 else 0
    ch = go.choice(n, size=k, replace=False) if k else np.zeros(0, np.int64)
    pc = go.choice(n, size=min(pivot_channels, n), replace=False) if pivot_channels > 0 else np.zeros(0, np.int64)
    blocks = np.unique(idx // ROW_BLOCK)
    pos = {}
    for i, r in enumerate(idx):
        pos.setdefault(int(r) // ROW_BLOCK, []).append((i, int(r) % ROW_BLOCK))
    for b in blocks:
        g = rng(seed, tag + "/x", n, int(b))
        blk = g.standard_normal((ROW_BLOCK, n), dtype=np.float32)
        if k:
            blk[:, ch] *= outlier_scale
        if b == 0 and pc.size:
            blk[0, pc] *= pivot_scale
        np.clip(blk, -clamp, clamp, out=blk)
        sel = pos[int(b)]
        out[[i for i, _ in sel]] = blk[[j for _, j in sel]].astype(dtype)
    return out


def _haar_orthogonal(g: np.random.Generator, n: int) -> np.ndarray:
    a = g.standard_normal((n, n))
    q, r = np.linalg.qr(a)
    return q * np.sign(np.diag(r))[None, :]


def well_conditioned(n: int, seed: int = 0, tag: str = "p", dtype=np.float16,
                     sigma_range: float = 0.5) -> np.ndarray:
    """Random invertible U diag(exp(s)) V^T, s ~ U(-sigma_range, sigma_range)."""
    g = rng(seed, tag + "/p", n)
    u = _haar_orthogonal(g, n)
    v = _haar_orthogonal(g, n)
    s = np.exp(g.uniform(-sigma_range, sigma_range, size=n))
    return ((u * s[None, :]) @ v.T).astype(dtype)


def weights(N: int, K: int, seed: int = 0, tag: str = "w", dtype=np.float16) -> np.ndarray:
    g = rng(seed, tag + "/w", N, K)
    return (g.standard_normal((N, K)) / np.sqrt(K)).astype(dtype)


def hadamard(n: int, dtype=np.float64) -> np.ndarray:
    """Normalised Sylvester Hadamard matrix H_n (n a power of two), H^T H = I."""
    if n < 1 or (n & (n - 1)) != 0:
        raise ValueError("hadamard: n must be a power of two")
    h = np.ones((1, 1))
    while h.shape[0] < n:
        h = np.block([[h, h], [h, -h]])
    return (h / np.sqrt(n)).astype(dtype)


def permutation(n: int, seed: int = 0, tag: str = "perm", dtype=np.float64) -> np.ndarray:
    g = rng(seed, tag + "/perm", n)
    p = np.zeros((n, n))
    p[np.arange(n), g.permutation(n)] = 1.0
    return p.astype(dtype)


def random_codes(rows: int, cols: int, seed: int = 0, tag: str = "codes") -> np.ndarray:
    """Uniform INT4 codes in [-8, 7] as int8 (used to feed the integer GEMM directly)."""
    g = rng(seed, tag + "/codes", rows, cols)
    return g.integers(-8, 8, size=(rows, cols), dtype=np.int8)


def random_scales(n: int, seed: int = 0, tag: str = "scales") -> np.ndarray:
    g = rng(seed, tag + "/scales", n)
    return (g.uniform(0.5, 2.0, size=n) * 1e-2).astype(np.float32)


# ---------------------------------------------------------------------------
# Workload table (BASELINE.json "configs"; shapes per SURVEY.md §8(a))
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Linear:
    name: str      # which activation feeds it (paper notation P_a, P_o, P_ug, P_d)
    n1: int
    n2: int
    N: int         # GEMM output features

    @property
    def K(self) -> int:
        return self.n1 * self.n2


CONFIGS = {
    # configs[0]: tiny parity case
    "C1": dict(desc="single linear 512 (16x32) -> 512, 32 tokens", T=32,
               linears=(Linear("P_a", 16, 32, 512),)),
    # configs[1]: LLaMA-2-7B q_proj
    "C2": dict(desc="LLaMA-2-7B q_proj 4096 (64x64) -> 4096, prefill 2048 tokens", T=2048,
               linears=(Linear("P_a", 64, 64, 4096),)),
    # configs[2]: LLaMA-3-8B layer linears (qkv fused N, gate+up fused N)
    "C3": dict(desc="LLaMA-3-8B layer linears, prefill 2048 tokens", T=2048,
               linears=(Linear("P_a", 64, 64, 6144), Linear("P_o", 64, 64, 4096),
                        Linear("P_ug", 64, 64, 28672), Linear("P_d", 112, 128, 4096))),
    # configs[3]: LLaMA-3-8B decode, batch 64 x 1 token
    "C4": dict(desc="LLaMA-3-8B decode, batch 64 x 1 token, all layer linears", T=64,
               linears=(Linear("P_a", 64, 64, 6144), Linear("P_o", 64, 64, 4096),
                        Linear("P_ug", 64, 64, 28672), Linear("P_d", 112, 128, 4096))),
    # configs[4]: LLaMA-3-70B linears, 16 x 2048 tokens (sharded over GPUs)
    "C5": dict(desc="LLaMA-3-70B linears, prefill 16x2048 tokens", T=32768,
               linears=(Linear("P_a", 64, 128, 10240), Linear("P_o", 64, 128, 8192),
                        Linear("P_ug", 64, 128, 57344), Linear("P_d", 128, 224, 8192))),
}


def config(name: str) -> dict:
    return CONFIGS[name]
