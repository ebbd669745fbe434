"""Digests for full-size oracle parity (TEST INFRASTRUCTURE, no arithmetic of the method).

At BASELINE.json's full sizes the oracle needs minutes per config (c4: ~10 min on 8
cores), too long to rerun inside ``pytest -m gpu``.  ``tests/golden/make_fullsize.py``
runs the oracle once -- it calls only ``oracle/`` and ``synth/`` -- and stores, per
config, SHA-256 digests of every output the oracle produces on the whole field (ranks,
C_0..C_d, D0, D_{d-1}, both unpaired-saddle lists) and an order-independent multiset
digest of the gradient vectors of fixed vertex chunks.  ``tests/test_gpu_fullsize_oracle.py``
computes the same digests from the CUDA path's outputs: equal digests <=> equal arrays
(element by element, up to SHA-256 / 64-bit multiset-hash collisions).  The field bytes
are digested too; if the GPU box generated a different field, the test reruns the
oracle live instead.
"""
from __future__ import annotations

import hashlib

import numpy as np

CFGS = ["c3", "c4", "c5a", "c5b"]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)


def _mix(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser, vectorised (uint64 wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        x = x + _G
        x = (x ^ (x >> np.uint64(30))) * _M1
        x = (x ^ (x >> np.uint64(27))) * _M2
        return x ^ (x >> np.uint64(31))


def multiset_digest(triples: np.ndarray) -> list:
    """Order-independent digest of (n, 3) int64 rows: [count, sum mod 2^64, xor]."""
    t = np.ascontiguousarray(triples, dtype=np.int64).view(np.uint64).reshape(-1, 3)
    if len(t) == 0:
        return [0, 0, 0]
    h = _mix(t[:, 0] ^ _mix(t[:, 1] ^ _mix(t[:, 2])))
    with np.errstate(over="ignore"):
        s = np.add.reduce(h, dtype=np.uint64)
    x = np.bitwise_xor.reduce(h)
    return [int(len(t)), int(s), int(x)]


def gradient_chunks(cfg: str, shape) -> list:
    """Vertex chunks whose gradient vectors are compared: every vertex for c3 / c5a /
    c5b; for c4 the six boundary faces plus 16 interior planes (5.8 M vertices).
    Each chunk is a list of (v0, v1) runs of consecutive vertex ids."""
    N = int(np.prod(shape))
    if cfg != "c4":
        step = {"c3": 1 << 20, "c5a": 1 << 23, "c5b": 1 << 24}[cfg]
        return [[(v, min(N, v + step))] for v in range(0, N, step)]
    Lz, Ly, Lx = shape
    P = Lx * Ly
    chunks = [[(0, P)], [((Lz - 1) * P, Lz * P)]]                      # z = 0, z = Lz-1
    chunks.append([(z * P, z * P + Lx) for z in range(Lz)])             # y = 0
    chunks.append([(z * P + (Ly - 1) * Lx, z * P + Ly * Lx) for z in range(Lz)])  # y = Ly-1
    # x = 0 and x = Lx-1: single vertices per row
    chunks.append([(z * P + y * Lx, z * P + y * Lx + 1) for z in range(Lz) for y in range(Ly)])
    chunks.append([(z * P + y * Lx + Lx - 1, z * P + y * Lx + Lx) for z in range(Lz) for y in range(Ly)])
    z0 = Lz // 2 - 8
    for i in range(4):
        chunks.append([((z0 + 4 * i) * P, (z0 + 4 * i + 4) * P)])
    return chunks


def chunk_vertices(chunk) -> np.ndarray:
    return np.concatenate([np.arange(a, b, dtype=np.int64) for a, b in chunk])
