"""Deterministic inputs: the reference's counter-based generator.

Vectorised numpy restatement of uniform_at / fill_uniform
(/root/reference/proj/include/fftconv/rng.hpp:21-47) so that benchmark and
test inputs are byte-identical to what the reference CPU path consumes for
the same (seed, role).  Roles: input=1, weights=2, grad_output=3
(rng.hpp:11-17).
"""
from __future__ import annotations

import numpy as np

ROLE_INPUT = 1
ROLE_WEIGHTS = 2
ROLE_GRAD_OUTPUT = 3

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _splitmix64(z):
    with np.errstate(over="ignore"):
        z = z + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def splitmix64(z: int) -> int:
    return int(_splitmix64(np.uint64(z)))


def uniform_at(seed: int, role: int, index) -> np.ndarray:
    """rng.hpp:32-37: element `index` of the (seed, role) stream, in [-1, 1)."""
    key = _splitmix64(np.uint64(seed) ^ _splitmix64(np.uint64(role)))
    h = _splitmix64(key ^ np.asarray(index, dtype=np.uint64))
    return 2.0 * ((h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) - 1.0


def fill_uniform(shape, seed: int, role: int, stream: int = 0, dtype=np.float32, offset: int = 0) -> np.ndarray:
    """rng.hpp:41-47: static_cast<T> of the double draw, in index order.
    `offset` starts at element `offset` of the stream (a slice of a larger
    tensor, e.g. one rank's minibatch shard, without generating the rest)."""
    n = int(np.prod(shape))
    r = int(role) | (int(stream) << 8)
    out = np.empty(n, dtype=dtype)
    chunk = 1 << 22
    for s in range(0, n, chunk):
        idx = np.arange(offset + s, offset + min(n, s + chunk), dtype=np.uint64)
        out[s:s + len(idx)] = uniform_at(seed, r, idx).astype(dtype)
    return out.reshape(shape)
