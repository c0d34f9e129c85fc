"""The reference's deterministic generator (``proj/core/include/radonkit/rng.hpp:13-38``):
raw ``std::mt19937`` words (seeded with ``uint32(seed ^ (seed >> 32))``) mapped
to [0, 1) as ``float(word >> 8) * 2^-24``.

std::mt19937's seeding recurrence is restated here; the tempered output is
produced by numpy's MT19937 bit generator after loading that state (the same
standard algorithm), so long draws are vectorised.
"""
from __future__ import annotations

import numpy as np


def _mt19937_key(seed32: int) -> np.ndarray:
    key = np.empty(624, np.uint32)
    x = seed32 & 0xFFFFFFFF
    key[0] = x
    for i in range(1, 624):
        x = (1812433253 * (x ^ (x >> 30)) + i) & 0xFFFFFFFF
        key[i] = x
    return key


class Rng:
    """rng.hpp:13-38."""

    def __init__(self, seed: int):
        seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self._bg = np.random.MT19937(0)
        self._bg.state = {"bit_generator": "MT19937", "state": {"key": _mt19937_key((seed ^ (seed >> 32)) & 0xFFFFFFFF),
                                                                "pos": 624}}

    def raw(self, n: int) -> np.ndarray:
        return self._bg.random_raw(int(n)).astype(np.uint32)

    def uniform(self, n: int = 1) -> np.ndarray:
        """[0, 1) as float32: float(eng() >> 8) * 0x1.0p-24f."""
        return (self.raw(n) >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)

    def uniform_pm1(self, n: int = 1) -> np.ndarray:
        """[-1, 1): 2.0f * uniform() - 1.0f (float arithmetic)."""
        return np.float32(2.0) * self.uniform(n) - np.float32(1.0)

    def uniform_tensor(self, shape, dtype=np.float32) -> np.ndarray:
        n = int(np.prod(shape))
        return self.uniform(n).astype(dtype).reshape(shape)

    def uniform_pm1_tensor(self, shape, dtype=np.float32) -> np.ndarray:
        n = int(np.prod(shape))
        return self.uniform_pm1(n).astype(dtype).reshape(shape)
