"""Counter-based splittable RNG (host side).

Same streams as the reference's ``tilecast.rng``
(/root/reference/pkg/src/tilecast/rng.py:18-93): a state is a ``(key,
counter)`` pair of u64; a draw finalises ``key + counter * GOLDEN`` with the
splitmix64 mixer; ``split`` salts the key with the child index. On the device
the same arithmetic lives in ``csrc/tilecast_b200.cu`` (``tc_seed_streams``,
``tc_policy_actions`` and the in-kernel reset draws); the host versions here
serve the scalar API and the tests.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
SPLIT_SALT = 0x3C6EF372FE94F82A
POLICY_STREAM = M64  # batch.py:150: the policy stream is split index 2**64-1


class RngState(NamedTuple):
    key: int
    counter: int


def mix(x: int) -> int:
    """splitmix64 finaliser on a wrapped u64 (rng.py:26-33)."""
    x &= M64
    x = ((x ^ (x >> 30)) * MIX1) & M64
    x = ((x ^ (x >> 27)) * MIX2) & M64
    return x ^ (x >> 31)


def from_seed(seed: int) -> RngState:
    return RngState(mix(seed & M64), 0)


def next_u64(state: RngState) -> tuple[int, RngState]:
    return (mix(state.key + state.counter * GOLDEN),
            RngState(state.key, (state.counter + 1) & M64))


def next_below(state: RngState, n: int) -> tuple[int, RngState]:
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    u, nxt = next_u64(state)
    return (u * n) >> 64, nxt


def split(state: RngState, index: int) -> RngState:
    return RngState(mix(state.key + SPLIT_SALT + (index & M64) * GOLDEN), 0)


def policy_key(seed: int) -> int:
    """Key of the dedicated action stream of a seeded rollout (batch.py:150)."""
    return split(from_seed(seed), POLICY_STREAM).key


def _mix_u64(x: np.ndarray) -> np.ndarray:
    x = x ^ (x >> np.uint64(30))
    x = x * np.uint64(MIX1)
    x = x ^ (x >> np.uint64(27))
    x = x * np.uint64(MIX2)
    return x ^ (x >> np.uint64(31))


def _mulhi_u64(x: np.ndarray, n: int) -> np.ndarray:
    """floor(x * n / 2**64) for u64 arrays via 32-bit limbs."""
    lo32 = np.uint64(0xFFFFFFFF)
    s32 = np.uint64(32)
    xl, xh = x & lo32, x >> s32
    nl, nh = np.uint64(n & 0xFFFFFFFF), np.uint64(n >> 32)
    ll, lh, hl, hh = xl * nl, xl * nh, xh * nl, xh * nh
    carry = ((ll >> s32) + (lh & lo32) + (hl & lo32)) >> s32
    return hh + (lh >> s32) + (hl >> s32) + carry


def policy_uniform(key: int, counters: np.ndarray, n: int) -> np.ndarray:
    """Vectorised ``next_below`` over counters of one stream (rng.py:62-93)."""
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    with np.errstate(over="ignore"):
        x = np.uint64(key) + counters.astype(np.uint64) * np.uint64(GOLDEN)
        return _mulhi_u64(_mix_u64(x), n).astype(np.int64)


def seed_streams(seed: int, base: int, n: int) -> tuple[np.ndarray, np.ndarray]:
    """Vectorised ``split(from_seed(seed), base + i)`` keys (batch.py:81-85)."""
    root = np.uint64(from_seed(seed).key)
    idx = np.arange(base, base + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        keys = _mix_u64(root + np.uint64(SPLIT_SALT) + idx * np.uint64(GOLDEN))
    return keys, np.zeros(n, dtype=np.uint64)
