"""Rollout digest in the order SURVEY.md §8(c) fixes (state arrays, then
rewards, dones, truncs, events, frames), shared by oracle and CUDA tests."""

from __future__ import annotations

import hashlib

import numpy as np

STATE_ORDER = ("px", "py", "dx", "dy", "health", "inv", "t", "rctr", "done", "agoal",
               "dopen", "ealive")


class Digest:
    def __init__(self):
        self.h = hashlib.blake2b(digest_size=16)
        self.reward_sum = 0.0
        self.dones = 0
        self.events_or = 0

    def frames(self, frames: np.ndarray) -> None:
        self.h.update(np.ascontiguousarray(frames).tobytes())

    def step(self, state: dict, rewards, dones, truncs, events, frames) -> None:
        for k in STATE_ORDER:
            self.h.update(np.ascontiguousarray(state[k]).tobytes())
        rewards = np.asarray(rewards, dtype=np.float64)
        dones = np.asarray(dones) != 0
        self.h.update(rewards.tobytes())
        self.h.update(dones.tobytes())
        self.h.update(np.asarray(truncs, dtype=np.uint8).tobytes())
        self.h.update(np.asarray(events, dtype=np.uint32).tobytes())
        self.frames(frames)
        self.reward_sum += float(rewards.sum())
        self.dones += int(dones.sum())
        self.events_or |= int(np.bitwise_or.reduce(np.asarray(events, dtype=np.uint32)))

    def hexdigest(self) -> str:
        return self.h.hexdigest()
