"""Frame-range sharding across GPUs and the end-of-run counter reduction
(SURVEY §8(e)).

The reference's Monte-Carlo engine claims frames from one global index space
and keys every frame's randomness by (seed, global frame index)
(sim.cpp:84-109, channel.hpp:13-22), so error counts do not depend on the
worker count (test_sim.cpp:37-66).  Across GPUs the same holds by
construction: rank r of W decodes global frames [frame0 + r*F, frame0 +
(r+1)*F) with no traffic on the decode path, and the only collective is one
SUM of four u64 counters per (SNR point), as in Acc::merge (sim.cpp:25-31).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def frame_range(rank: int, world: int, frames_per_rank: int, frame0: int = 0):
    """Weak scaling: a fixed per-rank batch, contiguous global ranges."""
    assert 0 <= rank < world
    start = frame0 + rank * frames_per_rank
    return start, start + frames_per_rank


def split_range(rank: int, world: int, total: int, frame0: int = 0):
    """Strong scaling: a fixed global set split into near-equal ranges."""
    a = frame0 + total * rank // world
    b = frame0 + total * (rank + 1) // world
    return a, b


@dataclass
class Counters:
    """PointStats counters (sim.hpp:30-41) that survive the reduction."""
    frames: int = 0
    bit_errors: int = 0
    frame_errors: int = 0
    esc_sum: int = 0

    def add_batch(self, payload_bits: np.ndarray, info: np.ndarray, esc: np.ndarray, ks=None):
        """run_frame's counting (sim.cpp:66-71): bit errors on the first K
        payload bits, a frame error if any (ks: per-frame K of a mixed batch)."""
        k = info.shape[1]
        diff = payload_bits[:, :k] != info
        if ks is not None:
            diff &= np.arange(k)[None, :] < np.asarray(ks)[:, None]
        be = diff.sum(1)
        self.frames += int(info.shape[0])
        self.bit_errors += int(be.sum())
        self.frame_errors += int((be > 0).sum())
        self.esc_sum += int(np.asarray(esc, np.int64).sum())

    def as_array(self):
        return np.array([self.frames, self.bit_errors, self.frame_errors, self.esc_sum], np.int64)

    @staticmethod
    def from_array(a):
        return Counters(int(a[0]), int(a[1]), int(a[2]), int(a[3]))

    def fer(self):
        return self.frame_errors / self.frames if self.frames else 0.0

    def ber(self, k: int):
        return self.bit_errors / (k * self.frames) if self.frames else 0.0


def all_reduce_counters(c: Counters, device=None) -> Counters:
    """One SUM of 4 x i64 over the default process group (nccl or gloo)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        return c
    t = torch.tensor(c.as_array(), dtype=torch.int64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return Counters.from_array(t.cpu().numpy())


def binomial_ci95(errors: int, frames: int):
    """sim.cpp:176-183 (normal approximation, clamped)."""
    if frames == 0:
        return 0.0, 1.0
    p = errors / frames
    half = 1.96 * np.sqrt(max(p * (1 - p), 0.0) / frames)
    return max(0.0, p - half), min(1.0, p + half)
