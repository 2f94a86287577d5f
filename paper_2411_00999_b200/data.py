"""Synthetic token stream of the reference trainer (host side).

A restatement of gnstk's portable RNG (proj/include/gnstk/rng.hpp:11-66) and
its MarkovDataset (proj/include/gnstk/dataset.hpp:13-45,
proj/src/dataset.cpp:19-80): a first-order Markov chain over V tokens whose
transition rows are normalised squared Gaussians.  The same seed gives the
same stream bit for bit (pinned against the reference in
tests/golden/trainer_cases.json), so the GPU trainer consumes exactly the
sequences the reference trainer does.  This is the trainer's data loader; it
is not on the kernel path.
"""
from __future__ import annotations

import math
from typing import List

import numpy as np

_M64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
_TRANSITION_TAG = 0x7472616E73  # dataset.cpp:15
_SEQUENCE_TAG = 0x73657175      # dataset.cpp:16


class SplitMix64:
    """rng.hpp:11-37: Weyl counter + avalanche finaliser."""

    def __init__(self, seed: int):
        self.state = seed & _M64

    def next(self) -> int:
        self.state = (self.state + _GOLDEN) & _M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def next_unit(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -53

    def next_unit_open(self) -> float:
        return float((self.next() >> 11) + 1) * 2.0 ** -53

    def next_below(self, n: int) -> int:
        v = int(self.next_unit() * float(n))
        return n - 1 if v >= n else v


def mix_seed(seed: int, tag: int) -> int:
    """rng.hpp:40-43."""
    return SplitMix64((seed ^ ((_GOLDEN * (tag + 1)) & _M64)) & _M64).next()


class GaussianStream:
    """rng.hpp:46-66: Box-Muller on SplitMix64 (cos first, sin as the spare)."""

    def __init__(self, seed: int):
        self.rng = SplitMix64(seed)
        self.spare = None

    def next(self) -> float:
        if self.spare is not None:
            s, self.spare = self.spare, None
            return s
        u1 = self.rng.next_unit_open()
        u2 = self.rng.next_unit()
        r = math.sqrt(-2.0 * math.log(u1))
        a = 2.0 * 3.14159265358979323846 * u2
        self.spare = r * math.sin(a)
        return r * math.cos(a)

    def draw(self, n: int) -> np.ndarray:
        return np.array([self.next() for _ in range(n)], dtype=np.float64)


class MarkovDataset:
    """dataset.cpp:19-80."""

    def __init__(self, vocab: int, seed: int):
        if vocab < 2:
            raise ValueError("dataset: vocab must be >= 2")
        self.vocab = int(vocab)
        self.stream = SplitMix64(mix_seed(seed, _SEQUENCE_TAG))
        gen = GaussianStream(mix_seed(seed, _TRANSITION_TAG))
        t = np.empty((vocab, vocab), dtype=np.float64)
        for r in range(vocab):
            w = [0.0] * vocab
            total = 0.0
            for c in range(vocab):  # sequential sum, as the reference
                z = gen.next()
                w[c] = z * z
                total += w[c]
            if total <= 0.0:
                total = 1.0
            t[r] = [v / total for v in w]
        self.transition = t
        self._cdf = []
        for r in range(vocab):
            acc, row = 0.0, []
            for c in range(vocab):
                acc += t[r, c]
                row.append(acc)
            row[-1] = 1.0
            self._cdf.append(row)

    def fill_sequence(self, n: int) -> List[int]:
        """One sequence of n tokens, advancing the stream (dataset.cpp:66-80)."""
        if n <= 0:
            return []
        V = self.vocab
        state = self.stream.next_below(V)
        out = [state]
        for _ in range(1, n):
            u = self.stream.next_unit()
            cdf = self._cdf[state]
            nxt = V - 1
            for c in range(V):
                if u < cdf[c]:
                    nxt = c
                    break
            state = nxt
            out.append(state)
        return out

    def entropy_rate(self) -> float:
        """sum_v pi_v H(row_v), pi by power iteration (dataset.cpp:85-110)."""
        V = self.vocab
        pi = [1.0 / V] * V
        for _ in range(500):
            nxt = [0.0] * V
            for r in range(V):
                for c in range(V):
                    nxt[c] += pi[r] * self.transition[r, c]
            delta = sum(abs(nxt[c] - pi[c]) for c in range(V))
            pi = nxt
            if delta < 1e-14:
                break
        h = 0.0
        for r in range(V):
            hr = 0.0
            for c in range(V):
                p = self.transition[r, c]
                if p > 0.0:
                    hr -= p * math.log(p)
            h += pi[r] * hr
        return h
