"""Exact replay of numpy ``Generator(PCG64)`` draws from raw 64-bit words.

The reference's search loops draw from ``np.random.default_rng(seed)``
(heuristics.py:266, 308). To evaluate many future candidates in one GPU
batch while keeping the reference's trajectory bit-for-bit, the host peeks
ahead: it takes raw words from a clone of the generator
(``random_raw``) and restates how numpy consumes them:

* ``random()`` -> one whole word, ``(w >> 11) * 2**-53``; the 32-bit
  buffer is left alone;
* ``integers(high)`` (int64, exclusive high <= 2**32) -> Lemire's bounded
  method on 32-bit draws, where a 32-bit draw takes the cached upper half of
  the previous word if one is buffered (``has_uint32``), else the low half
  of a fresh word (caching the high half); ``high == 1`` draws nothing.

The state of the stream is (word index, has_uint32, cached half). Tests pin
this against numpy itself over many seeds and ranges.
"""
from __future__ import annotations

import math
from bisect import bisect_left

import numpy as np

M32 = 0xFFFFFFFF
_D53 = 1.0 / 9007199254740992.0


class RawStream:
    """Consumption model over a fixed array of raw words."""

    __slots__ = ("w",)

    def __init__(self, words: np.ndarray):
        # numpy words, converted on access: the EA peeks ~V words per step
        # but reads only the few that hit
        self.w = np.asarray(words, np.uint64)

    def next32(self, st):
        i, has, u = st
        if has:
            return u, (i, 0, 0)
        if i >= len(self.w):
            raise IndexError("peek window exhausted")
        x = int(self.w[i])
        return x & M32, (i + 1, 1, x >> 32)

    def next64(self, st):
        i, has, u = st
        if i >= len(self.w):
            raise IndexError("peek window exhausted")
        return int(self.w[i]), (i + 1, has, u)

    def random(self, st):
        x, st = self.next64(st)
        return (x >> 11) * _D53, st

    def integers(self, st, high: int):
        """Generator.integers(high) for 1 <= high <= 2**32."""
        rng = high - 1
        if rng == 0:
            return 0, st
        v, st = self.next32(st)
        m = v * high
        left = m & M32
        if left < high:
            thr = (M32 - rng) % high
            while left < thr:
                v, st = self.next32(st)
                m = v * high
                left = m & M32
        return m >> 32, st


def peek(rng: np.random.Generator, nwords: int):
    """(RawStream over the next `nwords` raw words, start state) without
    moving `rng`."""
    bg = rng.bit_generator
    st = bg.state
    clone = type(bg)()
    clone.state = st
    words = clone.random_raw(nwords)
    return RawStream(words), (0, int(st["has_uint32"]), int(st["uinteger"]))


def commit(rng: np.random.Generator, state) -> None:
    """Move `rng` to stream state (words consumed, has_uint32, cached)."""
    i, has, u = state
    bg = rng.bit_generator
    if i:
        bg.advance(i)  # also clears the 32-bit buffer
    st = bg.state
    st["has_uint32"] = int(has)
    st["uinteger"] = int(u)
    bg.state = st


def ea_mutations(S: RawStream, words: np.ndarray, st, steps: int, V: int,
                 n_dev: int, p: float):
    """Mutation lists of `steps` (1+1) EA steps (heuristics.py:321-325: for
    each position, ``random() < p`` then ``integers(n_dev)``), vectorised
    over the runs of misses: random() draws are whole words and leave the
    32-bit buffer alone, so only the hits need the sequential model.
    Returns [(mutations, state after the step)]; raises IndexError when the
    peeked words run out (the caller shortens its window)."""
    W = len(words)
    # random() < p  <=>  (w >> 11) * 2^-53 < p  <=>  (w >> 11) < ceil(p * 2^53)
    # (the scalings by 2^53 are exact)  <=>  w < ceil(p * 2^53) * 2^11
    lim = math.ceil(p * 9007199254740992.0) << 11
    if lim >= 1 << 64:
        hits = list(range(W))
    else:
        hits = np.flatnonzero(words < np.uint64(lim)).tolist()
    hits.append(W)  # word indices with random() < p, then a sentinel
    out = []
    i, has, c = st
    for _ in range(steps):
        pos = 0
        muts = []
        while pos < V:
            rem = V - pos
            if i + rem > W:
                raise IndexError("peek window exhausted")
            j = hits[bisect_left(hits, i)]  # first hit at or after i
            if j >= i + rem:
                i += rem
                break
            pos += j - i
            i = j + 1
            val, (i, has, c) = S.integers((i, has, c), n_dev)
            muts.append((pos, val))
            pos += 1
        out.append((muts, (i, has, c)))
    return out


def peek_words(rng: np.random.Generator, nwords: int):
    """Like peek() but also returns the raw words as a numpy array."""
    bg = rng.bit_generator
    st = bg.state
    clone = type(bg)()
    clone.state = st
    words = clone.random_raw(nwords)
    return (RawStream(words), words,
            (0, int(st["has_uint32"]), int(st["uinteger"])))
