"""rng.py replays numpy's PCG64 Generator exactly (the basis of the exact
speculative SA / EA batches)."""
from __future__ import annotations

import random

import numpy as np

from paper_2308_00127_b200 import rng as R


def test_stream_model_matches_numpy():
    for seed in range(60):
        real = np.random.default_rng(seed)
        mirror = np.random.default_rng(seed)
        pr = random.Random(seed)
        for _ in range(20):
            S, st = R.peek(mirror, 200)
            for _ in range(pr.randint(1, 12)):
                if pr.random() < 0.4:
                    a = real.random()
                    b, st = S.random(st)
                else:
                    h = pr.choice([1, 2, 3, 5, 7, 30, 200, 1000, 2**31 + 11,
                                   2**32])
                    a = int(real.integers(h))
                    b, st = S.integers(st, h)
                assert a == b
            R.commit(mirror, st)
        s1, s2 = real.bit_generator.state, mirror.bit_generator.state
        assert s1["state"] == s2["state"]
        assert s1["has_uint32"] == s2["has_uint32"]
        if s1["has_uint32"]:
            assert s1["uinteger"] == s2["uinteger"]


def test_ea_mutations_match_reference_loop():
    for seed, V, n_dev in [(0, 32, 3), (1, 202, 3), (2, 17, 2), (3, 50, 4),
                           (4, 5, 1)]:
        p = 1.0 / V
        real = np.random.default_rng(seed)
        mirror = np.random.default_rng(seed)
        for _ in range(5):
            steps = 40
            S, words, st = R.peek_words(mirror, steps * (V + 2) + 64)
            got = R.ea_mutations(S, words, st, steps, V, n_dev, p)
            for muts, _ in got:
                want = []
                for pos in range(V):  # heuristics.py:323-325
                    if real.random() < p:
                        want.append((pos, int(real.integers(n_dev))))
                assert muts == want
            R.commit(mirror, got[-1][1])
        assert real.bit_generator.state["state"] == \
            mirror.bit_generator.state["state"]


def test_random_below_p_integer_threshold():
    """ea_mutations finds random() < p hits with one integer compare per
    raw word; it equals the float test, including words at the boundary."""
    import math
    for V in (1, 2, 3, 7, 32, 202, 220, 1002):
        p = 1.0 / V
        lim = math.ceil(p * 2.0 ** 53) << 11
        ws = np.random.default_rng(V).integers(
            0, 2 ** 64 - 1, size=100_000, dtype=np.uint64, endpoint=True)
        edge = [x for x in (lim - 1, lim, lim + 1, lim - 2048, lim + 2047)
                if 0 <= x < 2 ** 64]
        ws = np.concatenate([ws, np.array(edge, np.uint64)])
        want = ((ws >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) < p
        got = (ws < np.uint64(lim)) if lim < 2 ** 64 else \
            np.ones(len(ws), bool)
        assert np.array_equal(want, got), V
