"""Shared test scaffolding, restating P/tests/support.hpp (test infra).

* SplitMix64 — P/include/dim3/datagen.hpp:176-193
* random_instance — P/tests/support.hpp:108-153 (same draw order, so seeds
  41/61/201-205/301-306/501-510 give the same instances as the reference's
  own tests)
* oracle_pairs — P/tests/support.hpp:41-52 (brute-force y-indexed join)
"""
from __future__ import annotations

import math

import numpy as np

M64 = (1 << 64) - 1


def mix64(x: int) -> int:
    x &= M64
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & M64
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & M64
    x ^= x >> 31
    return x


class SplitMix64:
    def __init__(self, seed: int = 0):
        self.state = seed & M64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & M64
        return mix64(self.state)

    def bounded(self, n: int) -> int:
        return (self.next() * n) >> 64

    def unit(self) -> float:
        return float(self.next() >> 11) * (2.0 ** -53)


def random_instance(rng: SplitMix64, max_card=256, max_rows=5000, out_j_cap=500000):
    """Returns ((r_left, r_right), (s_left, s_right)) as uint64 arrays."""
    while True:
        xc = 1 + rng.bounded(max_card)
        yc = 1 + rng.bounded(max_card)
        zc = 1 + rng.bounded(max_card)

        def density():
            lg = -3.0 + rng.unit() * (math.log10(0.5) + 3.0)
            return math.pow(10.0, lg)

        def rows(a, b):
            want = density() * float(a) * float(b)
            n = int(want + 0.5)
            return min(max(n, 1), max_rows)

        nr = rows(xc, yc)
        ns = rows(zc, yc)
        est = float(nr) * float(ns) / float(yc)
        if est > float(out_j_cap):
            continue
        x_mul, x_add, z_mul, z_add, y_mul = 1, 0, 1, 0, 1
        mode = rng.bounded(4)
        if mode == 1:
            x_mul = 3 + rng.bounded(97)
            z_mul = 3 + rng.bounded(97)
            y_mul = 2 + rng.bounded(31)
        elif mode == 2:
            x_add = (1 << 32) + rng.bounded(1000)
            z_add = (1 << 33) + rng.bounded(1000)
        rl, rr, sl, sr = [], [], [], []
        for _ in range(nr):
            rl.append(rng.bounded(xc) * x_mul + x_add)
            rr.append(rng.bounded(yc) * y_mul)
        for _ in range(ns):
            sl.append(rng.bounded(zc) * z_mul + z_add)
            sr.append(rng.bounded(yc) * y_mul)
        u = lambda v: np.array(v, dtype=np.uint64)  # noqa: E731
        return (u(rl), u(rr)), (u(sl), u(sr))


def oracle_pairs(r, s) -> set:
    """P/tests/support.hpp:41-52."""
    by_y: dict[int, list[int]] = {}
    for z, y in zip(s[0].tolist(), s[1].tolist()):
        by_y.setdefault(y, []).append(z)
    out = set()
    for x, y in zip(r[0].tolist(), r[1].tolist()):
        for z in by_y.get(y, ()):
            out.add((x, z))
    return out


def pair_set(raw_x, raw_z) -> set:
    return set(zip(np.asarray(raw_x).tolist(), np.asarray(raw_z).tolist()))
