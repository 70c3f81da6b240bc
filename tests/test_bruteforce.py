"""Brute-force pin: C oracle vs exact rational arithmetic on 4^3 lattices (CPU, no GPU).

The initial state is dyadic (k / 2^20) so it is exact in both; the exact result is rounded only
once, at the comparison. Covers every operator, periodic and walled (NoSlip + UBB) lattices,
and the force term.
"""
from fractions import Fraction as Fr
from itertools import product

import numpy as np
import pytest

import lbminputs as LI
import oracle as O
from tests.bruteforce.exact import Exact

N = 4


def _dyadic_state(Q, seed):
    rng = np.random.default_rng(seed)
    _, w, _ = O.stencil_arrays(Q)
    f = w[:, None, None, None] * (1 + 0.05 * rng.uniform(-1, 1, (Q, N, N, N)))
    return np.round(f * 2 ** 20) / 2 ** 20


CASES = [
    ("srt", 19, (1.8,), (0, 0, 0), "periodic", 2),
    ("trt", 19, (1.6, 0.5), (1e-3, 0, -5e-4), "walls", 2),
    ("trt", 27, (1.3, 0.9), (0, 0, 0), "walls", 1),
    ("mrt", 19, (1.9, 1.3, 1.1, 0.8), (0, 0, 0), "walls", 1),
    ("kbc", 19, (1.9,), (0, 0, 0), "walls", 1),
    ("kbc", 27, (1.8,), (0, 0, 0), "walls", 1),
    ("cumulant", 19, (1.9, 1.2, 1.1, 0.8), (0, 0, 0), "walls", 1),
    ("cumulant", 27, (1.95, 1.2, 1.1, 0.9, 1.3, 0.7), (0, 0, 0), "periodic", 1),
    ("cumulant", 27, (1.95,), (0, 0, 0), "walls", 1),
    ("trt", 19, (1.6, 0.5), (1e-3, 0, -5e-4), "walls", 2, "incompressible"),
    ("srt", 27, (1.7,), (0, 0, 0), "periodic", 1, "incompressible"),
    ("mrt", 19, (1.9, 1.3, 1.1, 0.8), (0, 0, 0), "periodic", 1, "incompressible"),
    ("trt", 19, (1.6, 0.5), (0, 0, 0), "walls", 2, "moment_matched"),
    ("mrt", 19, (1.9, 1.3, 1.1, 0.8), (0, 0, 0), "walls", 1, "moment_matched"),
    ("srt", 27, (1.8,), (0, 0, 0), "periodic", 1, "moment_matched"),
]


@pytest.mark.parametrize("op,Q,rates,force,geom,steps,eq", [c if len(c) == 7 else c + ("compressible",) for c in CASES])
def test_oracle_matches_exact_rationals(op, Q, rates, force, geom, steps, eq):
    uw = (0.0625, -0.03125, 0.0)
    if geom == "walls":
        fl = np.zeros((N, N, N), np.uint8)
        fl[:, 0, :] = LI.NOSLIP
        fl[N - 1, 1:, :] = LI.UBB
        fl[0, 2, 1] = LI.NOSLIP
    else:
        fl = None
    m = O.Method(Q=Q, op=op, rates=rates, force=force, ubb_u=uw, nthreads=1, equilibrium=eq)
    d = O.Domain(m, N, N, N, flags=fl)
    f0 = _dyadic_state(Q, seed=11)
    got = d.run_pull(f0, steps)

    ex = Exact(Q, op, rates, force=force, ubb_u=uw, equilibrium=eq)
    fe = {(x, y, z): [Fr(float(f0[q, z, y, x])) for q in range(Q)] for x, y, z in product(range(N), repeat=3)}
    flags = {(x, y, z): int(fl[z, y, x]) if fl is not None else 0 for x, y, z in product(range(N), repeat=3)}
    for _ in range(steps):
        fe = ex.step_pull(fe, flags, (N, N, N))
    worst = 0.0
    for (x, y, z), vals in fe.items():
        if flags[(x, y, z)]:
            continue
        for q in range(Q):
            worst = max(worst, abs(float(vals[q]) - got[q, z, y, x]) / abs(float(vals[q])))
    assert worst <= 1e-14, worst
