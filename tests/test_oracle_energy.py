"""Pins for the oracle's energy model (PAPER.md:78-82 omega_AB; reading R3) and
Metropolis acceptance (PAPER.md:59-65 step 2c; reading R5).

The oracle's N_AB, local dN and acceptance are checked against closed forms,
special lattices, and brute-force full recomputation — never against
themselves.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O

NB = [(1, 0), (1, 1), (0, 1), (-1, 0), (-1, -1), (0, -1)]


def test_omega_formula():
    # PAPER.md:80, omega_AB = g_AB - (g_AA + g_BB)/2
    assert O.omega_from_gibbs(0.0, 0.0, 0.0) == 0.0
    assert O.omega_from_gibbs(1.0, 1.0, 1.0) == 0.0
    assert O.omega_from_gibbs(-2.0, 0.5, -1.0) == 2.0


@pytest.mark.parametrize("Lx,Ly", [(4, 4), (8, 4), (12, 8), (16, 16)])
def test_gibbs_energy_equals_const_plus_omega_nab(Lx, Ly):
    """sum over contacts of g = 3 nA gAA + 3 nB gBB + omega N_AB (6 contacts
    per site, 2 N_AA + N_AB = 6 nA): the paper's 'only one parameter'."""
    rng = np.random.default_rng(Lx * 100 + Ly)
    for _ in range(20):
        lat = (rng.random((Ly, Lx)) < rng.random()).astype(np.uint8)
        gAA, gAB, gBB = rng.normal(size=3)
        nA = int(lat.sum())
        nB = lat.size - nA
        omega = gAB - 0.5 * (gAA + gBB)
        lhs = O.gibbs_energy(lat, gAA, gAB, gBB)
        rhs = 3 * nA * gAA + 3 * nB * gBB + omega * O.n_ab(lat)
        assert lhs == pytest.approx(rhs, abs=1e-9)


def test_nab_special_lattices():
    Lx, Ly = 12, 12
    N = Lx * Ly
    assert O.n_ab(np.ones((Ly, Lx), np.uint8)) == 0
    assert O.n_ab(np.zeros((Ly, Lx), np.uint8)) == 0
    one = np.zeros((Ly, Lx), np.uint8)
    one[5, 7] = 1
    assert O.n_ab(one) == 6                       # isolated site: six unlike contacts
    rows = np.zeros((Ly, Lx), np.uint8)
    rows[0::2, :] = 1                             # row stripes: 4 unlike of 6 per site
    assert O.n_ab(rows) == 2 * N
    cols = np.zeros((Ly, Lx), np.uint8)
    cols[:, 0::2] = 1                             # column stripes: 4 unlike of 6
    assert O.n_ab(cols) == 2 * N
    y, x = np.mgrid[0:Ly, 0:Lx]
    three = (((x + y) % 3) == 0).astype(np.uint8)  # proper 3-colouring class
    assert O.n_ab(three) == 6 * int(three.sum())
    # translation invariance (periodic lattice)
    rng = np.random.default_rng(1)
    lat = (rng.random((Ly, Lx)) < 0.4).astype(np.uint8)
    assert O.n_ab(np.roll(np.roll(lat, 3, 0), 5, 1)) == O.n_ab(lat)


def _brute_nab(lat):
    """Independent count: unordered pairs via the three forward bonds."""
    Ly, Lx = lat.shape
    n = 0
    for (dx, dy) in [(1, 0), (1, 1), (0, 1)]:
        n += int((lat != np.roll(np.roll(lat, -dy, 0), -dx, 1)).sum())
    return n


@pytest.mark.parametrize("Lx,Ly", [(4, 4), (4, 8), (8, 4), (12, 8), (8, 12)])
def test_delta_nab_matches_full_recompute(Lx, Ly):
    rng = np.random.default_rng(Lx * 7 + Ly)
    for _ in range(6):
        lat = (rng.random((Ly, Lx)) < 0.5).astype(np.uint8)
        base = _brute_nab(lat)
        assert O.n_ab(lat) == base
        for y in range(Ly):
            for x in range(Lx):
                for dx, dy in NB:
                    tx, ty = (x + dx) % Lx, (y + dy) % Ly
                    sw = lat.copy()
                    sw[y, x], sw[ty, tx] = lat[ty, tx], lat[y, x]
                    assert O.delta_nab(lat, (x, y), (tx, ty)) == _brute_nab(sw) - base


def _threshold(dE):
    """Smallest u32 that is rejected (binary search on the oracle's rule)."""
    lo, hi = 0, 1 << 32
    while lo < hi:
        mid = (lo + hi) // 2
        if O.metropolis_accept(dE, mid):
            lo = mid + 1
        else:
            hi = mid
    return lo


@pytest.mark.parametrize("omega", [0.2, 0.5, 0.6, 1.0, 2.5])
def test_metropolis_detailed_balance_ratio(omega):
    """P(acc | dE) / P(acc | -dE) = exp(-dE) (PAPER.md:120 detailed balance)
    up to the 2^-32 resolution of u."""
    for dn in [2, 4, 6]:
        dE = omega * dn
        assert O.metropolis_accept(-dE, 0xFFFFFFFF)          # downhill: always
        p_up = _threshold(dE) / 2.0 ** 32
        p_down = 1.0
        assert abs(p_up / p_down - math.exp(-dE)) <= 2.0 ** -31
    assert O.metropolis_accept(0.0, 0xFFFFFFFF)              # dE = 0: always
