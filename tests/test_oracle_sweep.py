"""Pins for the oracle's MPKK sweep (readings R4-R6).

- composition conservation and energy bookkeeping;
- the 4x4 centre classes are conflict-free (pure geometry, reading R4), and
  the oracle's iteration result is independent of the centre visiting order;
- proposal statistics: class k_j uniform over 16, direction uniform over 6
  ("1/7 * 1/6" generalised);
- detailed balance / stationarity: on a 4x4 lattice, independent chains
  reproduce the exactly enumerated Boltzmann distribution (chi-square);
- omega = 0 ideal mixing (hypergeometric closed form);
- omega trend: larger omega -> fewer AB contacts, larger clusters
  (PAPER.md:170-192 microdomain formation).
"""
import itertools
import math

import numpy as np
import pytest
from scipy import stats as sps

from oracle import oracle as O

NB = [(1, 0), (1, 1), (0, 1), (-1, 0), (-1, -1), (0, -1)]


def test_conservation_and_bookkeeping():
    for (Lx, Ly, f, om) in [(8, 8, 0.5, 0.5), (16, 12, 0.3, 1.0), (12, 16, 0.7, -0.4)]:
        lat = O.init_random(Lx, Ly, f, seed=42)
        nA0 = O.composition(lat)
        assert nA0 == O.count_a_for(Lx * Ly, f)
        nab0 = O.n_ab(lat)
        st = O.run(lat, om, seed=42, n_sweeps=30)
        assert O.composition(lat) == nA0
        assert st["attempted"] == 30 * Lx * Ly
        assert st["accepted"] <= st["attempted"] - st["trivial"]
        assert O.n_ab(lat) - nab0 == st["dnab_sum"]


def test_determinism_and_seed_dependence():
    a = O.init_random(16, 16, 0.5, seed=7)
    b = a.copy()
    c = a.copy()
    O.run(a, 0.6, 99, 20)
    O.run(b, 0.6, 99, 20)
    O.run(c, 0.6, 100, 20)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, c)
    # run(n) == n single sweeps with consecutive sweep indices
    d = O.init_random(16, 16, 0.5, seed=7)
    for s in range(20):
        O.run(d, 0.6, 99, 1, first_sweep=s)
    assert np.array_equal(a, d)


def test_init_block_and_random():
    lat = O.init_block(10, 7, 0.5)
    assert lat.reshape(-1)[:35].all() and not lat.reshape(-1)[35:].any()
    assert O.count_a_for(63, 0.5) == 32          # round half up
    r1 = O.init_random(20, 20, 0.3, seed=5)
    r2 = O.init_random(20, 20, 0.3, seed=5)
    r3 = O.init_random(20, 20, 0.3, seed=5, replica=1)
    assert np.array_equal(r1, r2) and not np.array_equal(r1, r3)
    assert O.composition(r1) == 120
    # uniformity: per-site occupation over many seeds ~ fraction_A
    acc = np.zeros((8, 8))
    for s in range(2000):
        acc += O.init_random(8, 8, 0.25, seed=s)
    p = acc / 2000
    assert abs(p.mean() - 0.25) < 1e-12
    assert np.abs(p - 0.25).max() < 5 * math.sqrt(0.25 * 0.75 / 2000)


def _ball(Lx, Ly, x, y, r):
    out = {(x % Lx, y % Ly)}
    for _ in range(r):
        out = {((a + dx) % Lx, (b + dy) % Ly) for (a, b) in out for (dx, dy) in NB + [(0, 0)]}
    return out


@pytest.mark.parametrize("Lx,Ly", [(4, 4), (8, 4), (4, 8), (8, 8), (12, 8), (16, 16)])
def test_center_classes_are_conflict_free(Lx, Ly):
    """Reading R4: within one class (x=kx, y=ky mod 4) the read set of every
    centre (its partner and both their neighbourhoods, any direction) misses
    the write set (centre + any partner) of every other centre."""
    for kx in range(4):
        for ky in range(4):
            centres = [(x, y) for y in range(ky, Ly, 4) for x in range(kx, Lx, 4)]
            reads = {c: set().union(*[_ball(Lx, Ly, c[0] + dx, c[1] + dy, 1) for dx, dy in NB])
                     for c in centres}
            writes = {c: _ball(Lx, Ly, c[0], c[1], 1) for c in centres}
            for c in centres:
                for c2 in centres:
                    if c2 != c:
                        assert not (reads[c] & writes[c2]), (Lx, Ly, c, c2)


def test_iteration_order_independence():
    """The listing's 'For each domain d in D(k)' loop gives the same lattice
    for any visiting order (PAPER.md:100 'performed on each domain
    simultaneously')."""
    rng = np.random.default_rng(3)
    Lx, Ly = 16, 12
    for trial in range(6):
        lat0 = O.init_random(Lx, Ly, 0.5, seed=trial)
        O.run(lat0, 0.8, seed=11, n_sweeps=3)
        ref = None
        for perm in range(4):
            lat = lat0.copy()
            order = np.arange(Lx * Ly) if perm == 0 else rng.permutation(Lx * Ly)
            for j in range(16):
                O.iteration_ordered(lat, 0.8, 11, 5, 0, j, order)
            if ref is None:
                ref = lat
                full = lat0.copy()
                O.run(full, 0.8, seed=11, n_sweeps=1, first_sweep=5)
                assert np.array_equal(full, ref)
            else:
                assert np.array_equal(lat, ref)


def test_proposal_statistics():
    """k_j uniform over 16 classes; directions uniform over 6."""
    kc = np.zeros(16)
    for s in range(4000):
        for k in O.schedule(1234, s):
            kc[k] += 1
    assert sps.chisquare(kc).pvalue > 1e-4
    dc = np.zeros(6)
    for s in range(200):
        for (x, y) in [(1, 2), (5, 2), (9, 6), (13, 30)]:
            for j in range(16):
                d, _ = O.center_draw(77, s, 0, j, 1, 2, x, y)
                dc[d] += 1
    assert sps.chisquare(dc).pvalue > 1e-4


def _enumerate_4x4(nA):
    Lx = Ly = 4
    states, nabs = [], []
    for pos in itertools.combinations(range(16), nA):
        lat = np.zeros(16, np.uint8)
        lat[list(pos)] = 1
        lat = lat.reshape(Ly, Lx)
        states.append(lat.tobytes())
        nabs.append(O.n_ab(lat))
    return states, np.array(nabs)


def _chains_4x4(nA, omega, n_chains, burn):
    finals = []
    f = nA / 16.0
    for r in range(n_chains):
        lat = O.init_random(4, 4, f, seed=2024, replica=r)
        O.run(lat, omega, seed=2024, n_sweeps=burn, replica=r)
        finals.append(lat.tobytes())
    return finals


@pytest.mark.parametrize("omega", [0.0, 0.5, 1.0, -0.5])
def test_4x4_energy_levels_boltzmann(omega):
    """Detailed balance: independent chains on the 4x4
    torus, nA=8 (12870 states), sample the exactly enumerated Boltzmann
    distribution over N_AB levels: chi-square p > 1e-4."""
    states, nabs = _enumerate_4x4(8)
    index = {s: n for s, n in zip(states, nabs)}
    levels = np.unique(nabs)
    w = np.array([np.sum(np.exp(-omega * nabs[nabs == L])) for L in levels])
    p = w / w.sum()
    n = 5000
    obs = np.zeros(len(levels))
    # burn-in: at omega=1 the 12 two-stripe ground states need ~300 sweeps
    for s in _chains_4x4(8, omega, n, burn=400):
        obs[np.searchsorted(levels, index[s])] += 1
    exp_ = p * n
    keep = exp_ >= 5
    o = np.append(obs[keep], obs[~keep].sum())
    e = np.append(exp_[keep], exp_[~keep].sum())
    if e[-1] == 0:
        o, e = o[:-1], e[:-1]
    assert sps.chisquare(o, e).pvalue > 1e-4


def test_4x4_state_distribution_boltzmann():
    """State-level check with nA=3 (560 states) at omega=0.7."""
    omega = 0.7
    states, nabs = _enumerate_4x4(3)
    w = np.exp(-omega * nabs)
    p = w / w.sum()
    idx = {s: i for i, s in enumerate(states)}
    n = 12000
    obs = np.zeros(len(states))
    for s in _chains_4x4(3, omega, n, burn=200):
        obs[idx[s]] += 1
    assert sps.chisquare(obs, p * n).pvalue > 1e-4


def test_omega_zero_ideal_mixing():
    """omega=0: every exchange accepted, stationary state uniform over
    arrangements: E[N_AB] = 3N * 2 nA nB / (N (N-1))."""
    Lx = Ly = 8
    N = 64
    nA = 32
    vals = []
    for r in range(400):
        lat = O.init_block(Lx, Ly, 0.5)
        st = O.run(lat, 0.0, seed=5, n_sweeps=40, replica=r)
        assert st["accepted"] == st["attempted"] - st["trivial"]
        vals.append(O.n_ab(lat))
    vals = np.array(vals, float)
    expect = 3 * N * 2 * nA * (N - nA) / (N * (N - 1))
    se = vals.std(ddof=1) / math.sqrt(len(vals))
    assert abs(vals.mean() - expect) < 4 * se


def test_omega_trend_microdomains():
    """Larger omega (stronger AB repulsion) -> fewer AB contacts and larger
    A clusters (microdomain formation)."""
    Lx = Ly = 32
    res = []
    for om in [0.2, 0.6, 1.0]:
        lat = O.init_random(Lx, Ly, 0.5, seed=8)
        O.run(lat, om, seed=8, n_sweeps=400)
        nab, sizes = [], []
        for k in range(10):
            O.run(lat, om, seed=8, n_sweeps=20, first_sweep=400 + 20 * k)
            nab.append(O.n_ab(lat))
            cs = O.cluster_sizes(lat, 1)
            sizes.append(cs.mean())
        res.append((np.mean(nab), np.mean(sizes)))
    assert res[0][0] > res[1][0] > res[2][0]
    assert res[0][1] < res[1][1] < res[2][1]
