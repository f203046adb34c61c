"""Detailed balance at GPU scale: thousands of independent 4x4 replicas (one
chain each, distinct RNG counters) sampled after burn-in must reproduce the
exact Boltzmann distribution of N_AB over all C(16, 8) configurations
(E/kT = omega * N_AB, reading R3; PAPER.md:59-65 Metropolis, 122 detailed
balance).  The exact distribution is enumerated here with numpy; the test
shares nothing with the oracle or the kernels."""
import itertools
import math

import numpy as np
import pytest

from tests.test_gpu_parity import _gpu, _lat  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


def _nab(states):
    """N_AB of a batch of (n, 4, 4) 0/1 lattices on the triangular torus:
    bonds (1,0), (0,1), (1,1) in axial coordinates (R2)."""
    s = states.astype(np.int8)
    n = np.zeros(len(s), np.int64)
    for dy, dx in ((0, 1), (1, 0), (1, 1)):
        n += (s != np.roll(np.roll(s, -dy, axis=1), -dx, axis=2)).sum(axis=(1, 2))
    return n


def _exact_levels(omega):
    states = []
    for ones in itertools.combinations(range(16), 8):
        a = np.zeros(16, np.int8)
        a[list(ones)] = 1
        states.append(a.reshape(4, 4))
    nab = _nab(np.stack(states))
    levels, counts = np.unique(nab, return_counts=True)
    w = counts * np.exp(-omega * (levels - levels.min()))
    return levels, w / w.sum()


@pytest.mark.parametrize("omega", [0.0, 0.5, 1.0])
def test_4x4_replicas_sample_boltzmann(omega):
    from paper_1309_4349_b200 import kk
    R, burn = 8192, 400
    L = _lat(4, 4, 0.5, omega, 777, replicas=R, init=kk.KK_INIT_RANDOM)
    L.sweep(burn)
    nab = L.energy()[0]
    levels, p = _exact_levels(omega)
    obs = np.array([(nab == v).sum() for v in levels], np.float64)
    assert obs.sum() == R                          # every sample is a valid N_AB level
    exp = p * R
    keep = exp >= 5                                # pool sparse levels into one cell
    o = np.append(obs[keep], obs[~keep].sum())
    e = np.append(exp[keep], exp[~keep].sum())
    if e[-1] < 5:
        o, e = o[:-1], e[:-1]
        o[-1] += obs[~keep].sum()
        e[-1] += exp[~keep].sum()
    chi2 = float(((o - e) ** 2 / e).sum())
    dof = len(o) - 1
    # p < 1e-4 bound via Wilson-Hilferty for the chi-square tail
    z = ((chi2 / dof) ** (1 / 3) - (1 - 2 / (9 * dof))) / math.sqrt(2 / (9 * dof))
    assert z < 3.72, (omega, chi2, dof, o.tolist(), e.round(1).tolist())
    # and the mean energy to within 5 standard errors
    mean_exact = float((p * levels).sum())
    sd = math.sqrt(float((p * (levels - mean_exact) ** 2).sum()))
    assert abs(nab.mean() - mean_exact) < 5 * sd / math.sqrt(R)
