"""Pins for the oracle's cluster analysis (clusters over the
six nearest neighbours; the paper's Hoshen-Kopelman labelling has a unique
cluster multiset, which is what is compared).

Cross-checked against scipy.ndimage.label with the triangular-lattice
structuring element plus an independent periodic-boundary merge.
"""
from collections import Counter

import numpy as np
import pytest
from scipy import ndimage

from oracle import oracle as O

# neighbours (dx,dy): (+-1,0) (0,+-1) (1,1) (-1,-1) -> structure[dy+1][dx+1]
TRI = np.array([[1, 1, 0], [1, 1, 1], [0, 1, 1]])
NB = [(1, 0), (1, 1), (0, 1), (-1, 0), (-1, -1), (0, -1)]


def _scipy_periodic_sizes(lat, target):
    Ly, Lx = lat.shape
    mask = lat == target
    lab, n = ndimage.label(mask, structure=TRI)
    parent = list(range(n + 1))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    for y in range(Ly):
        for x in range(Lx):
            if not mask[y, x]:
                continue
            for dx, dy in NB:
                nx, ny = x + dx, y + dy
                if 0 <= nx < Lx and 0 <= ny < Ly:
                    continue                      # interior bonds: scipy did these
                nx, ny = nx % Lx, ny % Ly
                if mask[ny, nx]:
                    a, b = find(lab[y, x]), find(lab[ny, nx])
                    if a != b:
                        parent[max(a, b)] = min(a, b)
    roots = [find(v) for v in lab[mask]]
    return sorted(Counter(roots).values())


def test_special_cases():
    Lx, Ly = 12, 8
    assert O.cluster_sizes(np.ones((Ly, Lx), np.uint8), 1).tolist() == [Lx * Ly]
    assert O.cluster_sizes(np.zeros((Ly, Lx), np.uint8), 1).tolist() == []
    one = np.zeros((Ly, Lx), np.uint8)
    one[3, 4] = 1
    assert O.cluster_sizes(one, 1).tolist() == [1]
    assert O.cluster_sizes(one, 0).tolist() == [Lx * Ly - 1]
    # (1,-1) diagonal is NOT a bond on the triangular lattice; (1,1) is
    d = np.zeros((Ly, Lx), np.uint8)
    d[2, 2] = d[3, 3] = 1
    assert O.cluster_sizes(d, 1).tolist() == [2]
    d = np.zeros((Ly, Lx), np.uint8)
    d[3, 2] = d[2, 3] = 1
    assert sorted(O.cluster_sizes(d, 1).tolist()) == [1, 1]
    # a row wraps around the torus into one cluster
    r = np.zeros((Ly, Lx), np.uint8)
    r[5, :] = 1
    assert O.cluster_sizes(r, 1).tolist() == [Lx]
    # row stripes: every A row is its own cluster
    s = np.zeros((Ly, Lx), np.uint8)
    s[0::2, :] = 1
    assert O.cluster_sizes(s, 1).tolist() == [Lx] * (Ly // 2)
    # proper 3-colouring class: all isolated
    y, x = np.mgrid[0:12, 0:12]
    t = (((x + y) % 3) == 0).astype(np.uint8)
    assert O.cluster_sizes(t, 1).tolist() == [1] * int(t.sum())


@pytest.mark.parametrize("Lx,Ly", [(8, 8), (12, 8), (16, 20), (40, 40)])
def test_matches_scipy_label_periodic(Lx, Ly):
    rng = np.random.default_rng(Lx * Ly)
    for f in [0.1, 0.3, 0.5, 0.55, 0.7, 0.9]:
        for _ in range(5):
            lat = (rng.random((Ly, Lx)) < f).astype(np.uint8)
            for target in (0, 1):
                got = sorted(O.cluster_sizes(lat, target).tolist())
                assert got == _scipy_periodic_sizes(lat, target)
                assert sum(got) == int((lat == target).sum())


def test_translation_invariance():
    rng = np.random.default_rng(9)
    lat = (rng.random((16, 24)) < 0.5).astype(np.uint8)
    ref = O.cluster_histogram(lat, 1)
    for sy, sx in [(1, 0), (0, 5), (7, 11)]:
        assert O.cluster_histogram(np.roll(np.roll(lat, sy, 0), sx, 1), 1) == ref


def test_framed_tile_tiling_rule():
    """The rule test_gpu_parity's 65536^2 cluster test relies on, checked by
    brute force on a 3 x 2 tiling: a tile with a B frame (row 0, column 0)
    inside an A ring (rows 1, t-1, columns 1, t-1) keeps every A cluster and
    every interior B cluster inside its tile, and the frames join into one B
    cluster."""
    from tests import inputs
    t = 64
    tile = inputs.random_lattice(t, t, 0.5, seed=4242)
    tile[1, :] = tile[t - 1, :] = 1
    tile[:, 1] = tile[:, t - 1] = 1
    tile[0, :] = 0
    tile[:, 0] = 0
    big = np.tile(tile, (2, 3))
    n = 6
    assert O.cluster_histogram(big, 1) == [(sz, c * n) for sz, c in O.cluster_histogram(tile, 1)]
    hb = dict(O.cluster_histogram(tile, 0))
    frame = 2 * t - 1
    hb[frame] -= 1
    assert O.cluster_histogram(big, 0) == sorted([(sz, c * n) for sz, c in hb.items() if c] + [(frame * n, 1)])
