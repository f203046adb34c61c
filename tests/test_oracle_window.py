"""Pin for the halo depth of temporal blocking / slab decomposition
(reading R8): running T iterations on a window that extends hy = 3T rows
beyond an interior band reproduces the full-lattice result on that band.
This is the light-cone argument the GPU tiles and the multi-GPU slabs rely on
(a site's value after one iteration depends only on sites within distance 3).
"""
import numpy as np
import pytest

from oracle import oracle as O


def _full_iterations(lat, omega, seed, sweep, j0, T):
    """Reference: iterations j0..j0+T-1 of `sweep` on the full periodic
    lattice via the ordered-iteration entry point (row-major order)."""
    Ly, Lx = lat.shape
    order = np.arange(Lx * Ly)
    for j in range(j0, j0 + T):
        O.iteration_ordered(lat, omega, seed, sweep, 0, j, order)


@pytest.mark.parametrize("T", [1, 2, 4, 8, 16])
def test_window_halo_3T_reproduces_interior(T):
    Lx, Ly = 16, 64
    hy = 3 * T
    rng = np.random.default_rng(T)
    for trial in range(4):
        lat = O.init_random(Lx, Ly, 0.5, seed=trial)
        O.run(lat, 0.7, seed=3, n_sweeps=2)
        y0, H = int(rng.integers(0, Ly)), 12
        rows = [(y0 - hy + r) % Ly for r in range(H + 2 * hy)]
        win = np.ascontiguousarray(lat[rows])
        j0 = 16 - T if T < 16 else 0
        O.window_iterations(win, Ly, y0 - hy, 0.7, 3, 9, 0, j0, T, hy, hy + H)
        ref = lat.copy()
        _full_iterations(ref, 0.7, 3, 9, j0, T)
        assert np.array_equal(win[hy:hy + H], ref[[(y0 + r) % Ly for r in range(H)]])


def test_window_too_shallow_halo_can_fail():
    """Sanity of the pin itself: with a shallow halo (hy = 3 < 3T) differences
    appear for some seed, so the window test is not vacuous."""
    Lx, Ly, T = 32, 64, 8
    hy = 3
    bad = 0
    for trial in range(8):
        lat = O.init_random(Lx, Ly, 0.5, seed=trial)
        y0, H = 20, 8
        rows = [(y0 - hy + r) % Ly for r in range(H + 2 * hy)]
        win = np.ascontiguousarray(lat[rows])
        O.window_iterations(win, Ly, y0 - hy, 0.0, 3, 9, 0, 0, T, hy, hy + H)
        ref = lat.copy()
        _full_iterations(ref, 0.0, 3, 9, 0, T)
        bad += not np.array_equal(win[hy:hy + H], ref[[(y0 + r) % Ly for r in range(H)]])
    assert bad > 0
