"""Parity of the resident kernel (whole replica in shared memory, periodic
wrap kept as rebuilt copies; kk_pass.cu resident_kernel) with the oracle, and
of the tile kernel on the same shapes — both must give the oracle's lattice,
counters and N_AB bit for bit (north_star: "bit-exact agreement with the CPU
oracle on every config").

KK_RESIDENT=2 forces the resident kernel whenever the replica fits, 0 forces
the tile kernel; the default (1) picks the resident kernel when the tile
kernel would use <= 2 CTAs per replica.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests import inputs
from tests.test_gpu_parity import _gpu, _lat, _run_parity  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("Lx,Ly,R", [
    (64, 4, 1),      # smallest resident shape: two lattice words, 4 rows
    (64, 8, 2),
    (68, 12, 1),     # tail of 4 bits, W = 3 (minimum with a tail)
    (96, 16, 1),     # no tail, W = 3
    (100, 20, 3),    # tail of 4 bits
    (120, 8, 1),     # tail of 24 bits
    (128, 32, 1),
    (400, 40, 2),    # tail of 16 bits (the paper's width)
    (1000, 44, 1),   # Lx % 32 = 8
    (4096, 12, 1),   # wide and short
])
@pytest.mark.parametrize("mode", [2, 0])
def test_resident_and_tile_paths_match_oracle(Lx, Ly, R, mode):
    _run_parity(Lx, Ly, 0.5, 0.7, Lx * 7 + Ly, 5, R=R, env={"KK_RESIDENT": mode})


@pytest.mark.parametrize("omega", [0.0, 0.6, -1.0, 5.0])
def test_resident_omega(omega):
    _run_parity(100, 28, 0.3, omega, 11, 8, env={"KK_RESIDENT": 2})


def test_resident_arbitrary_start_stripes():
    """Striped start (domain walls on the wrap seams) and a random start."""
    stripes = np.stack([inputs.striped_lattice(72, 16)] * 2)
    _run_parity(72, 16, 0.5, 1.0, 17, 20, R=2, start=stripes, env={"KK_RESIDENT": 2})
    start = inputs.random_lattice(100, 24, 0.45, seed=9, replicas=2)
    _run_parity(100, 24, 0.5, 0.8, 4242, 15, R=2, start=start, env={"KK_RESIDENT": 2})


def test_resident_mid_sweep_start():
    """kk_pass (tile kernel, T=4) leaves the handle at iteration j=4; kk_sweep
    (resident kernel) must continue from (sweep 0, j=4); three more passes
    finish sweep 2 — the whole run equals 3 oracle sweeps."""
    from paper_1309_4349_b200 import kk
    Lx, Ly, seed, om = 100, 20, 31337, 0.9
    L = _lat(Lx, Ly, 0.5, om, seed, iters_per_pass=4, env={"KK_RESIDENT": 2})
    ref = O.init_random(Lx, Ly, 0.5, seed)
    L.run_pass(kk.REGION_ALL, None, None)
    L.pass_commit()
    L.sweep(2)
    for _ in range(3):
        L.run_pass(kk.REGION_ALL, None, None)
        L.pass_commit()
    assert L.sweep_index() == 3
    ost = O.run(ref, om, seed, 3)
    assert np.array_equal(L.get_lattice()[0], ref)
    st = L.stats()[0]
    assert list(st) == [ost["attempted"], ost["trivial"], ost["accepted"], ost["dnab_sum"]]


def test_config3_replica_batch_sample():
    """BASELINE configs[3] (1024 x 400x400 replicas, resident by default):
    all replicas conserve composition and keep N_AB = N_AB(0) + sum dN; a
    sample of replicas matches the oracle bit for bit after 2 sweeps."""
    R, Lx, Ly, seed, om = 1024, 400, 400, 2024, 0.6
    L = _lat(Lx, Ly, 0.5, om, seed, replicas=R)
    nab0 = L.energy()[0]
    L.sweep(2)
    st = L.stats()
    nab1 = L.energy()[0]
    assert (L.composition() == O.count_a_for(Lx * Ly, 0.5)).all()
    assert np.array_equal(nab1 - nab0, st[:, 3])
    assert (st[:, 0] == 2 * Lx * Ly).all()
    got = L.get_lattice()
    for r in [0, 1, 517, 1023]:
        ref = O.init_random(Lx, Ly, 0.5, seed, replica=r)
        ost = O.run(ref, om, seed, 2, replica=r)
        assert np.array_equal(got[r], ref), r
        assert list(st[r]) == [ost["attempted"], ost["trivial"], ost["accepted"], ost["dnab_sum"]]


@pytest.mark.parametrize("nt", [128, 256, 512])
@pytest.mark.parametrize("Lx,Ly,R", [(100, 20, 3), (400, 40, 2), (64, 64, 5)])
def test_resident_cta_sizes(Lx, Ly, R, nt):
    """All resident CTA sizes (KK_RES_THREADS) give the oracle's result."""
    _run_parity(Lx, Ly, 0.4, 0.8, 5 + nt, 4, R=R, env={"KK_RESIDENT": 2, "KK_RES_THREADS": nt})


# ---- band kernel (lattice spread over all SMs' shared memory, 3*TB-row halos
# exchanged between neighbouring bands through L2 every TB iterations)
@pytest.mark.parametrize("Lx,Ly", [(1000, 1776), (2048, 1184), (400, 2368), (4096, 1776)])
def test_band_kernel_matches_oracle(Lx, Ly):
    from paper_1309_4349_b200 import kk
    env = {"KK_RESIDENT": 0, "KK_CLUSTER": 0, "KK_BAND": 2}
    for key, v in env.items():
        os.environ[key] = str(v)
    try:
        assert kk.plan(Lx, Ly, n_sm=0)["kernel"] == "band"
    finally:
        for key in env:
            os.environ.pop(key, None)
    _run_parity(Lx, Ly, 0.5, 0.7, Lx + 3 * Ly, 4, env=env)


def test_band_kernel_mid_sweep_start_and_omega():
    from paper_1309_4349_b200 import kk
    Lx, Ly, seed, om = 2048, 1184, 99, 1.1
    L = _lat(Lx, Ly, 0.4, om, seed, iters_per_pass=4, env={"KK_RESIDENT": 0, "KK_CLUSTER": 0, "KK_BAND": 2})
    ref = O.init_random(Lx, Ly, 0.4, seed)
    L.run_pass(kk.REGION_ALL, None, None)      # tile kernel: iterations 0..3 of sweep 0
    L.pass_commit()
    L.sweep(2)                                  # band kernel from (sweep 0, j = 4)
    for _ in range(3):
        L.run_pass(kk.REGION_ALL, None, None)
        L.pass_commit()
    ost = O.run(ref, om, seed, 3)
    assert np.array_equal(L.get_lattice()[0], ref)
    assert list(L.stats()[0]) == [ost["attempted"], ost["trivial"], ost["accepted"], ost["dnab_sum"]]


def test_config2_4096_band_and_tile_agree():
    """BASELINE configs[2] (4096^2): the band kernel (KK_BAND=2, opt-in) and
    the default (planar tile) kernel give the identical lattice and counters,
    equal to the oracle's."""
    from paper_1309_4349_b200 import kk
    A = _lat(4096, 4096, 0.5, 0.6, 4096, init=kk.KK_INIT_RANDOM, env={"KK_BAND": 2})
    B = _lat(4096, 4096, 0.5, 0.6, 4096, init=kk.KK_INIT_RANDOM)
    A.sweep(3)
    B.sweep(3)
    assert np.array_equal(A.get_packed(), B.get_packed())
    assert np.array_equal(A.stats(), B.stats())
    ref = O.init_random(4096, 4096, 0.5, 4096)
    O.run(ref, 0.6, 4096, 3)
    assert np.array_equal(A.get_lattice()[0], ref)


# ---- cluster kernel (opt-in): the band kernel inside one thread-block cluster
# per replica, 3-row halos read from the neighbouring CTAs' shared memory
@pytest.mark.parametrize("Lx,Ly,R,C", [(64, 64, 1, 16), (400, 400, 1, 16), (400, 40, 1, 8), (100, 32, 2, 8),
                                       (128, 96, 3, 4), (68, 16, 1, 2), (1000, 64, 1, 16)])
def test_cluster_kernel_matches_oracle(Lx, Ly, R, C):
    _run_parity(Lx, Ly, 0.5, 0.8, Lx + Ly + C, 4, R=R, env={"KK_CLUSTER": C})


def test_cluster_kernel_mid_sweep_start():
    from paper_1309_4349_b200 import kk
    Lx, Ly, seed, om = 400, 80, 555, 0.7
    L = _lat(Lx, Ly, 0.5, om, seed, iters_per_pass=4, env={"KK_CLUSTER": 8})
    ref = O.init_random(Lx, Ly, 0.5, seed)
    L.run_pass(kk.REGION_ALL, None, None)      # tile kernel: iterations 0..3 of sweep 0
    L.pass_commit()
    L.sweep(2)                                  # cluster kernel from (sweep 0, j = 4)
    for _ in range(3):
        L.run_pass(kk.REGION_ALL, None, None)
        L.pass_commit()
    ost = O.run(ref, om, seed, 3)
    assert np.array_equal(L.get_lattice()[0], ref)
    assert list(L.stats()[0]) == [ost["attempted"], ost["trivial"], ost["accepted"], ost["dnab_sum"]]


@pytest.mark.parametrize("tb", [2, 4, 8])
@pytest.mark.parametrize("Lx,Ly,R,C", [(400, 400, 1, 8), (100, 96, 2, 4), (256, 512, 1, 16), (1000, 96, 1, 2)])
def test_cluster_kernel_temporal_blocking(Lx, Ly, R, C, tb):
    """Halos of 3*TB rows exchanged every TB iterations (KK_CLUSTER_TB)."""
    from paper_1309_4349_b200 import kk
    rows_per_band = Ly // C
    if rows_per_band < 3 * tb + 4:
        pytest.skip("bands too short for this TB")
    _run_parity(Lx, Ly, 0.5, 0.8, Lx + Ly + C + tb, 5, R=R, env={"KK_CLUSTER": C, "KK_CLUSTER_TB": tb})


def test_cluster_kernel_temporal_blocking_mid_sweep():
    from paper_1309_4349_b200 import kk
    Lx, Ly, seed, om = 400, 160, 556, 0.7
    L = _lat(Lx, Ly, 0.5, om, seed, iters_per_pass=4, env={"KK_CLUSTER": 4, "KK_CLUSTER_TB": 4})
    ref = O.init_random(Lx, Ly, 0.5, seed)
    L.run_pass(kk.REGION_ALL, None, None)      # tile kernel: iterations 0..3 of sweep 0
    L.pass_commit()
    L.sweep(2)                                  # cluster kernel from (sweep 0, j = 4), blocks across sweeps
    for _ in range(3):
        L.run_pass(kk.REGION_ALL, None, None)
        L.pass_commit()
    ost = O.run(ref, om, seed, 3)
    assert np.array_equal(L.get_lattice()[0], ref)
    assert list(L.stats()[0]) == [ost["attempted"], ost["trivial"], ost["accepted"], ost["dnab_sum"]]


@pytest.mark.parametrize("Lx,Ly,tb", [(4096, 4096, 2), (4096, 4096, 4), (128, 3584, 8), (2048, 2048, 2)])
def test_band_kernel_temporal_blocking(Lx, Ly, tb):
    """Band kernel with 3*TB-row halos exchanged through L2 every TB iterations
    (148 bands; 2048^2 has 13-14-row bands, 3584 rows give 24-row bands)."""
    _run_parity(Lx, Ly, 0.5, 0.7, Lx + tb, 2, env={"KK_RESIDENT": 0, "KK_CLUSTER": 0, "KK_BAND": 2,
                                                    "KK_BAND_TB": tb})


def test_cluster_default_for_replica_batch():
    """16 replicas of 400^2 run on 16 eight-CTA clusters by default (128 SMs);
    every replica must equal the oracle."""
    from paper_1309_4349_b200 import kk
    p = kk.plan(400, 400, replicas=16, n_sm=0)
    assert p["kernel"] == "cluster" and p["ctas"] == 128
    _run_parity(400, 400, 0.5, 0.7, 16, 2, R=16)


@pytest.mark.parametrize("Lx,Ly,env", [(512, 448, {"KK_CLUSTER": 4, "KK_CLUSTER_TB": 8}),
                                        (128, 3584, {"KK_RESIDENT": 0, "KK_CLUSTER": 0, "KK_BAND": 2,
                                                     "KK_BAND_TB": 8})])
def test_temporal_blocks_spanning_two_sweeps(Lx, Ly, env):
    """Blocks of 8 iterations starting at j = 4 cover iterations 12..15 of one
    sweep and 0..3 of the next (schedules of two sweeps in one block); the
    band case has 148 bands of 24 rows, the shortest that hold 3*8-row halos."""
    from paper_1309_4349_b200 import kk
    seed, om = 918, 0.75
    L = _lat(Lx, Ly, 0.5, om, seed, iters_per_pass=4, env=env)
    ref = O.init_random(Lx, Ly, 0.5, seed)
    L.run_pass(kk.REGION_ALL, None, None)      # tile kernel: iterations 0..3 of sweep 0
    L.pass_commit()
    L.sweep(2)                                  # blocks 4..11, 12..3, 4..11, 12..3
    for _ in range(3):
        L.run_pass(kk.REGION_ALL, None, None)
        L.pass_commit()
    ost = O.run(ref, om, seed, 3)
    assert np.array_equal(L.get_lattice()[0], ref)
    assert list(L.stats()[0]) == [ost["attempted"], ost["trivial"], ost["accepted"], ost["dnab_sum"]]
