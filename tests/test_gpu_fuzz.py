"""Seeded random configurations through every sweep path (tile kernel with all
T, resident kernel, band kernel, mixed kk_pass / kk_sweep calls) against the
oracle: lattice, counters, N_AB, composition and both cluster histograms must
match bit for bit.  The configurations are drawn once from a fixed seed, so
the test is deterministic."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.test_gpu_parity import _gpu, _lat  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


def _configs(n=40, seed=20261018):
    rng = np.random.default_rng(seed)
    out = []
    for k in range(n):
        Lx = int(rng.choice([4, 8, 12, 32, 60, 64, 68, 96, 100, 128, 132, 200, 256, 400, 1000]))
        Ly = int(rng.integers(1, 33)) * 4
        R = int(rng.choice([1, 1, 2, 3]))
        T = int(rng.choice([1, 2, 4, 8]))
        path = str(rng.choice(["default", "tile", "resident", "band", "cluster"]))
        omega = float(np.round(rng.uniform(-2.0, 3.0), 3))
        f = float(np.round(rng.uniform(0.0, 1.0), 3))
        sweeps = int(rng.integers(1, 6))
        split = bool(rng.integers(0, 2))      # start with single passes (kk_pass) before kk_sweep
        out.append((k, Lx, Ly, R, T, path, omega, f, sweeps, split))
    return out


ENV = {"default": {}, "tile": {"KK_RESIDENT": 0, "KK_BAND": 0, "KK_CLUSTER": 0},
       "resident": {"KK_RESIDENT": 2, "KK_CLUSTER": 0}, "band": {"KK_RESIDENT": 0, "KK_BAND": 2, "KK_CLUSTER": 0},
       "cluster": {"KK_CLUSTER": 4}}


@pytest.mark.parametrize("k,Lx,Ly,R,T,path,omega,f,sweeps,split", _configs())
def test_fuzz_config_matches_oracle(k, Lx, Ly, R, T, path, omega, f, sweeps, split):
    from paper_1309_4349_b200 import kk
    seed = 7919 * k + 13
    L = _lat(Lx, Ly, f, omega, seed, replicas=R, iters_per_pass=T, env=ENV[path])
    refs = [O.init_random(Lx, Ly, f, seed, replica=r) for r in range(R)]
    assert np.array_equal(L.get_lattice(), np.stack(refs))
    passes = 0
    if split and T < 16:
        passes = int(np.random.default_rng(k).integers(1, 16 // T + 1))
        for _ in range(passes):
            L.run_pass(kk.REGION_ALL, None, None)
            L.pass_commit()
    L.sweep(sweeps)
    # the oracle runs whole sweeps: finish the started sweep with passes
    if passes and passes % (16 // T):
        for _ in range(16 // T - passes % (16 // T)):
            L.run_pass(kk.REGION_ALL, None, None)
            L.pass_commit()
    total = sweeps + (passes + 16 // T - 1) // (16 // T) if passes else sweeps
    assert L.sweep_index() == total
    got = L.get_lattice()
    st = L.stats()
    nab = L.energy()[0]
    comp = L.composition()
    for r in range(R):
        ost = O.run(refs[r], omega, seed, total, replica=r)
        assert np.array_equal(got[r], refs[r]), f"replica {r}"
        assert list(st[r]) == [ost["attempted"], ost["trivial"], ost["accepted"], ost["dnab_sum"]]
        assert nab[r] == O.n_ab(refs[r])
        assert comp[r] == int(refs[r].sum())
    for target in (0, 1):
        h = L.cluster_histogram(target)
        for r in range(R):
            assert h[r] == O.cluster_histogram(refs[r], target)
    L.close()
