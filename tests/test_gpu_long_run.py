"""Long-run parity at the BASELINE configs' full length: the paper's 400x400
lattice over 10^5 MPKK sweeps (configs[1]) and 64x64 over 10^4 sweeps
(configs[0]) must end in exactly the oracle's state.  The oracle's results
are stored in tests/golden/long_run.json by tests/golden/make_long_run.py,
which calls only oracle/ (~20 CPU minutes, so they are precomputed)."""
import hashlib
import json
import os

import numpy as np
import pytest

from tests.test_gpu_parity import _gpu, _lat  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "long_run.json")


def _runs():
    with open(GOLDEN) as fh:
        return json.load(fh)["runs"]


@pytest.mark.parametrize("run", _runs(), ids=lambda r: r["name"])
def test_long_run_matches_oracle_state(run):
    L = _lat(run["Lx"], run["Ly"], run["f"], run["omega"], run["seed"])
    L.sweep(run["sweeps"])
    lat = L.get_lattice()[0]
    st = L.stats()[0]
    assert hashlib.sha256(np.ascontiguousarray(lat, np.uint8).tobytes()).hexdigest() == run["sha256"]
    assert int(L.energy()[0][0]) == run["n_ab"] and int(L.composition()[0]) == run["n_a"]
    assert list(st) == [run["attempted"], run["trivial"], run["accepted"], run["dnab_sum"]]
