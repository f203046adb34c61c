"""Long-run parity at the BASELINE configs' full length: the paper's 400x400
lattice over 10^5 MPKK sweeps (configs[1]) and 64x64 over 10^4 sweeps
(configs[0]) must end in exactly the oracle's state; likewise thousands of
sweeps of lattices run on the planar tile kernel.  The oracle's results are
stored in tests/golden/long_run*.json by tests/golden/make_long_run*.py,
which call only oracle/ (~25 CPU minutes, so they are precomputed)."""
import hashlib
import json
import os

import numpy as np
import pytest

from tests.test_gpu_parity import _gpu, _lat  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "long_run.json")
GOLDEN_PLANAR = os.path.join(os.path.dirname(__file__), "golden", "long_run_planar.json")
PLANAR_ENV = {"KK_PLANAR": 2, "KK_RESIDENT": 0, "KK_CLUSTER": 0, "KK_BAND": 0}


def _runs():
    out = []
    for path, env in ((GOLDEN, None), (GOLDEN_PLANAR, PLANAR_ENV)):
        with open(path) as fh:
            out += [dict(r, env=env) for r in json.load(fh)["runs"]]
    return out


@pytest.mark.parametrize("run", _runs(), ids=lambda r: r["name"])
def test_long_run_matches_oracle_state(run):
    if run["env"]:
        from paper_1309_4349_b200 import kk
        for k, v in run["env"].items():
            os.environ[k] = str(v)
        try:
            assert kk.plan(run["Lx"], run["Ly"], n_sm=0)["kernel"] == "planar"
        finally:
            for k in run["env"]:
                os.environ.pop(k, None)
    L = _lat(run["Lx"], run["Ly"], run["f"], run["omega"], run["seed"], env=run["env"])
    L.sweep(run["sweeps"])
    lat = L.get_lattice()[0]
    st = L.stats()[0]
    assert hashlib.sha256(np.ascontiguousarray(lat, np.uint8).tobytes()).hexdigest() == run["sha256"]
    assert int(L.energy()[0][0]) == run["n_ab"] and int(L.composition()[0]) == run["n_a"]
    assert list(st) == [run["attempted"], run["trivial"], run["accepted"], run["dnab_sum"]]
