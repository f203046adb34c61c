"""Writes tests/golden/long_run.json: the oracle's state after long runs of
BASELINE configs[1] (the paper's 400x400 lattice, 10^5 sweeps) and configs[0]
(64x64, 10^4 sweeps), as a SHA-256 of the final lattice plus N_AB, the
composition and the counters.  Calls only oracle/ (no GPU code); takes ~20
minutes single-threaded.  Usage: python tests/golden/make_long_run.py"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

RUNS = [
    {"name": "configs1_400x400_f0.5_w0.6_1e5", "Lx": 400, "Ly": 400, "f": 0.5, "omega": 0.6, "seed": 1309,
     "sweeps": 100000},
    {"name": "configs1_400x400_f0.3_w1.0_2e4", "Lx": 400, "Ly": 400, "f": 0.3, "omega": 1.0, "seed": 4349,
     "sweeps": 20000},
    {"name": "configs0_64x64_f0.5_w0.5_1e4", "Lx": 64, "Ly": 64, "f": 0.5, "omega": 0.5, "seed": 20240601,
     "sweeps": 10000},
]


def main():
    out = []
    for r in RUNS:
        t0 = time.time()
        lat = O.init_random(r["Lx"], r["Ly"], r["f"], r["seed"])
        st = O.run(lat, r["omega"], r["seed"], r["sweeps"])
        rec = dict(r)
        rec.update({"sha256": hashlib.sha256(lat.astype("uint8").tobytes()).hexdigest(),
                    "n_ab": int(O.n_ab(lat)), "n_a": int(lat.sum()),
                    "attempted": st["attempted"], "trivial": st["trivial"], "accepted": st["accepted"],
                    "dnab_sum": st["dnab_sum"], "oracle_seconds": round(time.time() - t0, 1)})
        out.append(rec)
        print(json.dumps(rec), flush=True)
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "long_run.json"), "w") as fh:
        json.dump({"source": "tests/golden/make_long_run.py (oracle only)", "runs": out}, fh, indent=1)


if __name__ == "__main__":
    main()
