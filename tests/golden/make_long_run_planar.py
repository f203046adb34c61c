"""Writes tests/golden/long_run_planar.json: the oracle's state after long runs
on lattices whose rows are whole 128-site groups (the planar tile kernel's
domain, run with KK_PLANAR=2 by tests/test_gpu_long_run.py), as a SHA-256 of
the final lattice plus N_AB, the composition and the counters.  Calls only
oracle/ (no GPU code); takes ~6 minutes single-threaded.
Usage: python tests/golden/make_long_run_planar.py"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

RUNS = [
    {"name": "planar_1024x1024_f0.5_w0.6_2000", "Lx": 1024, "Ly": 1024, "f": 0.5, "omega": 0.6, "seed": 6172,
     "sweeps": 2000},
    {"name": "planar_512x512_f0.3_w1.0_5000", "Lx": 512, "Ly": 512, "f": 0.3, "omega": 1.0, "seed": 1309,
     "sweeps": 5000},
    {"name": "planar_1536x384_f0.45_w-0.4_3000", "Lx": 1536, "Ly": 384, "f": 0.45, "omega": -0.4, "seed": 77,
     "sweeps": 3000},
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
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "long_run_planar.json"), "w") as fh:
        json.dump({"source": "tests/golden/make_long_run_planar.py (oracle only)", "runs": out}, fh, indent=1)


if __name__ == "__main__":
    main()
