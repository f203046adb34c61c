"""GPU CCL vs oracle stress: random lattices, sizes spanning several CCL tiles.
Saves the first failing lattice to gpurun_out/ccl_fail_*.npy."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
rng = np.random.default_rng(0)
fails = 0
for trial in range(60):
    Lx = int(rng.choice([8, 40, 64, 400, 520, 1024]))
    Ly = int(rng.choice([4, 32, 36, 64, 100, 400]))
    R = int(rng.choice([1, 2]))
    f = float(rng.choice([0.3, 0.5, 0.6]))
    lat = (rng.random((R, Ly, Lx)) < f).astype(np.uint8)
    L = kk.Lattice(Lx, Ly, 0.5, 0.5, 1, replicas=R, init=kk.KK_INIT_EMPTY)
    L.set_lattice(lat)
    for target in (0, 1):
        got = L.cluster_histogram(target)
        for r in range(R):
            ref = O.cluster_histogram(lat[r], target)
            if got[r] != ref:
                fails += 1
                da, db = dict(got[r]), dict(ref)
                diff = [(k, da.get(k), db.get(k)) for k in sorted(set(da) | set(db)) if da.get(k) != db.get(k)]
                print(f"FAIL Lx={Lx} Ly={Ly} R={R} r={r} f={f} target={target} diff={diff[:8]}", flush=True)
                if fails <= 3:
                    np.save(f"gpurun_out/ccl_fail_{fails}.npy", lat[r])
    L.close()
print("fails", fails)
