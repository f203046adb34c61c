"""The paper's parameter study on the GPU (BASELINE configs[1]; PAPER.md
Figs. 6-11): 400 x 400 lattices at 50:50 and 30:70 composition, omega/kT from
0.2 to 1.0, 10^5 MPKK sweeps each from a random start, sampling energy and the
cluster-size histogram of the minority/A lipid every `--every` sweeps over the
second half of the run.

All (f, omega) points run concurrently: one handle per point, each on its own
CUDA stream (one resident-kernel CTA per lattice), so the whole study takes
seconds.  Prints one JSON line per point and a summary table; the trend to
look for is fewer unlike contacts (lower N_AB per site) and
larger A clusters as omega grows — microdomain formation.

Usage: python tools/paper_study.py [--sweeps 100000] [--every 1000] [--out file]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweeps", type=int, default=100000)
    ap.add_argument("--every", type=int, default=1000)
    ap.add_argument("--L", type=int, default=400)
    ap.add_argument("--seed", type=int, default=1309)
    ap.add_argument("--seeds", type=int, default=1, help="independent replicas per (f, omega) point")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    if a.seeds > 1 and "KK_CLUSTER" not in os.environ:
        # each handle's plan assumes it has the GPU to itself: with several
        # replicas per handle it would take one 8-CTA cluster per replica, and
        # 18 such handles oversubscribe the SMs; one SM per replica (resident
        # kernel) is the better split for many concurrent handles
        os.environ["KK_CLUSTER"] = "0"
    if a.seeds == 1 and "KK_CLUSTER" not in os.environ:
        # one lattice per handle would take a 16-CTA cluster; 18 concurrent
        # handles fit the GPU at once with 8-CTA clusters (144 SMs)
        os.environ["KK_CLUSTER"] = "8"
    omegas = [0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0]
    fracs = [0.5, 0.3]
    pts = [(f, om) for f in fracs for om in omegas]
    streams = [torch.cuda.Stream() for _ in pts]
    lats = [kk.Lattice(a.L, a.L, f, om, a.seed + i, replicas=a.seeds) for i, (f, om) in enumerate(pts)]
    N = a.L * a.L
    acc = [{"nab": [], "mean_size": [], "largest": [], "n_clusters": []} for _ in pts]
    t0 = time.perf_counter()
    done = 0
    while done < a.sweeps:
        chunk = min(a.every, a.sweeps - done)
        for L, s in zip(lats, streams):
            L.sweep(chunk, s)
        done += chunk
        if done <= a.sweeps // 2:
            continue
        for i, (L, s) in enumerate(zip(lats, streams)):
            nab = L.energy(stream=s)[0]
            for r, h in enumerate(L.cluster_histogram(1, stream=s)):
                sizes = np.array([sz for sz, _ in h], np.float64)
                counts = np.array([c for _, c in h], np.float64)
                acc[i]["nab"].append(int(nab[r]) / N)
                acc[i]["n_clusters"].append(counts.sum())
                acc[i]["mean_size"].append(float((sizes * counts).sum() / counts.sum()))
                acc[i]["largest"].append(float(sizes.max() / N))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    rows = []
    for (f, om), L, d in zip(pts, lats, acc):
        st = L.stats().sum(axis=0)
        row = {"fraction_A": f, "omega_kT": om, "sweeps": a.sweeps, "replicas": a.seeds, "samples": len(d["nab"]),
               "nab_per_site": float(np.mean(d["nab"])), "mean_cluster_size_A": float(np.mean(d["mean_size"])),
               "clusters_A": float(np.mean(d["n_clusters"])), "largest_A_fraction": float(np.mean(d["largest"])),
               "acceptance": float(st[2] / max(st[0], 1))}
        rows.append(row)
        print(json.dumps(row), flush=True)
    total = a.sweeps * N * len(pts) * a.seeds
    print(f"# {len(pts)} x {a.seeds} lattices of {a.L}x{a.L}, {a.sweeps} sweeps each: {wall:.1f} s wall, "
          f"{total / wall / 1e9:.1f} G site-updates/s aggregate (incl. sampling)", flush=True)
    print("# f     omega  N_AB/site  <cluster size>  largest/N  acceptance")
    for r in rows:
        print(f"# {r['fraction_A']:.1f}   {r['omega_kT']:.1f}    {r['nab_per_site']:.4f}     "
              f"{r['mean_cluster_size_A']:10.1f}    {r['largest_A_fraction']:.4f}    {r['acceptance']:.4f}")
    if a.out:
        with open(a.out, "w") as fh:
            for r in rows:
                fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
