"""Single 400^2 lattice (cluster kernel) and the 1024 x 400^2 batch (resident
kernel): site-updates/s with the library in KK_LIB — used to compare the
normal build with a probe build whose draws are replaced by a few integer ops
(-DKK_NOPHILOX_PROBE on a local patch; timing only, wrong results).
Usage: KK_LIB=... python tools/cluster_probe.py"""
import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_1309_4349_b200 import kk
torch.cuda.set_device(0); s = torch.cuda.current_stream()
for (L, R) in [(400, 1), (400, 1024)]:
    lat = kk.Lattice(L, L, 0.5, 0.6, 3, replicas=R)
    lat.sweep(20, s); torch.cuda.synchronize()
    n = 400 if R == 1 else 20
    best = 0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); lat.sweep(n, s); e1.record(s); torch.cuda.synchronize()
        best = max(best, n * L * L * R / e0.elapsed_time(e1) / 1e6)
    print(f"{R} x {L}^2 {kk.plan(L, L, replicas=R, n_sm=0)['kernel']}: {best:.2f} G/s", flush=True)
    lat.close()
