"""Tile-shape / CTA-size sweep of the planar pass kernel on one lattice state.

A master handle is equilibrated for W sweeps; every candidate plan gets its own
handle loaded with the master's packed lattice (device copy), runs S sweeps
(CUDA events) and reports G site-updates/s.

  python tools/planar_tune.py L [W] [S] "twi,thi,nt;twi,thi,nt;..."
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

L = int(sys.argv[1])
W = int(sys.argv[2]) if len(sys.argv) > 2 else 20
S = int(sys.argv[3]) if len(sys.argv) > 3 else 6
cands = [tuple(int(x) for x in c.split(",")) for c in sys.argv[4].split(";")] if len(sys.argv) > 4 else []
torch.cuda.set_device(0)
s = torch.cuda.current_stream()
M = kk.Lattice(L, L, 0.5, 0.6, 20261018)
M.sweep(W, s)
st = M.stats(reset=True)[0]
buf = torch.empty(L * L // 32, dtype=torch.int32, device="cuda")
M.copy_packed_device(buf.data_ptr(), False, s)
torch.cuda.synchronize()
print(f"{L}^2 after {W} sweeps: trivial {st[1] / st[0]:.3f}", flush=True)
M.close()
for twi, thi, nt in [(0, 0, 0)] + cands:
    env = {"KK_TWI": twi, "KK_THI": thi, "KK_PASS_THREADS": nt}
    for k, v in env.items():
        if v:
            os.environ[k] = str(v)
        else:
            os.environ.pop(k, None)
    try:
        H = kk.Lattice(L, L, 0.5, 0.6, 20261018, init=kk.KK_INIT_EMPTY)
        p = kk.plan(L, L, n_sm=0)
    except kk.KKError as e:
        print(f"twi={twi} thi={thi} nt={nt}: {e}")
        continue
    H.copy_packed_device(buf.data_ptr(), True, s)
    H.sweep(1, s)
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        H.sweep(S, s)
        e1.record(s)
        torch.cuda.synchronize()
        best = max(best, S * L * L / e0.elapsed_time(e1) / 1e6)
    print(f"TWI={p['tile_words']:4d} THI={p['tile_rows']:4d} nt={p['threads']} ctas={p['ctas']:5d} "
          f"boxes={p['tma_boxes']} smem={p['smem_bytes']}: {best:7.1f} G/s", flush=True)
    H.close()
