"""Double-buffered host I/O of the C ABI (kk_upload_packed_async /
kk_commit_upload / kk_snapshot / kk_download_packed_async; "copy
whole data to device memory, then perform simulations and move it back"):
stream-ordered copies through the handle's staging buffers, overlapping the
sweeps, must deliver exactly the oracle's lattices."""
import numpy as np
import pytest

from oracle import oracle as O
from tests import inputs
from tests.test_gpu_parity import _gpu  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("Lx,Ly,planar", [(512, 256, 2), (1000, 64, 0)])
def test_pipelined_upload_sweep_download(Lx, Ly, planar, monkeypatch):
    import torch
    from paper_1309_4349_b200 import kk
    monkeypatch.setenv("KK_PLANAR", str(planar))
    monkeypatch.setenv("KK_RESIDENT", "0")
    monkeypatch.setenv("KK_CLUSTER", "0")
    om, seed, steps, n = 0.7, 31, 3, 2
    L = kk.Lattice(Lx, Ly, 0.5, om, seed, init=kk.KK_INIT_EMPTY)
    W = L.W
    starts = [inputs.random_lattice(Lx, Ly, 0.3 + 0.2 * k, seed=k) for k in range(steps)]
    hin = [None] * steps
    for k, s in enumerate(starts):   # packed layout: ceil(Lx/32) words per row, unused bits zero
        p = np.zeros((Ly, W), np.uint32)
        pk = np.packbits(s, axis=1, bitorder="little")
        pk = np.pad(pk, ((0, 0), (0, 4 * W - pk.shape[1])))
        p[:] = pk.view(np.uint32)
        hin[k] = torch.from_numpy(p.view(np.int32)).pin_memory()
    hout = [torch.zeros(Ly * W, dtype=torch.int32).pin_memory() for _ in range(steps)]
    comp, cp = torch.cuda.current_stream(), torch.cuda.Stream()
    L.upload_async(hin[0].data_ptr(), cp)
    for k in range(steps):
        L.commit_upload(comp)
        if k + 1 < steps:
            L.upload_async(hin[k + 1].data_ptr(), cp)     # overlaps step k's sweeps
        L.sweep(n, comp)
        L.snapshot(comp)
        L.download_async(hout[k].data_ptr(), cp)          # overlaps step k+1
    torch.cuda.synchronize()
    for k in range(steps):
        ref = starts[k].copy()
        O.run(ref, om, seed, n, first_sweep=k * n)
        got = inputs.unpack_rows(hout[k].numpy().view(np.uint32).reshape(1, Ly, W), Lx)[0]
        assert np.array_equal(got, ref), k
