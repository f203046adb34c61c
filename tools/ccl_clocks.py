"""Phase clocks of the CCL tile kernel (library built with -DKK_CCL_CLK):
KK_LIB=paper_1309_4349_b200/libkk_cclclk.so python tools/ccl_clocks.py [L] [sweeps]
Phases of ccl_runs_kernel: load + run ids, unions, run sizes, root sizes,
roots -> hist/nodes, node + edge export; thread 0 of every CTA, summed."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100
torch.cuda.set_device(0)
lib = kk.load()
lib.kk_debug_ccl_clocks.argtypes = [ctypes.c_void_p]
lat = kk.Lattice(L, L, 0.5, 0.6, 7)
lat.sweep(n)
lat.cluster_histogram(1)
buf = (ctypes.c_ulonglong * 16)()
lib.kk_debug_ccl_clocks(buf)
lat.cluster_histogram(1)
torch.cuda.synchronize()
lib.kk_debug_ccl_clocks(buf)
names = ["load + run ids", "unions", "run sizes", "root sizes", "roots->hist/nodes", "node+edge export"]
tot = sum(buf[k] for k in range(len(names)))
for k, nm in enumerate(names):
    print(f"{nm:20s} {buf[k] / tot:6.3f}")
