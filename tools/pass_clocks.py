"""Phase clocks of one tile-kernel CTA (build with -DKK_PASS_CLK, KK_LIB=...).
Usage: KK_LIB=variants/libkk_clk.so python tools/pass_clocks.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
lib = kk.load()
out = np.zeros(16, np.uint64)
for L_ in (4096, 65536):
    L = kk.Lattice(L_, L_, 0.5, 0.6, 3, init=kk.KK_INIT_BLOCK)
    L.sweep(1)
    torch.cuda.synchronize()
    lib.kk_debug_pass_clocks(out.ctypes.data_as(ctypes.c_void_p))
    n = 20 if L_ == 4096 else 2
    L.sweep(n)
    torch.cuda.synchronize()
    lib.kk_debug_pass_clocks(out.ctypes.data_as(ctypes.c_void_p))
    passes = 2 * n
    us = out.astype(np.float64) / passes / 1.965e3
    print(f"{L_}^2 per pass (us, CTA (1,1)): setup+staging {us[0]:.2f} | items {us[1]:.2f} | "
          f"iteration barriers {us[2]:.2f} | write-back {us[3]:.2f}", flush=True)
    L.close()
