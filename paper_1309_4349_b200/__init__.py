"""paper_1309_4349_b200 — B200-native Massive Parallel Kawasaki Kinetics.

The hot path (MPKK sweeps, observables, cluster labelling) lives in
``libkk.so`` (CUDA, sm_100a, C ABI in ``include/kk.h``); ``kk`` is its thin
ctypes binding and ``distributed`` drives row slabs across GPUs with
torch.distributed.
"""
from .kk import (KK_INIT_BLOCK, KK_INIT_EMPTY, KK_INIT_RANDOM, REGION_ALL,  # noqa: F401
                 REGION_BOUNDARY, REGION_INTERIOR, KKError, Lattice, launch_count, load)
