"""Seeded synthetic inputs shared by the oracle and the CUDA path in tests.

Holds none of the method's arithmetic: only numpy random lattices with the
shapes and compositions of the paper's workloads.
"""
import numpy as np


def random_lattice(Lx, Ly, fraction_A, seed, replicas=None):
    """Bernoulli(fraction_A) sites (1 = A) — arbitrary, not exact-composition."""
    rng = np.random.default_rng(seed)
    shape = (Ly, Lx) if replicas is None else (replicas, Ly, Lx)
    return (rng.random(shape) < fraction_A).astype(np.uint8)


def striped_lattice(Lx, Ly, period=4):
    """Non-random start with structure: horizontal stripes of A/B."""
    y = np.arange(Ly)[:, None]
    return np.broadcast_to(((y // period) % 2 == 0), (Ly, Lx)).astype(np.uint8).copy()


def unpack_rows(packed, Lx):
    """Packed uint32 rows (bit x%32 of word x/32) -> uint8 sites."""
    b = np.unpackbits(packed.view(np.uint8), axis=-1, bitorder="little")
    return b[..., :Lx]
