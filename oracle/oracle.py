"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``oracle/kk_oracle.c``, the plain single-threaded C
implementation of the MPKK path of arXiv:1309.4349 (see that file's header for
the passage each function follows).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module; the product package ``paper_1309_4349_b200`` never does.

Lattices are numpy ``uint8`` arrays of shape ``(Ly, Lx)``, 1 = lipid A, 0 = B.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from collections import Counter
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kk_oracle.c")
_LIB = os.path.join(_HERE, "libkk_oracle.so")

_u8p = ctypes.POINTER(ctypes.c_uint8)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u32p = ctypes.POINTER(ctypes.c_uint32)


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-shared", "-fPIC",
             "-o", _LIB, _SRC, "-lm"])
    return _LIB


class Stats(ctypes.Structure):
    _fields_ = [("attempted", ctypes.c_int64), ("trivial", ctypes.c_int64),
                ("accepted", ctypes.c_int64), ("dnab_sum", ctypes.c_int64)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.kko_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
        L.kko_count_a_for.argtypes = [ctypes.c_int64, ctypes.c_double]
        L.kko_count_a_for.restype = ctypes.c_int64
        L.kko_init_block.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_double, _u8p]
        L.kko_init_random.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                      ctypes.c_uint64, ctypes.c_uint32, _u8p]
        L.kko_omega_from_gibbs.argtypes = [ctypes.c_double] * 3
        L.kko_omega_from_gibbs.restype = ctypes.c_double
        L.kko_n_ab.argtypes = [ctypes.c_int64, ctypes.c_int64, _u8p]
        L.kko_n_ab.restype = ctypes.c_int64
        L.kko_gibbs_energy.argtypes = [ctypes.c_int64, ctypes.c_int64, _u8p] + [ctypes.c_double] * 3
        L.kko_gibbs_energy.restype = ctypes.c_double
        L.kko_composition.argtypes = [ctypes.c_int64, _u8p]
        L.kko_composition.restype = ctypes.c_int64
        L.kko_delta_nab.argtypes = [ctypes.c_int64, ctypes.c_int64, _u8p] + [ctypes.c_int64] * 4
        L.kko_delta_nab.restype = ctypes.c_int64
        L.kko_metropolis_accept.argtypes = [ctypes.c_double, ctypes.c_uint32]
        L.kko_metropolis_accept.restype = ctypes.c_int
        L.kko_schedule.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                   ctypes.POINTER(ctypes.c_int)]
        L.kko_center_draw.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                      ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int64, ctypes.c_int64,
                                      ctypes.POINTER(ctypes.c_int), _u32p]
        L.kko_sweep.argtypes = [ctypes.c_int64, ctypes.c_int64, _u8p, ctypes.c_double,
                                ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                ctypes.POINTER(Stats)]
        L.kko_run.argtypes = [ctypes.c_int64, ctypes.c_int64, _u8p, ctypes.c_double,
                              ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64,
                              ctypes.c_uint32, ctypes.POINTER(Stats)]
        L.kko_iteration_ordered.argtypes = [ctypes.c_int64, ctypes.c_int64, _u8p,
                                            ctypes.c_double, ctypes.c_uint64, ctypes.c_uint32,
                                            ctypes.c_uint32, ctypes.c_int, _i64p,
                                            ctypes.c_int64, ctypes.POINTER(Stats)]
        L.kko_window_iterations.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.c_int64, _u8p, ctypes.c_double,
                                            ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                            ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                            ctypes.c_int64, ctypes.POINTER(Stats)]
        L.kko_clusters.argtypes = [ctypes.c_int64, ctypes.c_int64, _u8p, ctypes.c_int, _i64p]
        L.kko_clusters.restype = ctypes.c_int64
        _lib = L
    return _lib


def _u8(a: np.ndarray):
    assert a.dtype == np.uint8 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u8p)


# --------------------------------------------------------------------------- RNG
def philox4x32_10(ctr, key):
    c = (ctypes.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (ctypes.c_uint32 * 4)()
    lib().kko_philox4x32_10(c, k, o)
    return [int(v) for v in o]


def schedule(seed: int, sweep: int, replica: int = 0):
    ks = (ctypes.c_int * 16)()
    lib().kko_schedule(seed, sweep, replica, ks)
    return [int(v) for v in ks]


def center_draw(seed, sweep, replica, j, kx, ky, x, y):
    d = ctypes.c_int()
    u = ctypes.c_uint32()
    lib().kko_center_draw(seed, sweep, replica, j, kx, ky, x, y, ctypes.byref(d), ctypes.byref(u))
    return int(d.value), int(u.value)


# ----------------------------------------------------------------------- lattice
def count_a_for(N: int, fraction_A: float) -> int:
    return int(lib().kko_count_a_for(N, fraction_A))


def init_block(Lx, Ly, fraction_A):
    a = np.zeros((Ly, Lx), np.uint8)
    lib().kko_init_block(Lx, Ly, fraction_A, _u8(a))
    return a


def init_random(Lx, Ly, fraction_A, seed, replica=0):
    a = np.zeros((Ly, Lx), np.uint8)
    lib().kko_init_random(Lx, Ly, fraction_A, seed, replica, _u8(a))
    return a


def omega_from_gibbs(gAA, gAB, gBB):
    return float(lib().kko_omega_from_gibbs(gAA, gAB, gBB))


def n_ab(lat):
    Ly, Lx = lat.shape
    return int(lib().kko_n_ab(Lx, Ly, _u8(np.ascontiguousarray(lat))))


def gibbs_energy(lat, gAA, gAB, gBB):
    Ly, Lx = lat.shape
    return float(lib().kko_gibbs_energy(Lx, Ly, _u8(np.ascontiguousarray(lat)), gAA, gAB, gBB))


def composition(lat):
    return int(lib().kko_composition(lat.size, _u8(np.ascontiguousarray(lat))))


def delta_nab(lat, c, t):
    Ly, Lx = lat.shape
    return int(lib().kko_delta_nab(Lx, Ly, _u8(np.ascontiguousarray(lat)), c[0], c[1], t[0], t[1]))


def metropolis_accept(dE, u32):
    return bool(lib().kko_metropolis_accept(dE, u32))


# ------------------------------------------------------------------------ sweeps
def run(lat, omega, seed, n_sweeps, first_sweep=0, replica=0):
    """Run ``n_sweeps`` MPKK sweeps in place; returns the accumulated stats."""
    Ly, Lx = lat.shape
    st = Stats()
    lib().kko_run(Lx, Ly, _u8(lat), omega, seed, first_sweep, n_sweeps, replica, ctypes.byref(st))
    return st.as_dict()


def iteration_ordered(lat, omega, seed, sweep, replica, j, order):
    Ly, Lx = lat.shape
    order = np.ascontiguousarray(order, dtype=np.int64)
    st = Stats()
    lib().kko_iteration_ordered(Lx, Ly, _u8(lat), omega, seed, sweep, replica, j,
                                order.ctypes.data_as(_i64p), order.size, ctypes.byref(st))
    return st.as_dict()


def window_iterations(win, Ly_global, y_origin, omega, seed, sweep, replica, j0, T,
                      count_r0, count_r1):
    Hw, Lx = win.shape
    st = Stats()
    lib().kko_window_iterations(Lx, Ly_global, y_origin, Hw, _u8(win), omega, seed, sweep,
                                replica, j0, T, count_r0, count_r1, ctypes.byref(st))
    return st.as_dict()


# ---------------------------------------------------------------------- clusters
def cluster_sizes(lat, target=1):
    Ly, Lx = lat.shape
    out = np.zeros(Lx * Ly, np.int64)
    n = lib().kko_clusters(Lx, Ly, _u8(np.ascontiguousarray(lat)), target,
                           out.ctypes.data_as(_i64p))
    return out[:n]


def cluster_histogram(lat, target=1):
    """Sparse cluster-size histogram: sorted list of (size, count)."""
    return sorted(Counter(cluster_sizes(lat, target).tolist()).items())


@dataclass
class Replica:
    lat: np.ndarray
    omega: float
    seed: int
    replica: int = 0
    sweep: int = 0

    def sweeps(self, n):
        st = run(self.lat, self.omega, self.seed, n, self.sweep, self.replica)
        self.sweep += n
        return st
