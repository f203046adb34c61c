"""Thin Python binding of libkk.so (include/kk.h) — argument marshalling only.

Every step of the MPKK path runs in the library's sm_100a
kernels; this module converts numpy arrays / torch streams / device pointers to
the C ABI and raises on any non-zero status.  There is no CPU fallback: if the
library or a CUDA device is missing, the calls fail loudly.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkk.so")

KK_INIT_RANDOM, KK_INIT_BLOCK, KK_INIT_EMPTY = 0, 1, 2
REGION_ALL, REGION_INTERIOR, REGION_BOUNDARY = 0, 1, 2

_i64 = ctypes.c_int64
_p = ctypes.c_void_p


class KKError(RuntimeError):
    pass


class Config(ctypes.Structure):
    _fields_ = [("Lx", ctypes.c_int64), ("Ly", ctypes.c_int64), ("y_begin", ctypes.c_int64),
                ("y_count", ctypes.c_int64), ("replicas", ctypes.c_int64),
                ("fraction_A", ctypes.c_double), ("omega_kT", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("init_mode", ctypes.c_int32),
                ("iters_per_pass", ctypes.c_int32), ("device", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class Plan(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int32), ("iters_per_pass", ctypes.c_int32), ("tile_rows", ctypes.c_int32),
                ("tile_words", ctypes.c_int32), ("tiles_x", ctypes.c_int32), ("bands", ctypes.c_int32),
                ("halo_rows", ctypes.c_int32), ("threads", ctypes.c_int32), ("smem_bytes", ctypes.c_int32),
                ("pass_pdl", ctypes.c_int32), ("ctas", ctypes.c_int64), ("tma_boxes", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


KERNEL_NAMES = {0: "tile", 1: "resident", 2: "band", 3: "cluster", 4: "planar"}


# symbol -> (restype, argtypes); the ABI surface declared in include/kk.h
SIGNATURES = {
    "kk_create": (ctypes.c_int, [ctypes.POINTER(_p), _i64, _i64, ctypes.c_double, ctypes.c_double, ctypes.c_uint64]),
    "kk_create_ex": (ctypes.c_int, [ctypes.POINTER(_p), ctypes.POINTER(Config)]),
    "kk_plan_config": (ctypes.c_int, [ctypes.POINTER(Config), ctypes.c_int, ctypes.POINTER(Plan)]),
    "kk_destroy": (ctypes.c_int, [_p]),
    "kk_sweep": (ctypes.c_int, [_p, _i64, _p]),
    "kk_energy": (ctypes.c_int, [_p, _p, _p, _p, _p]),
    "kk_composition": (ctypes.c_int, [_p, _p, _p]),
    "kk_stats": (ctypes.c_int, [_p, _p, ctypes.c_int, _p]),
    "kk_cluster_histogram": (ctypes.c_int, [_p, ctypes.c_int, _p, _i64, ctypes.POINTER(_i64), _p]),
    "kk_cluster_slab": (ctypes.c_int, [_p, ctypes.c_int, _p, _i64, ctypes.POINTER(_i64), _p, _p, _p, _i64,
                                       ctypes.POINTER(_i64), _p]),
    "kk_cluster_join": (ctypes.c_int, [_i64, _i64, _p, _p, _p, _p, _i64, _p, _i64, ctypes.POINTER(_i64), _p]),
    "kk_get_lattice": (ctypes.c_int, [_p, _p, _p]),
    "kk_set_lattice": (ctypes.c_int, [_p, _p, _p]),
    "kk_get_lattice_packed": (ctypes.c_int, [_p, _p, _p]),
    "kk_set_lattice_packed": (ctypes.c_int, [_p, _p, _p]),
    "kk_copy_lattice_packed_device": (ctypes.c_int, [_p, _p, ctypes.c_int, _p, _p]),
    "kk_acceptance_table": (ctypes.c_int, [_p, _p]),
    "kk_init_select_hist": (ctypes.c_int, [_p, ctypes.c_int, _p, _p, _p]),
    "kk_init_select_ties": (ctypes.c_int, [_p, _p, _p, _i64, ctypes.POINTER(_i64), _p]),
    "kk_init_select_apply": (ctypes.c_int, [_p, _p, _p, _p]),
    "kk_words_per_row": (ctypes.c_int, [_p, ctypes.POINTER(_i64)]),
    "kk_halo_rows": (ctypes.c_int, [_p, ctypes.POINTER(_i64)]),
    "kk_sweep_index": (ctypes.c_int, [_p, ctypes.POINTER(_i64)]),
    "kk_pack_halo": (ctypes.c_int, [_p, _p, _p, _p]),
    "kk_pass": (ctypes.c_int, [_p, ctypes.c_int, _p, _p, _p]),
    "kk_pass_commit": (ctypes.c_int, [_p]),
    "kk_upload_packed_async": (ctypes.c_int, [_p, _p, _p]),
    "kk_commit_upload": (ctypes.c_int, [_p, _p]),
    "kk_snapshot": (ctypes.c_int, [_p, _p]),
    "kk_download_packed_async": (ctypes.c_int, [_p, _p, _p]),
    "kk_init_select_choose": (ctypes.c_int, [ctypes.c_int, _p, _i64, _p, _p]),
    "kk_init_select_cut": (ctypes.c_int, [_p, _i64, _i64, _p, _p]),
    "kk_hist_merge": (ctypes.c_int, [_p, _i64, _p, _i64, ctypes.POINTER(_i64)]),
    "kk_launch_count": (ctypes.c_int64, []),
    "kk_last_error": (ctypes.c_char_p, []),
    "kk_version": (ctypes.c_char_p, []),
}

_lib = None


def load(path: str = None):
    """Load libkk.so (raises if it was not built — no fallback).  KK_LIB may
    point at an alternative build of the same library (tuning experiments)."""
    global _lib
    if path is None:
        path = os.environ.get("KK_LIB", LIB_PATH)
    if _lib is None:
        if not os.path.exists(path):
            raise KKError(f"{path} not found: build it with `python -m paper_1309_4349_b200.build`")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        msg = load().kk_last_error().decode(errors="replace")
        raise KKError(f"{what} failed ({rc}): {msg}")


def stream_ptr(stream) -> Optional[int]:
    """torch.cuda.Stream | int | None -> cudaStream_t as an int."""
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


def cluster_join(Lx: int, nslabs: int, top_ids: int, bot_ids: int, offsets, sizes: int, n_nodes: int,
                 stream=None):
    """Merged open clusters across slab boundaries: rows [(size, count)]."""
    lib = load()
    n = _i64()
    off = np.ascontiguousarray(offsets, np.int64)
    cap = 4096
    while True:
        buf = np.zeros((cap, 2), np.int64)
        rc = lib.kk_cluster_join(int(Lx), int(nslabs), top_ids, bot_ids, off.ctypes.data, sizes, int(n_nodes),
                                 buf.ctypes.data, cap, ctypes.byref(n), stream_ptr(stream))
        if rc == -4 and n.value > cap:
            cap = int(n.value)
            continue
        _check(rc, "kk_cluster_join")
        return buf[: n.value]


def select_choose(level: int, hist: np.ndarray, need: np.ndarray, prefix: np.ndarray):
    """kk_init_select_choose: one radix-select level (need, prefix updated in place)."""
    hist = np.ascontiguousarray(hist, np.int64)
    assert need.dtype == np.int64 and prefix.dtype == np.uint32 and need.flags["C_CONTIGUOUS"]
    _check(load().kk_init_select_choose(int(level), hist.ctypes.data, int(hist.shape[0]), need.ctypes.data,
                                        prefix.ctypes.data), "kk_init_select_choose")


def select_cut(ties: np.ndarray, replicas: int, need: np.ndarray) -> np.ndarray:
    """kk_init_select_cut: per replica, index of the last tie taken + 1."""
    ties = np.ascontiguousarray(ties, np.int64).reshape(-1, 2)
    need = np.ascontiguousarray(need, np.int64)
    cut = np.zeros(replicas, np.int64)
    _check(load().kk_init_select_cut(ties.ctypes.data if len(ties) else None, len(ties), int(replicas),
                                     need.ctypes.data, cut.ctypes.data), "kk_init_select_cut")
    return cut


def hist_merge(rows) -> list:
    """kk_hist_merge: (size, count) pairs in any order -> sorted merged histogram."""
    rows = np.ascontiguousarray(np.asarray(rows, np.int64).reshape(-1, 2))
    out = np.zeros((max(len(rows), 1), 2), np.int64)
    n = _i64()
    _check(load().kk_hist_merge(rows.ctypes.data if len(rows) else None, len(rows), out.ctypes.data, len(out),
                                ctypes.byref(n)), "kk_hist_merge")
    return [tuple(r) for r in out[: n.value].tolist()]


def plan(Lx: int, Ly: int, replicas: int = 1, iters_per_pass: int = 0, y_begin: int = 0,
         y_count: Optional[int] = None, n_sm: int = 148, init: int = KK_INIT_EMPTY) -> dict:
    """kk_plan_config: the kernel and launch shape kk_create would choose (no
    GPU needed when n_sm > 0)."""
    cfg = Config(Lx=Lx, Ly=Ly, y_begin=y_begin, y_count=Ly if y_count is None else y_count, replicas=replicas,
                 fraction_A=0.5, omega_kT=0.5, seed=1, init_mode=init, iters_per_pass=iters_per_pass,
                 device=-1, reserved=0)
    out = Plan()
    _check(load().kk_plan_config(ctypes.byref(cfg), int(n_sm), ctypes.byref(out)), "kk_plan_config")
    d = {name: getattr(out, name) for name, _ in Plan._fields_ if name != "reserved"}
    d["kernel"] = KERNEL_NAMES[d["kernel"]]
    return d


def launch_count() -> int:
    return int(load().kk_launch_count())


class Lattice:
    """One handle: `replicas` independent Lx x Ly lattices, or a row slab of a
    larger lattice (multi-GPU).  Mirrors the C ABI call for call."""

    def __init__(self, Lx: int, Ly: int, fraction_A: float, omega_kT: float, seed: int,
                 replicas: int = 1, init: int = KK_INIT_RANDOM, iters_per_pass: int = 0,
                 y_begin: int = 0, y_count: Optional[int] = None, device: int = -1):
        lib = load()
        self.Lx, self.Ly, self.replicas = int(Lx), int(Ly), int(replicas)
        self.y_begin = int(y_begin)
        self.rows = int(Ly if y_count is None else y_count)
        self.omega = float(omega_kT)
        cfg = Config(Lx=self.Lx, Ly=self.Ly, y_begin=self.y_begin, y_count=self.rows,
                     replicas=self.replicas, fraction_A=float(fraction_A), omega_kT=self.omega,
                     seed=int(seed) & 0xFFFFFFFFFFFFFFFF, init_mode=int(init),
                     iters_per_pass=int(iters_per_pass), device=int(device), reserved=0)
        h = _p()
        _check(lib.kk_create_ex(ctypes.byref(h), ctypes.byref(cfg)), "kk_create_ex")
        self._h = h
        w = _i64()
        _check(lib.kk_words_per_row(h, ctypes.byref(w)), "kk_words_per_row")
        self.W = int(w.value)
        hy = _i64()
        _check(lib.kk_halo_rows(h, ctypes.byref(hy)), "kk_halo_rows")
        self.halo_rows = int(hy.value)

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            load().kk_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # -- hot path
    def sweep(self, n: int = 1, stream=None):
        _check(load().kk_sweep(self._h, int(n), stream_ptr(stream)), "kk_sweep")

    def pack_halo(self, send_top: int, send_bot: int, stream=None):
        _check(load().kk_pack_halo(self._h, send_top, send_bot, stream_ptr(stream)), "kk_pack_halo")

    def run_pass(self, region: int, halo_top: Optional[int], halo_bot: Optional[int], stream=None):
        _check(load().kk_pass(self._h, int(region), halo_top, halo_bot, stream_ptr(stream)), "kk_pass")

    def pass_commit(self):
        _check(load().kk_pass_commit(self._h), "kk_pass_commit")

    # -- observables
    def energy(self, halo_bot: Optional[int] = None, stream=None):
        nab = np.zeros(self.replicas, np.int64)
        e = np.zeros(self.replicas, np.float64)
        _check(load().kk_energy(self._h, nab.ctypes.data, e.ctypes.data, halo_bot, stream_ptr(stream)),
               "kk_energy")
        return nab, e

    def composition(self, stream=None):
        na = np.zeros(self.replicas, np.int64)
        _check(load().kk_composition(self._h, na.ctypes.data, stream_ptr(stream)), "kk_composition")
        return na

    def stats(self, reset: bool = False, stream=None):
        out = np.zeros((self.replicas, 4), np.int64)
        _check(load().kk_stats(self._h, out.ctypes.data, int(reset), stream_ptr(stream)), "kk_stats")
        return out

    def cluster_histogram(self, target: int = 1, stream=None):
        """Per replica: sorted list of (size, count)."""
        lib = load()
        n = _i64()
        # start from twice the last size seen: a too-small buffer makes the
        # library relabel the lattice on the retry
        cap = max(8192, 2 * getattr(self, "_hist_rows", 0))
        while True:
            buf = np.zeros((cap, 3), np.int64)
            rc = lib.kk_cluster_histogram(self._h, int(target), buf.ctypes.data, cap, ctypes.byref(n),
                                          stream_ptr(stream))
            self._hist_rows = max(getattr(self, "_hist_rows", 0), int(n.value))
            if rc == -4 and n.value > cap:
                cap = int(n.value)
                continue
            _check(rc, "kk_cluster_histogram")
            break
        rows = buf[: n.value]
        # rows are sorted by replica: split at the replica boundaries
        cuts = np.searchsorted(rows[:, 0], np.arange(self.replicas + 1))
        sizes, counts = rows[:, 1].tolist(), rows[:, 2].tolist()
        return [list(zip(sizes[cuts[r]:cuts[r + 1]], counts[cuts[r]:cuts[r + 1]]))
                for r in range(self.replicas)]

    def cluster_histogram_total(self, target: int = 1, stream=None):
        """Cluster-size histogram summed over all replicas: sorted [(size, count)]
        (the ensemble statistics of a replica batch; numpy aggregation of the
        per-replica rows, no per-row Python work)."""
        rows = self.cluster_histogram_raw(target, capacity=max(1 << 16, 2 * getattr(self, "_hist_rows", 0)),
                                          stream=stream)
        self._hist_rows = max(getattr(self, "_hist_rows", 0), len(rows))
        if len(rows) == 0:
            return []
        sizes, inv = np.unique(rows[:, 1], return_inverse=True)
        counts = np.zeros(len(sizes), np.int64)
        np.add.at(counts, inv, rows[:, 2])
        return list(zip(sizes.tolist(), counts.tolist()))

    def cluster_histogram_raw(self, target: int = 1, capacity: int = 1 << 16, stream=None):
        """Rows (replica, size, count) as an int64 array (no per-replica lists)."""
        lib = load()
        n = _i64()
        buf = np.zeros((capacity, 3), np.int64)
        rc = lib.kk_cluster_histogram(self._h, int(target), buf.ctypes.data, capacity, ctypes.byref(n),
                                      stream_ptr(stream))
        if rc == -4:
            return self.cluster_histogram_raw(target, int(n.value), stream)
        _check(rc, "kk_cluster_histogram")
        return buf[: n.value]

    # -- distributed random start (include/kk.h kk_init_select_*)
    def select_hist(self, level: int, prefix: Optional[np.ndarray]):
        out = np.zeros((self.replicas, 2048), np.int64)
        pre = None if prefix is None else np.ascontiguousarray(prefix, np.uint32)
        _check(load().kk_init_select_hist(self._h, int(level), None if pre is None else pre.ctypes.data,
                                          out.ctypes.data, None), "kk_init_select_hist")
        return out

    def select_ties(self, K: np.ndarray, capacity: int = 1024):
        K = np.ascontiguousarray(K, np.uint32)
        n = _i64()
        while True:
            out = np.zeros((max(capacity, 1), 2), np.int64)
            rc = load().kk_init_select_ties(self._h, K.ctypes.data, out.ctypes.data, capacity,
                                            ctypes.byref(n), None)
            if rc == -4:
                capacity = int(n.value)
                continue
            _check(rc, "kk_init_select_ties")
            return out[: n.value]

    def select_apply(self, K: np.ndarray, cut: np.ndarray):
        K = np.ascontiguousarray(K, np.uint32)
        cut = np.ascontiguousarray(cut, np.int64)
        _check(load().kk_init_select_apply(self._h, K.ctypes.data, cut.ctypes.data, None),
               "kk_init_select_apply")

    def cluster_slab(self, target: int, top_ids: int, bot_ids: int, open_sizes: int, open_cap: int,
                     stream=None):
        """Slab-local clusters: returns (complete rows [(size, count)], n_open)."""
        lib = load()
        nh, no = _i64(), _i64()
        cap = max(8192, 2 * getattr(self, "_slab_rows", 0))   # a retry relabels the slab
        while True:
            buf = np.zeros((cap, 2), np.int64)
            rc = lib.kk_cluster_slab(self._h, int(target), buf.ctypes.data, cap, ctypes.byref(nh), top_ids,
                                     bot_ids, open_sizes, int(open_cap), ctypes.byref(no), stream_ptr(stream))
            self._slab_rows = max(getattr(self, "_slab_rows", 0), int(nh.value))
            if rc == -4 and nh.value > cap:
                cap = int(nh.value)
                continue
            _check(rc, "kk_cluster_slab")
            return buf[: nh.value], int(no.value)

    def acceptance_table(self):
        out = np.zeros(7, np.uint32)
        _check(load().kk_acceptance_table(self._h, out.ctypes.data), "kk_acceptance_table")
        return out

    def sweep_index(self) -> int:
        s = _i64()
        _check(load().kk_sweep_index(self._h, ctypes.byref(s)), "kk_sweep_index")
        return int(s.value)

    # -- lattice transfer
    def get_lattice(self, stream=None) -> np.ndarray:
        out = np.zeros((self.replicas, self.rows, self.Lx), np.uint8)
        _check(load().kk_get_lattice(self._h, out.ctypes.data, stream_ptr(stream)), "kk_get_lattice")
        return out

    def set_lattice(self, a: np.ndarray, stream=None):
        a = np.ascontiguousarray(a, dtype=np.uint8).reshape(self.replicas, self.rows, self.Lx)
        _check(load().kk_set_lattice(self._h, a.ctypes.data, stream_ptr(stream)), "kk_set_lattice")

    def get_packed(self, out: Optional[np.ndarray] = None, stream=None) -> np.ndarray:
        if out is None:
            out = np.zeros((self.replicas, self.rows, self.W), np.uint32)
        _check(load().kk_get_lattice_packed(self._h, out.ctypes.data, stream_ptr(stream)),
               "kk_get_lattice_packed")
        return out

    def set_packed(self, a: np.ndarray, stream=None):
        assert a.dtype == np.uint32 and a.flags["C_CONTIGUOUS"] and a.size == self.replicas * self.rows * self.W
        _check(load().kk_set_lattice_packed(self._h, a.ctypes.data, stream_ptr(stream)),
               "kk_set_lattice_packed")

    def set_packed_ptr(self, host_ptr: int, stream=None):
        """Upload from a (pinned) host buffer given by address."""
        _check(load().kk_set_lattice_packed(self._h, host_ptr, stream_ptr(stream)), "kk_set_lattice_packed")

    # -- double-buffered host I/O (include/kk.h kk_upload_packed_async ...)
    def upload_async(self, host_ptr: int, copy_stream=None):
        _check(load().kk_upload_packed_async(self._h, host_ptr, stream_ptr(copy_stream)), "kk_upload_packed_async")

    def commit_upload(self, stream=None):
        _check(load().kk_commit_upload(self._h, stream_ptr(stream)), "kk_commit_upload")

    def snapshot(self, stream=None):
        _check(load().kk_snapshot(self._h, stream_ptr(stream)), "kk_snapshot")

    def download_async(self, host_ptr: int, copy_stream=None):
        _check(load().kk_download_packed_async(self._h, host_ptr, stream_ptr(copy_stream)),
               "kk_download_packed_async")

    def copy_packed_device(self, dev_ptr: int, to_lattice: bool, stream=None):
        if to_lattice:
            rc = load().kk_copy_lattice_packed_device(self._h, None, 1, dev_ptr, stream_ptr(stream))
        else:
            rc = load().kk_copy_lattice_packed_device(self._h, dev_ptr, 0, None, stream_ptr(stream))
        _check(rc, "kk_copy_lattice_packed_device")
