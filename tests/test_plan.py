"""Host-side execution planning (kk_plan_config, no GPU needed): which kernel
kk_sweep launches and the tile shape the cost model picks.  The plan never
changes results (the GPU parity tests run every kernel against the oracle);
these checks pin the decisions DESIGN.md documents and the invariants every
plan must satisfy."""
import itertools
import os

import pytest

from paper_1309_4349_b200 import kk

SMEM_2_PER_SM = 113 * 1024     # two 512-thread tile CTAs per SM (228 KB per SM)


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_1309_4349_b200 import build
    build.build()
    saved = {k: os.environ.pop(k, None) for k in ("KK_RESIDENT", "KK_BAND", "KK_THI", "KK_TWI", "KK_T", "KK_PLANAR",
                                                  "KK_RES_THREADS", "KK_PASS_THREADS", "KK_CLUSTER", "KK_CLUSTER_TB",
                                                  "KK_BAND_TB")}
    yield
    for k, v in saved.items():
        if v is not None:
            os.environ[k] = v


def test_bench_lattice_plan(monkeypatch):
    p = kk.plan(65536, 65536)
    assert p["kernel"] == "planar" and p["iters_per_pass"] == 8 and p["halo_rows"] == 24
    assert p["tile_words"] == 128 and 300 <= p["tile_rows"] <= 400   # widest TMA tile, as tall as fits
    assert p["smem_bytes"] <= 227 * 1024 and p["tma_boxes"] >= 1
    assert p["ctas"] == p["tiles_x"] * p["bands"] >= 148 * 16
    assert p["threads"] == 768
    assert p["pass_pdl"] == 0                       # early CTAs would idle in slots
    # the row-major tile kernel's plan (KK_PLANAR=0; every lattice with Lx % 128 != 0)
    monkeypatch.setenv("KK_PLANAR", "0")
    t = kk.plan(65536, 65536)
    assert t["kernel"] == "tile" and t["tile_words"] == 64 and 540 <= t["tile_rows"] <= 600
    assert SMEM_2_PER_SM < t["smem_bytes"] <= 227 * 1024 and t["threads"] == 640 and t["pass_pdl"] == 0
    monkeypatch.setenv("KK_TALL", "0")              # two CTAs per SM: the cost-model tiles
    q = kk.plan(65536, 65536)
    monkeypatch.delenv("KK_TALL")
    assert q["tile_words"] == 64 and 300 <= q["tile_rows"] <= 340 and q["smem_bytes"] <= SMEM_2_PER_SM
    assert q["threads"] == 384                      # many waves: 80-register CTAs
    assert kk.plan(16384, 16384)["threads"] == 512  # too few waves for tall tiles
    monkeypatch.delenv("KK_PLANAR")


def test_planar_cost_model_picks_the_measured_shapes():
    """The refitted planar cost model (halo groups weighted; 512-thread CTAs
    for one-wave grids with <= 512 items per iteration) reproduces the shapes
    measured fastest on a B200 after the R6 revision (planar
    kernel: 4096^2 64 x 56 at 512 threads 352 vs 32 x 112 326 G/s; 8192^2
    128 x 112 574 vs 64 x 224 555; 16384^2 128 x 224 666; 65536^2 128 x 340)."""
    want = {4096: (64, 56, 512), 8192: (128, 112, 768), 16384: (128, 224, 768), 65536: (128, 340, 768)}
    for L, (twi, thi, nt) in want.items():
        p = kk.plan(L, L, n_sm=148)
        assert (p["kernel"], p["tile_words"], p["tile_rows"], p["threads"]) == ("planar", twi, thi, nt), (L, p)


def test_mid_size_lattice_fills_every_sm(monkeypatch):
    p = kk.plan(4096, 4096)
    assert p["kernel"] == "planar" and p["ctas"] >= 128
    assert p["pass_pdl"] == 1                       # one wave: next pass launches under this one
    assert kk.plan(5120, 5120)["kernel"] == "planar"
    r = kk.plan(2048, 2048)                         # too few 32-centre items: row-major tile kernel
    assert r["kernel"] == "tile" and r["ctas"] <= 296 and r["threads"] == 384 and r["pass_pdl"] == 1
    assert kk.plan(8192, 8192)["kernel"] == "planar"   # the planar kernel replaced the band kernel
    assert kk.plan(16384, 16384)["kernel"] == "planar"
    q = kk.plan(12000, 8192)                        # rows not whole 128-site groups: band kernel
    assert q["kernel"] == "band" and q["ctas"] == 148 and q["threads"] == 1024
    monkeypatch.setenv("KK_PLANAR", "0")
    assert kk.plan(8192, 8192)["kernel"] == "band"
    assert kk.plan(4096, 4096)["threads"] == 640    # one wave, > 384 items per iteration
    assert kk.plan(16384, 16384)["kernel"] == "tile"   # bands no longer fit in shared memory
    monkeypatch.setenv("KK_PLANAR", "2")            # planar whenever the rows allow
    assert kk.plan(1024, 1024)["kernel"] == "planar"


def test_small_and_replica_batches_are_resident():
    assert kk.plan(64, 64)["kernel"] == "resident"
    assert kk.plan(400, 400)["kernel"] == "cluster"              # the paper's lattice: one 16-CTA cluster
    assert kk.plan(400, 400)["ctas"] == 16
    assert kk.plan(400, 400, replicas=4)["ctas"] == 4 * 16      # up to 4 replicas: 16-CTA clusters
    assert kk.plan(400, 400, replicas=5)["ctas"] == 5 * 8
    assert kk.plan(256, 256)["ctas"] == 8                        # < 320 rows: 8-CTA clusters
    assert kk.plan(400, 400, replicas=16)["ctas"] == 16 * 8     # 16 clusters of 8 CTAs fit on 148 SMs
    assert kk.plan(400, 400, replicas=37)["ctas"] == 37 * 4     # then clusters of 4, of 2
    assert kk.plan(400, 400, replicas=74)["ctas"] == 74 * 2
    assert kk.plan(400, 400, replicas=75)["kernel"] == "resident"  # enough replicas to fill SMs one each
    p = kk.plan(400, 400, replicas=1024)                           # BASELINE configs[3]
    assert p["kernel"] == "resident" and p["ctas"] == 1024 and p["threads"] == 256
    assert kk.plan(400, 400, replicas=100)["threads"] == 512     # all replicas co-resident
    assert kk.plan(1024, 1024)["kernel"] == "tile"                # one replica too big to stay resident
    assert kk.plan(1024, 1024, replicas=148)["kernel"] == "resident"


def test_slabs_never_use_the_resident_or_band_kernels():
    p = kk.plan(65536, 8 * 65536, y_begin=65536, y_count=65536)
    assert p["kernel"] == "planar"
    q = kk.plan(400, 800, y_begin=400, y_count=400)
    assert q["kernel"] == "tile"


def test_overrides(monkeypatch):
    monkeypatch.setenv("KK_CLUSTER", "0")
    assert kk.plan(400, 400)["kernel"] == "resident"
    monkeypatch.setenv("KK_CLUSTER", "16")
    assert kk.plan(400, 400)["ctas"] == 16
    monkeypatch.delenv("KK_CLUSTER")
    monkeypatch.setenv("KK_RESIDENT", "0")
    assert kk.plan(400, 400)["kernel"] == "tile"
    monkeypatch.setenv("KK_BAND", "2")
    assert kk.plan(4096, 4096)["kernel"] == "band"
    assert kk.plan(4096, 4096)["ctas"] == 148
    monkeypatch.setenv("KK_BAND", "0")
    assert kk.plan(12000, 8192)["kernel"] == "tile"
    monkeypatch.delenv("KK_BAND")
    monkeypatch.delenv("KK_RESIDENT")
    monkeypatch.setenv("KK_THI", "64")
    monkeypatch.setenv("KK_TWI", "16")
    p = kk.plan(65536, 65536)
    assert (p["tile_rows"], p["tile_words"]) == (64, 16)
    monkeypatch.setenv("KK_THI", "100000")   # cannot fit in shared memory
    with pytest.raises(kk.KKError):
        kk.plan(65536, 65536)


@pytest.mark.parametrize("Lx,Ly,R,T", list(itertools.product([4, 36, 64, 100, 400, 1000, 4096, 65536],
                                                               [4, 12, 400, 4096, 65536], [1, 3],
                                                               [0, 1, 4])))
def test_plan_invariants(Lx, Ly, R, T):
    if Lx * Ly * R > 65536 * 65536:
        pytest.skip("beyond one GPU")
    p = kk.plan(Lx, Ly, replicas=R, iters_per_pass=T)
    W = (Lx + 31) // 32
    assert p["tile_rows"] % 4 == 0 and p["tile_rows"] * p["bands"] >= Ly
    assert p["tile_rows"] * (p["bands"] - 1) < Ly                 # no empty band
    assert p["tile_words"] * p["tiles_x"] >= W and p["tile_words"] * (p["tiles_x"] - 1) < W
    assert 0 < p["smem_bytes"] <= 227 * 1024
    assert p["halo_rows"] == 3 * (T or 8)
    if p["kernel"] == "tile":
        assert p["ctas"] == p["tiles_x"] * p["bands"] * R
        assert p["smem_bytes"] <= SMEM_2_PER_SM or os.environ.get("KK_THI") or p["threads"] == 640
    elif p["kernel"] == "planar":
        assert Lx % 128 == 0 and Lx * Ly * R >= 1 << 24
        assert p["ctas"] == p["tiles_x"] * p["bands"] * R and p["tile_words"] % 4 == 0
        assert p["threads"] in (512, 640, 768, 896)
    elif p["kernel"] == "resident":
        assert p["ctas"] == R and Lx >= 64 and p["threads"] in (128, 256, 512)
    elif p["kernel"] == "cluster":
        assert p["ctas"] % R == 0 and p["ctas"] // R in (2, 4, 8, 16) and p["ctas"] <= 148 and Ly >= 192


def test_invalid_configs_fail_without_a_gpu():
    for bad in [dict(Lx=10, Ly=8), dict(Lx=8, Ly=6), dict(Lx=8, Ly=8, iters_per_pass=3),
                dict(Lx=8, Ly=16, y_begin=2, y_count=8)]:
        with pytest.raises(kk.KKError):
            kk.plan(**bad)
