"""Pins for the oracle's Philox4x32-10 (north_star part 3; reading R6).

Pinned against (a) the Random123 known-answer vectors (tests/golden) and
(b) an independent implementation: Triton's numpy interpreter of
``tl.randint4x`` (counter = (offset, 0, 0, 0), key = (seed lo, seed hi)).
"""
import math
import os
import subprocess
import sys

import pytest

from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def _kat_rows():
    rows = []
    with open(GOLDEN) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(t, 16) for t in line.split()]
            rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,out", _kat_rows())
def test_philox_known_answers(ctr, key, out):
    assert O.philox4x32_10(ctr, key) == out


_TRITON_SCRIPT = r"""
import os, sys
os.environ["TRITON_INTERPRET"] = "1"
import torch, triton, triton.language as tl
@triton.jit
def k(out, seed, N: tl.constexpr):
    off = tl.arange(0, N)
    a, b, c, d = tl.randint4x(seed, off, n_rounds=10)
    tl.store(out + off * 4 + 0, a); tl.store(out + off * 4 + 1, b)
    tl.store(out + off * 4 + 2, c); tl.store(out + off * 4 + 3, d)
seed = int(sys.argv[1])
o = torch.zeros(64 * 4, dtype=torch.int32)
k[(1,)](o, seed, N=64)
print(" ".join(str(v & 0xFFFFFFFF) for v in o.tolist()))
"""


@pytest.mark.parametrize("seed", [0, 12345, 0x1234_5678_9ABC])
def test_philox_matches_triton_interpreter(seed):
    try:
        import triton  # noqa: F401
    except Exception:
        pytest.skip("triton not importable")
    r = subprocess.run([sys.executable, "-c", _TRITON_SCRIPT, str(seed)],
                       capture_output=True, text=True, timeout=600)
    if r.returncode != 0:
        pytest.skip("triton interpreter unavailable: " + r.stderr[-200:])
    ref = [int(t) for t in r.stdout.split()]
    key = (seed & 0xFFFFFFFF, seed >> 32)
    for off in range(64):
        assert O.philox4x32_10((off, 0, 0, 0), key) == ref[4 * off:4 * off + 4]


def test_schedule_and_draw_layout():
    """k_j are the 16 nibbles of words 0,1 of philox((0,0,s,tag 0x10)); the
    centre draw (reading R6) takes the centre's word w from
    philox(2g+(p>>2), l, s, c3)[p&3] and splits 6 w = d 2^32 + u32 into the
    direction d and the acceptance uniform u32 — checked against Philox."""
    seed, s = 987654321, 17
    key = (seed & 0xFFFFFFFF, seed >> 32)
    w = O.philox4x32_10((0, 0, s, 0x10), key)
    ks = O.schedule(seed, s)
    assert ks == [(w[j // 8] >> (4 * (j % 8))) & 15 for j in range(16)]
    for (x, y, kx, ky, j) in [(1, 2, 1, 2, 3), (5, 2, 1, 2, 3), (12, 8, 0, 0, 15), (31, 35, 3, 3, 0),
                              (157, 6, 1, 2, 9), (4096 + 28, 40, 0, 0, 7)]:
        i, l = (x - kx) // 4, (y - ky) // 4
        g, p = i >> 3, i & 7
        c3 = (2 << 8) | j
        ww = O.philox4x32_10((2 * g + (p >> 2), l, s, c3), key)[p & 3]
        d, uu = O.center_draw(seed, s, 2, j, kx, ky, x, y)
        assert d == (6 * ww) >> 32 and 0 <= d < 6
        assert uu == (6 * ww) % 2 ** 32


@pytest.mark.parametrize("omega", [0.2, 0.5, 0.6, 1.0, 2.5])
def test_split_word_acceptance_is_boltzmann_for_every_direction(omega):
    """R6's split 6 w = d 2^32 + u32 of a uniform 32-bit w: for every direction
    d the probability that u32 passes the acceptance rule (u32 2^-32 <
    exp(-dE)) is exp(-dE) to within 8 * 2^-32 — so the acceptance law does not
    depend on the proposed direction (detailed balance).
    Counted exactly: the w of class d are the integers in [d 2^32 / 6,
    (d+1) 2^32 / 6), and u32 = 6 w - d 2^32 steps by 6 over them."""
    two32 = 2 ** 32
    for dn in [2, 4, 6]:
        pe = math.exp(-omega * dn)
        for d in range(6):
            lo = -(-d * two32 // 6)            # first w of class d
            hi = -(-(d + 1) * two32 // 6)      # first w of class d + 1
            u0 = 6 * lo - d * two32            # its u32 (0, 2 or 4)
            # accepted w: u0 + 6 k < pe 2^32 (the oracle's rule, in exact arithmetic up to fp64 of pe)
            lim = pe * two32
            k_max = math.ceil((lim - u0) / 6)  # number of k >= 0 with u0 + 6k < lim
            n_acc = max(0, min(hi - lo, k_max))
            assert abs(n_acc / (hi - lo) - pe) <= 8 / two32
            # and the oracle's own rule agrees at the boundary of that count
            assert O.metropolis_accept(omega * dn, u0 + 6 * (n_acc - 1))
            assert not O.metropolis_accept(omega * dn, u0 + 6 * n_acc)
