"""Host-side steps of the C ABI (no GPU): the distributed random start's bin
choice and tie cut (kk_init_select_choose / kk_init_select_cut, R7)
and the cluster-histogram merge (kk_hist_merge, R9), each pinned against its
plain definition written out with numpy / Python on random inputs."""
import numpy as np
import pytest

from paper_1309_4349_b200 import kk


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_1309_4349_b200 import build
    build.build()


def _choose_def(level, hist, need, prefix):
    """Smallest bin whose cumulative count reaches need; need -> rank in bin."""
    nb = 1024 if level == 2 else 2048
    need, prefix = need.copy(), prefix.astype(np.uint64).copy()
    for r in range(hist.shape[0]):
        cum = 0
        b = 0
        while b < nb - 1 and cum + hist[r, b] < need[r]:
            cum += hist[r, b]
            b += 1
        need[r] -= cum
        prefix[r] = ((prefix[r] << (10 if level == 2 else 11)) | b) & 0xFFFFFFFF
    return need, prefix.astype(np.uint32)


@pytest.mark.parametrize("level", [0, 1, 2])
def test_select_choose_matches_definition(level):
    rng = np.random.default_rng(level)
    R = 7
    hist = rng.integers(0, 5, (R, 2048)).astype(np.int64)
    hist[3] = 0
    hist[3, 17] = 9                      # a single populated bin
    tot = hist[:, : (1024 if level == 2 else 2048)].sum(1)
    need = np.array([1 + rng.integers(0, max(int(t), 1)) for t in tot], np.int64)
    need[3] = 9
    prefix = rng.integers(0, 1 << 20, R).astype(np.uint32)
    exp_need, exp_prefix = _choose_def(level, hist, need, prefix)
    kk.select_choose(level, hist, need, prefix)
    assert np.array_equal(need, exp_need) and np.array_equal(prefix, exp_prefix)
    assert prefix[3] & 0x3FF == 17 if level == 2 else prefix[3] & 0x7FF == 17


def test_select_cut_matches_definition():
    rng = np.random.default_rng(5)
    R = 5
    ties = np.stack([rng.integers(0, R, 300), rng.choice(10**9, 300, replace=False)], 1).astype(np.int64)
    need = np.array([int((ties[:, 0] == r).sum()) // 2 for r in range(R)], np.int64)
    need[1] = 0
    cut = kk.select_cut(ties, R, need)
    for r in range(R):
        idx = np.sort(ties[ties[:, 0] == r, 1])
        assert cut[r] == (idx[need[r] - 1] + 1 if need[r] > 0 else 0)
    need[2] = 10**6                      # more than there are ties
    with pytest.raises(kk.KKError):
        kk.select_cut(ties, R, need)


def test_hist_merge_matches_definition():
    rng = np.random.default_rng(9)
    rows = np.stack([rng.integers(1, 40, 500), rng.integers(0, 7, 500)], 1)
    exp = {}
    for sz, c in rows.tolist():
        exp[sz] = exp.get(sz, 0) + c
    assert kk.hist_merge(rows) == sorted((s, c) for s, c in exp.items() if c)
    assert kk.hist_merge(np.zeros((0, 2), np.int64)) == []
