"""The committed roofline counters (profiles/pass_kernel_counters.json) match
the bench lattice's launch plan and the current pass-kernel sources, so the
bench line's roofline.achieved / frac come from a capture of the kernel that
actually runs (bench.py refuses stale counters; this test fails first)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1309_4349_b200 import kk  # noqa: E402


def test_committed_counters_match_plan_and_sources():
    plan = kk.plan(65536, 65536, iters_per_pass=8, n_sm=148)
    cnt, why = bench.kernel_counters(plan)
    assert cnt is not None, why
    assert 10.0 < cnt["thread_inst_per_update"] < 60.0
    assert 0.0 < cnt["dram_bytes_per_update"] < 1.0


def test_source_fingerprint_is_per_kernel_and_deterministic():
    a = bench.pass_source_sha256("planar")
    assert a != bench.pass_source_sha256("tile")
    assert a == bench.pass_source_sha256("planar")
