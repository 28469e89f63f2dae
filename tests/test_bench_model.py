"""The bench's algorithmic-bytes model against SURVEY.md §8(d) D.3's computed figures (the
roofline denominators the bench reports are only as good as these)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import workloads  # noqa: E402


def test_b_agent_matches_survey_table():
    # B_agent = 4(4Hd*nnz + 4Hd*Hd + 4Hd + 5Hd + 5) + 16Hd + 32
    ps, tiny = workloads.paper_scale(), workloads.tiny()
    assert bench.policy_bytes(ps, 1, 98, split=False) == 68276   # Hd=32 dense
    assert bench.policy_bytes(ps, 1, 30, split=False) == 33460   # nnz ~ 30
    assert bench.policy_bytes(ps, 1, 37, split=False) == 37044   # nnz ~ 37 (C3)
    assert bench.policy_bytes(tiny, 1, 50, split=False) == 7892  # tiny dense


def test_step_bytes_is_survey_b_step():
    # B_step = sum_alive B_agent + H*W/2 + births * 8P (the split's P-row traffic not counted)
    ps = workloads.paper_scale()
    agents, nnz, births = 5000, 50000, 30
    want = 4 * (4 * 32 * nnz) + agents * (4 * (4 * 32 * 32 + 4 * 32 + 5 * 32 + 5) + 16 * 32 + 32) \
        + ps.rows * ps.cols // 2 + births * 8 * ps.n_params
    assert bench.step_bytes(ps, agents, nnz, births) == want
    # SURVEY's C1 dense rows: 68.5 MB at A = 1000 and 560 MB at A = 8192
    assert abs(bench.step_bytes(ps, 1000, 98 * 1000, 0) / 1e6 - 68.5) < 0.5
    assert abs(bench.step_bytes(ps, 8192, 98 * 8192, 0) / 1e6 - 560) < 1.0


def test_split_kernels_partition_the_agent_bytes():
    # the split policy (P row instead of W_hh + b) plus the P rows equal the unsplit policy
    # plus the P traffic the split adds (P written, P and h read: 16Hd + 4Hd + 16Hd bytes)
    ps = workloads.paper_scale()
    a, nnz, Hd = 100, 900, 32
    split = bench.policy_bytes(ps, a, nnz, split=True) + bench.hh_bytes(ps, a)
    assert split - bench.policy_bytes(ps, a, nnz, split=False) == a * (16 * Hd + 4 * Hd + 16 * Hd)
    assert bench.split_policy(ps) and not bench.split_policy(workloads.ensemble())
