"""bench.py accounting (CPU): algorithmic FLOPs and compulsory bytes match BASELINE.md §3."""
import pytest

import bench
from paper_2002_02145_b200 import ConvPreset
from paper_2002_02145_b200.workloads import ALL


@pytest.mark.parametrize("name,gflop,mb", [
    ("cfg1", 6.47, 45.1), ("cfg2", 2.88, 112.5), ("cfg3", 12.95, 113.0), ("cfg5", 473.52, 824.4),
    ("r50_stem", 60.42, 1644.4), ("r50_l2_ds_1x1s2_256_512", 52.61, 617.1),
    ("r50_l4_3x3_512_512", 59.19, 60.8),
])
def test_flops_and_bytes_match_baseline_md(name, gflop, mb):
    conv, c_log, _ = ALL[name]
    p = ConvPreset.parse(conv)
    assert abs(p.flops(c_log) / 1e9 - gflop) < 0.01
    assert abs(bench.compulsory_bytes(p, c_log) / 1e6 - mb) < 0.15


def test_all_workloads_parse():
    assert len(ALL) == 4 + 23
    for conv, c_log, _ in ALL.values():
        p = ConvPreset.parse(conv)
        assert p.gemm_block == 16 and 0 < c_log <= p.nIfm
