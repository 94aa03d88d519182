"""bench.py accounting (CPU): algorithmic FLOPs and compulsory bytes match BASELINE.md §3."""
import pytest

from paper_2002_02145_b200 import measure
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
    assert abs(measure.compulsory_bytes(p, c_log) / 1e6 - mb) < 0.15


def test_all_workloads_parse():
    assert len(ALL) == 4 + 23
    for conv, c_log, _ in ALL.values():
        p = ConvPreset.parse(conv)
        assert p.gemm_block == 16 and 0 < c_log <= p.nIfm


def test_reference_arm_does_not_load_the_product():
    """bench.py --impl reference runs the reference's CPU driver: its process must not map
    libpsconv.so (the descriptor is parsed in pure Python, workloads.py loaded by path)."""
    import subprocess
    import sys
    code = ("import sys, bench; wl = bench._workloads(); d = bench.Desc(wl.ALL['cfg3'][0]); "
            "assert d.flops(128) == 12947816448; "
            "assert bench.run_config('cfg3', wl.ALL['cfg3'][0], 128, d.nImg)['images'] == 56; "
            "assert not any('paper_2002_02145_b200' in m for m in sys.modules), sorted(sys.modules); "
            "maps = open('/proc/self/maps').read(); assert 'libpsconv' not in maps")
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.check_call([sys.executable, "-c", code], cwd=root)


def test_sample_images_cover_every_128_image_group():
    import bench
    assert bench.sample_images(2048) == list(range(0, 2048, 128)) + [2047]
    assert bench.sample_images(28) == [0, 27]
