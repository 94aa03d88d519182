"""Nest-document front end: the reference's textual nest format
(loopnest.hpp:340-523) -> the computation the GPU path runs. CPU-only (parsing/recognition)."""
import os

import pytest

ps = pytest.importorskip("paper_2002_02145_b200")
HERE = os.path.dirname(__file__)
REF_SAMPLES = "/root/reference/proj/samples"


def _read(name):
    with open(os.path.join(HERE, "golden", "nests", name)) as f:
        return f.read()


def test_conv_document_permuted_and_renamed():
    info = ps.parse_nest(_read("conv_cfg3_perm.nest"))
    assert info.kind == "conv"
    assert str(info.preset) == "conv:2,128,128,28,28,3,3,2,2,16"
    assert info.recipe == "perm=kj,ki,oj,ofm_tile,ifm_tile"
    # the recipe is a legal reference recipe for that descriptor
    ps.emit_driver(info.preset, info.recipe)


def test_gemm_document():
    info = ps.parse_nest(_read("gemm_96.nest"))
    assert info.kind == "gemm" and (info.M, info.N, info.K) == (200, 64, 96)
    assert str(info.preset) == "conv:200,64,96,1,1,1,1,1,1,16"


@pytest.mark.skipif(not os.path.isdir(REF_SAMPLES), reason="reference samples not mounted")
def test_reference_samples():
    with open(os.path.join(REF_SAMPLES, "conv2d.nest")) as f:
        info = ps.parse_nest(f.read())
    # samples/conv2d.nest is the reference default preset (presets.hpp:14-23)
    assert info.kind == "conv" and str(info.preset) == "conv:2,32,32,4,4,3,3,1,1,16"
    assert info.recipe == "perm=ofm_tile,ifm_tile,oj,kj,ki"
    with open(os.path.join(REF_SAMPLES, "matmul.nest")) as f:
        info = ps.parse_nest(f.read())
    assert info.kind == "gemm" and (info.M, info.N, info.K) == (4, 4, 4)


@pytest.mark.parametrize("text,msg", [
    ("loop i lower 0 upper 4\nstmt S\nread A[i*i]\nwrite A[i]", "non-affine"),
    ("loop i lower 0 upper N\nstmt S\nwrite A[i]", "unbound parameter"),
    ("loop i lower 0\nstmt S\nwrite A[i]", "lower' and 'upper"),
    ("frobnicate 3\n", "unknown directive"),
    ("param M = 4\nloop i lower 0 upper M\nloop j lower 0 upper M\nstmt S\nread A[i][j]\nwrite C[i][j]",
     "two read operands"),
    ("loop i lower 0 upper 4\nloop j lower 0 upper i\nstmt S\nread A[i][j]\nread B[j][i]\nwrite C[i][j]",
     "non-rectangular"),
])
def test_rejections(text, msg):
    with pytest.raises(ps.ConfigRejectedError) as e:
        ps.parse_nest(text)
    assert msg in str(e.value)
