"""C ABI (CPU): the library loads, exports every entry point include/psconv.h declares, and
fails loudly (status 1, message) on GPU entry points when no device is present."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_2002_02145_b200 as ps
from paper_2002_02145_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(ROOT, "include", "psconv.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = set(re.findall(
        r"^(?:const\s+)?(?:int|void|int64_t|double|char)\s*\*?\s*([a-z_0-9]+)\s*\(", txt, flags=re.M))
    return sorted(names)


def test_every_declared_symbol_exported():
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(_lib.lib, n), f"{n} declared in psconv.h but not exported"
    assert set(names) <= set(_lib.EXPORTED), set(names) - set(_lib.EXPORTED)


def test_version_and_last_error():
    assert "sm_100a" in ps.version()
    with pytest.raises(ps.ConfigRejectedError) as e:
        ps.ConvPreset.parse("conv:1,2,3")
    assert "10 integers" in str(e.value)


def test_plan_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(ps.Error):
        ps.ConvPlan(ps.ConvPreset(), "3xtf32", 0)


def test_no_cpu_fallback_in_product():
    """The product package must not import the oracle (test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2002_02145_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".hpp")):
                src = open(os.path.join(root, f)).read()
                assert "import oracle" not in src and "oracle.h" not in src, f


@pytest.mark.parametrize("csv", ["conv:2,32,32,4,4,3,3,1,1,16", "conv:1,16,32,5,7,3,3,2,2,16",
                                 "conv:1,32,16,9,13,1,1,1,1,16"])
def test_cpu_microkernel_contract(csv):
    """gemm_microkernel(out, flt, in) (presets.hpp:116-123) driven by the identity nest equals
    the oracle; brgemm_f32 folds the (ifm_tile, kj, ki) calls into one."""
    p = ps.ConvPreset.parse(csv)
    x = oracle.pad_input(p, oracle.fill_input(p, 3))
    w = oracle.fill_filter(p, 4)
    ref = oracle.conv_fig5(p, x, w)
    mk = ps.gemm_microkernel(p)
    out = np.zeros_like(ref)
    out_br = np.zeros_like(ref)
    fp = ctypes.POINTER(ctypes.c_float)
    Kb, Cb = p.nOfm // 16, p.nIfm // 16
    for img in range(p.nImg):
        for ot in range(Kb):
            for oj in range(p.ofh):
                flts, ins = [], []
                for it in range(Cb):
                    for kj in range(p.kh):
                        for ki in range(p.kw):
                            o = out[img, ot, oj]
                            f = w[ot, it, kj, ki]
                            i = x[img, it, oj * p.stride_h + kj, ki]
                            mk(o.ctypes.data_as(fp), f.ctypes.data_as(fp), i.ctypes.data_as(fp))
                            flts.append(f.ctypes.data)
                            ins.append(i.ctypes.data)
                ps.brgemm(p, out_br[img, ot, oj].ctypes.data, flts, ins)
    assert oracle.rel_l2(out, ref) < 1e-6
    assert oracle.rel_l2(out_br, ref) < 1e-6


def test_microkernel_dispatch_reuses_shapes():
    a = ps.gemm_microkernel(ps.ConvPreset())
    b = ps.gemm_microkernel(ps.ConvPreset())
    assert ctypes.cast(a, ctypes.c_void_p).value == ctypes.cast(b, ctypes.c_void_p).value
