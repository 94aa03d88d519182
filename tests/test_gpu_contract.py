"""GPU tests of the conv_fwd contract (include/psconv.h) beyond numeric parity:

* split-K is deterministic: the partials of a split tile are combined in split order by the
  tile's last unit, so repeated launches are bitwise identical (the reference values
  byte-identical output, /root/reference/proj/README.md:170-172);
* conv_fwd allocates nothing and never synchronises (split-K scratch is plan-owned), so a
  split-K call can be captured into a CUDA graph on its first use;
* the host-buffer entry with a (c,s)-folded plan, the f16x2 input-scale slot under graph
  replay interleaved with eager calls, and the blocked-layout packing entry points
  (conv_pack_input / conv_pack_filter / conv_unpack_output) against numpy.
"""
import numpy as np
import pytest

import oracle
from tests.cases import seeds

torch = pytest.importorskip("torch")
ps = pytest.importorskip("paper_2002_02145_b200")

TOL = {"3xtf32": 1e-5, "tf32": 5e-3, "f16x2": 1e-5}
DEV = "cuda:0"


def _inputs(p, c_log, cfg_id):
    sx, sw = seeds(cfg_id)
    x = torch.empty(p.input_elems(), device=DEV)
    w = torch.empty(p.filter_elems(), device=DEV)
    ps.fill_input(p, sx, x, c_logical=c_log)
    ps.fill_filter(p, sw, w, c_logical=c_log)
    ref = oracle.conv(p, oracle.fill_input(p, sx, c_log), oracle.fill_filter(p, sw, c_log)).ravel()
    return x, w, ref


SPLIT_CASES = [
    # (conv, mode, recipe): tail split, a second round of units, every tile split (kt:1),
    # CTA pairs, two epilogue groups, 3xTF32 chunks with TMEM-resident A
    ("conv:8,64,64,56,56,3,3,1,1,16,1,1,56,56", "tf32", "gpu=bn:64,box:8x8x2,ks:3"),
    ("conv:8,64,64,56,56,3,3,1,1,16,1,1,56,56", "3xtf32", "gpu=bn:64,box:8x8x2,ks:4"),
    ("conv:8,64,64,56,56,3,3,1,1,16,1,1,56,56", "tf32", "gpu=bn:64,box:8x8x2,ks:3,kt:1"),
    ("conv:8,64,64,56,56,3,3,1,1,16,1,1,56,56", "tf32", "gpu=bn:64,box:8x8x2,ks:2,cl:2"),
    ("conv:6,512,512,7,7,3,3,1,1,16,1,1,7,7", "3xtf32", "gpu=bn:256,box:7x1x18,ks:2,eg:2"),
    ("conv:6,512,512,7,7,3,3,1,1,16,1,1,7,7", "tf32", "gpu=bn:128,box:1x7x18,ks:5,kt:1,eg:2"),
    ("conv:6,512,512,7,7,3,3,1,1,16,1,1,7,7", "f16x2", "gpu=bn:256,box:7x1x18,ks:3"),
]


@pytest.mark.gpu
@pytest.mark.parametrize("conv,mode,recipe", SPLIT_CASES)
def test_split_k_bitwise_reproducible(conv, mode, recipe):
    p = ps.ConvPreset.parse(conv)
    x, w, ref = _inputs(p, p.nIfm, 31)
    plan = ps.ConvPlan(p, mode=mode, device=0, recipe=recipe)
    assert "ks:" in plan.recipe, plan.recipe
    ys = [torch.full((p.output_elems(),), float("nan"), device=DEV) for _ in range(6)]
    for y in ys:
        plan.forward(x, w, y)
    torch.cuda.synchronize()
    err = oracle.rel_l2(ys[0].cpu().numpy(), ref)
    assert err <= TOL[mode], f"relL2 {err:.3e} ({plan.recipe})"
    for i, y in enumerate(ys[1:], 1):
        assert torch.equal(y, ys[0]), f"launch {i} differs bitwise from launch 0 ({plan.recipe})"


@pytest.mark.gpu
def test_split_k_accumulate_reproducible():
    """`+=` with every tile split: the combined tile is added once (no per-partial atomics)."""
    p = ps.ConvPreset.parse("conv:6,512,512,7,7,3,3,1,1,16,1,1,7,7")
    x, w, ref = _inputs(p, 512, 32)
    base = torch.randn(p.output_elems(), generator=torch.Generator().manual_seed(3)).to(DEV)
    plan = ps.ConvPlan(p, mode="3xtf32", device=0, recipe="gpu=bn:128,box:1x7x18,ks:3,kt:1")
    outs = []
    for _ in range(3):
        y = base.clone()
        plan.forward(x, w, y, accumulate=True)
        outs.append(y)
    torch.cuda.synchronize()
    assert oracle.rel_l2(outs[0].cpu().numpy(), base.cpu().numpy() + ref) <= 1e-5
    assert all(torch.equal(o, outs[0]) for o in outs)


@pytest.mark.gpu
def test_split_k_first_call_capturable():
    """No allocation or synchronisation inside conv_fwd: the very first call of a fresh
    split-K plan can be captured into a CUDA graph (a cudaMalloc or cudaStreamSynchronize
    under capture would invalidate it)."""
    p = ps.ConvPreset.parse("conv:8,64,64,56,56,3,3,1,1,16,1,1,56,56")
    x, w, ref = _inputs(p, 64, 33)
    plan = ps.ConvPlan(p, mode="tf32", device=0, recipe="gpu=bn:64,box:8x8x2,ks:3")
    y = torch.full((p.output_elems(),), float("nan"), device=DEV)
    side = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        plan.forward(x, w, y, stream=side)
    for _ in range(2):
        y.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert oracle.rel_l2(y.cpu().numpy(), ref) <= TOL["tf32"]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
def test_forward_host_folded_plan(mode):
    """conv_fwd_host with a fold:C plan: the host filter is the caller's UNFOLDED KCRS16c16k
    (kw taps), larger than the plan's folded operand -- it must be staged whole."""
    p = ps.ConvPreset.parse("conv:12,64,16,28,28,7,7,2,2,16,3,3,56,56")
    sx, sw = seeds(34)
    x = oracle.fill_input(p, sx, 3)
    w = oracle.fill_filter(p, sw, 3)
    ref = oracle.conv(p, x, w).ravel()
    plan = ps.ConvPlan(p, mode=mode, device=0, recipe="gpu=bn:64,fold:3")
    assert "fold:3" in plan.recipe
    hy = torch.full((p.output_elems(),), float("nan")).pin_memory()
    plan.forward_host(torch.from_numpy(x.ravel()).pin_memory(), torch.from_numpy(w.ravel()).pin_memory(), hy)
    torch.cuda.synchronize()
    err = oracle.rel_l2(hy.numpy(), ref)
    assert err <= TOL[mode], f"relL2 {err:.3e}"
    yd = torch.full((p.output_elems(),), float("nan"), device=DEV)
    plan.forward(torch.from_numpy(x.ravel()).to(DEV), torch.from_numpy(w.ravel()).to(DEV), yd)
    torch.cuda.synchronize()
    assert torch.equal(yd.cpu(), hy), "host path differs from the device path"


@pytest.mark.gpu
def test_f16x2_graph_replay_interleaved_with_eager():
    """f16x2 derives a power-of-two input scale from |max| of the call's input: a graph
    replay on a large-magnitude input and eager calls on a small-magnitude one must not see
    each other's |max| (every call clears the slot before its pre-pass)."""
    p = ps.ConvPreset.parse("conv:8,64,64,14,14,3,3,1,1,16,1,1,14,14")
    sx, sw = seeds(35)
    xh = oracle.fill_input(p, sx, 64)
    wh = oracle.fill_filter(p, sw, 64)
    big, small = 3.0e4, 1.0e-3
    ref_big = oracle.conv(p, (xh * big).astype(np.float32), wh).ravel()
    ref_small = oracle.conv(p, (xh * small).astype(np.float32), wh).ravel()
    xb = torch.from_numpy((xh * big).astype(np.float32).ravel()).to(DEV)
    xs = torch.from_numpy((xh * small).astype(np.float32).ravel()).to(DEV)
    w = torch.from_numpy(wh.ravel()).to(DEV)
    plan = ps.ConvPlan(p, mode="f16x2", device=0)
    plan.prepack(w)
    yb = torch.full((p.output_elems(),), float("nan"), device=DEV)
    ys = torch.full((p.output_elems(),), float("nan"), device=DEV)
    g = plan.graph(xb, None, yb)
    for _ in range(3):
        g.replay()
        plan.forward(xs, None, ys, prepacked=True)
        torch.cuda.synchronize()
        assert oracle.rel_l2(yb.cpu().numpy(), ref_big) <= 1e-5
        assert oracle.rel_l2(ys.cpu().numpy(), ref_small) <= 1e-5


# ---------------------------------------------------------------- blocked-layout packing
def _np_pack_input(nchw, p, c_log):
    n, _, h, w = nchw.shape
    cp = np.zeros((n, p.nIfm, h, w), np.float32)
    cp[:, :c_log] = nchw
    return np.ascontiguousarray(cp.reshape(n, p.nIfm // 16, 16, h, w).transpose(0, 1, 3, 4, 2))


def _np_pack_filter(kcrs, p, c_log):
    k, _, r, s = kcrs.shape
    cp = np.zeros((k, p.nIfm, r, s), np.float32)
    cp[:, :c_log] = kcrs
    # KCRS16c16k [K/16][C/16][R][S][16c][16k] (presets.hpp:93-97 filter subscripts)
    return np.ascontiguousarray(cp.reshape(k // 16, 16, p.nIfm // 16, 16, r, s).transpose(0, 2, 4, 5, 3, 1))


@pytest.mark.gpu
@pytest.mark.parametrize("conv,c_log", [
    ("conv:3,32,48,9,11,3,3,1,1,16,1,1,9,11", 48),
    ("conv:2,64,16,16,16,7,7,2,2,16,3,3,32,32", 3),   # stem-like: C = 3 zero-padded to 16
])
def test_pack_unpack_against_numpy(conv, c_log):
    p = ps.ConvPreset.parse(conv)
    rng = np.random.default_rng(7)
    nchw = rng.standard_normal((p.nImg, c_log, p.ifh, p.ifw)).astype(np.float32)
    kcrs = rng.standard_normal((p.nOfm, c_log, p.kh, p.kw)).astype(np.float32)
    xb = torch.empty(p.input_elems(), device=DEV)
    wb = torch.empty(p.filter_elems(), device=DEV)
    ps.pack_input(p, torch.from_numpy(nchw).to(DEV), xb, c_logical=c_log)
    ps.pack_filter(p, torch.from_numpy(kcrs).to(DEV), wb, c_logical=c_log)
    torch.cuda.synchronize()
    assert np.array_equal(xb.cpu().numpy(), _np_pack_input(nchw, p, c_log).ravel())
    assert np.array_equal(wb.cpu().numpy(), _np_pack_filter(kcrs, p, c_log).ravel())
    # pack -> conv (blocked) -> unpack == the plain NCHW convolution (float64 reference)
    y = torch.empty(p.output_elems(), device=DEV)
    ps.ConvPlan(p, mode="3xtf32", device=0).forward(xb, wb, y)
    yk = torch.empty(p.output_elems(), device=DEV)
    ps.unpack_output(p, y, yk)
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(torch.from_numpy(nchw).double(), torch.from_numpy(kcrs).double(),
                                     stride=(p.stride_h, p.stride_w), padding=(p.pad_h, p.pad_w))
    got = yk.cpu().double().reshape(ref.shape)
    assert float((got - ref).norm() / ref.norm()) <= 1e-5
    # unpack is exactly the inverse blocking of the output
    yb = y.cpu().numpy().reshape(p.nImg, p.nOfm // 16, p.ofh, p.ofw, 16)
    assert np.array_equal(yk.cpu().numpy(), yb.transpose(0, 1, 4, 2, 3).ravel())
