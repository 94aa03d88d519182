"""GPU parity: the sm_100a path through the C ABI vs the CPU oracle on the same seeded inputs.

Tolerances are BASELINE.json north_star's: relative L2 <= 1e-5 (3xTF32), <= 5e-3 (TF32);
max-abs is reported. Full-size BASELINE shapes are checked on image subsets (every image
is an independent unit: SURVEY.md §8e), with seeds keyed by global image index.
"""
import numpy as np
import pytest

import oracle
from tests.cases import ALL, BASELINE, R50, seeds, with_images

torch = pytest.importorskip("torch")
ps = pytest.importorskip("paper_2002_02145_b200")

TOL = {"3xtf32": 1e-5, "tf32": 5e-3, "f16x2": 1e-5}


def _run_gpu(p, c_logical, sx, sw, mode, recipe=None, img_begin=0, img_count=None,
             accumulate=False, out_init=None):
    dev = torch.device("cuda:0")
    x = torch.empty(p.input_elems(), dtype=torch.float32, device=dev)
    w = torch.empty(p.filter_elems(), dtype=torch.float32, device=dev)
    y = torch.full((p.output_elems(),), float("nan"), dtype=torch.float32, device=dev)
    if out_init is not None:
        y.copy_(torch.from_numpy(out_init.ravel()).to(dev))
    ps.fill_input(p, sx, x, c_logical=c_logical)
    ps.fill_filter(p, sw, w, c_logical=c_logical)
    plan = ps.ConvPlan(p, mode=mode, device=0, recipe=recipe)
    plan.forward(x, w, y, img_begin=img_begin, img_count=img_count, accumulate=accumulate)
    torch.cuda.synchronize()
    return x.cpu().numpy(), w.cpu().numpy(), y.cpu().numpy(), plan.recipe


def _check(name, conv, c_logical, cfg_id, mode, n_img, recipe=None):
    p = ps.ConvPreset.parse(with_images(conv, n_img))
    sx, sw = seeds(cfg_id)
    xg, wg, yg, rec = _run_gpu(p, c_logical, sx, sw, mode, recipe)
    x = oracle.fill_input(p, sx, c_logical)
    w = oracle.fill_filter(p, sw, c_logical)
    assert np.array_equal(xg, x.ravel()), "device generator != host generator (input)"
    assert np.array_equal(wg, w.ravel()), "device generator != host generator (filter)"
    ref = oracle.conv(p, x, w).ravel()
    assert np.isfinite(yg).all(), f"{name}: non-finite / unwritten outputs ({rec})"
    err = oracle.rel_l2(yg, ref)
    mx = oracle.max_abs(yg, ref)
    print(f"{name} {mode} N={n_img} recipe={rec} relL2={err:.3e} maxabs={mx:.3e}")
    assert err <= TOL[mode], f"{name} {mode}: relL2 {err:.3e} > {TOL[mode]} (maxabs {mx:.3e}, {rec})"


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
def test_default_preset(mode):
    # the reference's default preset conv:2,32,32,4,4,3,3,1,1,16 (presets.hpp:14-23)
    _check("default", "conv:2,32,32,4,4,3,3,1,1,16", 32, 0, mode, 2)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
@pytest.mark.parametrize("name", list(BASELINE))
def test_baseline_shapes(name, mode):
    conv, c_log, cid = BASELINE[name]
    n = {"cfg1": 4, "cfg2": 4, "cfg3": 4, "cfg5": 40}[name]
    _check(name, conv, c_log, cid, mode, n)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(R50))
def test_resnet50_layers(name):
    conv, c_log, cid = R50[name]
    p = ps.ConvPreset.parse(conv)
    n = max(1, min(16, 200000 // (p.ofh * p.ofw)))
    _check(name, conv, c_log, cid, "3xtf32", n)


@pytest.mark.gpu
@pytest.mark.parametrize("recipe", [
    "perm=ofm_tile,ifm_tile,oj,kj,ki",
    "perm=oj,ofm_tile,ifm_tile,kj,ki",
    "perm=kj,ki,oj,ofm_tile,ifm_tile",
    "perm=ifm_tile,ofm_tile,oj,kj,ki;tile=oj:2",
    "perm=oj,ofm_tile,ifm_tile,kj,ki;gpu=bn:32,box:56x2x1",
    "perm=ofm_tile,ifm_tile,oj,kj,ki;gpu=bn:64,box:8x8x2",
    "perm=ofm_tile,ifm_tile,oj,kj,ki;gpu=bn:16,box:7x3x5",
])
def test_recipes(recipe):
    _check("cfg1-recipe", BASELINE["cfg1"][0], 64, 1, "3xtf32", 3, recipe)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
@pytest.mark.parametrize("conv,c_log,recipe", [
    # Cb=4: channel-block groups, one packed A box per stage (64 rows per block)
    ("conv:3,64,64,20,20,3,3,1,1,16,1,1,20,20", 64, "gpu=bn:64,box:8x4x2,cl:1,kg:4"),
    ("conv:3,64,64,20,20,3,3,1,1,16,1,1,20,20", 64, "gpu=bn:64,box:8x4x2,cl:1,kg:2"),
    # box rows not a multiple of 8 -> one A box per channel block (8 KB pitch)
    ("conv:3,64,64,20,20,3,3,1,1,16,1,1,20,20", 64, "gpu=bn:32,box:7x3x2,cl:1,kg:4"),
    # Cb=3 (kg does not divide it): kps consecutive k-steps, partial last stage (27 = 6*4+3)
    ("conv:2,32,48,9,9,3,3,1,1,16,1,1,9,9", 48, "gpu=bn:32,box:9x9x1,cl:1,kg:4"),
    ("conv:2,32,48,9,9,3,3,2,2,16,1,1,18,18", 48, "gpu=bn:16,box:9x9x1,cl:1,kg:2"),
    # stem-like: Cb=1, 7x7/s2, 49 k-steps
    ("conv:2,64,16,16,16,7,7,2,2,16,3,3,32,32", 3, "gpu=bn:64,box:16x8x1,cl:1,kg:4"),
])
def test_stage_geometry(conv, c_log, recipe, mode):
    """Pipeline stages of kps k-steps: grouped channel blocks (packed or per-block A boxes)
    and consecutive-k-step stages with a partial last stage; CTA pair where the mode allows."""
    _check("stages", conv, c_log, 7, mode, ps.ConvPreset.parse(conv).nImg, recipe)
    if mode == "tf32":
        _check("stages-pair", conv, c_log, 7, mode, ps.ConvPreset.parse(conv).nImg,
               recipe.replace("cl:1", "cl:2"))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
@pytest.mark.parametrize("conv,c_log,recipe", [
    ("conv:3,64,64,20,20,3,3,1,1,16,1,1,20,20", 64, "gpu=bn:64,halo:1"),
    ("conv:3,64,64,20,20,3,3,1,1,16,1,1,20,20", 64, "gpu=bn:32,halo:1,kg:1"),
    ("conv:3,64,64,20,20,3,3,1,1,16,1,1,20,20", 64, "gpu=bn:64,halo:1,kg:2"),
    ("conv:2,64,64,56,56,3,3,1,1,16,1,1,56,56", 64, "gpu=bn:64,halo:1"),
    ("conv:4,256,256,14,14,3,3,1,1,16,1,1,14,14", 256, "gpu=bn:256,halo:1"),
    ("conv:4,256,256,14,14,3,3,1,1,16,1,1,14,14", 256, "gpu=bn:128,halo:1"),
    # ragged last row block (21 = 3*6 + 3), non-square, Cb = 3
    ("conv:2,32,48,21,19,3,3,1,1,16,1,1,21,19", 48, "gpu=bn:32,halo:1"),
    # 5x5 / pad 2, and an unpadded ("valid") 3x3
    ("conv:2,32,32,12,12,5,5,1,1,16,2,2,12,12", 32, "gpu=bn:32,halo:1"),
    ("conv:2,32,32,10,10,3,3,1,1,16,0,0,12,12", 32, "gpu=bn:32,halo:1"),
])
def test_halo_mode(conv, c_log, recipe, mode):
    """Halo mode: whole output rows at the padded pitch, the input halo loaded once per
    channel block and the R*S shifted operands addressed in place; with the filter slice
    resident in smem (auto when bn == nOfm and it fits) and with the B ring (br:0)."""
    n = ps.ConvPreset.parse(conv).nImg
    for br in ("", ",br:0"):
        _check("halo" + br, conv, c_log, 9, mode, n, recipe + br + (",cl:1" if mode == "tf32" else ""))
        if mode == "tf32":
            _check("halo-pair" + br, conv, c_log, 9, mode, n, recipe + br + ",cl:2")


@pytest.mark.gpu
@pytest.mark.parametrize("mode,recipe", [
    ("tf32", "gpu=bn:64,halo:1,br:1,cl:1"),
    ("tf32", "gpu=bn:64,halo:1,br:1,cl:2"),
    ("tf32", "gpu=bn:64,halo:1,br:1,kg:2"),
    ("3xtf32", "gpu=bn:32,halo:1,br:1"),
])
def test_halo_resident_filter(mode, recipe):
    """br:1 -- the whole filter slice resident in shared memory, only halo tiles stream."""
    conv = "conv:2,64,64,56,56,3,3,1,1,16,1,1,56,56" if "bn:64" in recipe else \
        "conv:3,32,32,20,20,3,3,1,1,16,1,1,20,20"
    _check("halo-br", conv, int(conv.split(",")[1]), 9, mode, ps.ConvPreset.parse(conv).nImg, recipe)


@pytest.mark.gpu
def test_image_range_and_accumulate():
    """conv_fwd on [img_begin, img_begin+count) touches only those images; FLAG_ACCUMULATE
    reproduces the reference body's `+=` (presets.hpp:112)."""
    p = ps.ConvPreset.parse(with_images(BASELINE["cfg3"][0], 6))
    sx, sw = seeds(3)
    base = np.random.default_rng(0).standard_normal(p.output_elems()).astype(np.float32)
    xg, wg, yg, _ = _run_gpu(p, 128, sx, sw, "3xtf32", img_begin=2, img_count=3,
                             accumulate=True, out_init=base)
    x = oracle.fill_input(p, sx, 128)
    w = oracle.fill_filter(p, sw, 128)
    ref = base.reshape(6, -1).copy()
    conv = oracle.conv(p, x, w).reshape(6, -1)
    ref[2:5] += conv[2:5]
    yg = yg.reshape(6, -1)
    assert np.array_equal(yg[:2], ref[:2]) and np.array_equal(yg[5:], ref[5:])
    assert oracle.rel_l2(yg[2:5], ref[2:5]) <= 1e-5


@pytest.mark.gpu
def test_deep_output_staging_other_entries():
    """os:8 through the other entry points: an image sub-range, the host-buffer path (chunked,
    three device slots) and CUDA-graph replay give the plain device result bit for bit."""
    p = ps.ConvPreset.parse("conv:96,128,64,28,28,1,1,1,1,16,0,0,28,28")
    sx, sw = seeds(23)
    dev = torch.device("cuda:0")
    x = torch.empty(p.input_elems(), device=dev)
    w = torch.empty(p.filter_elems(), device=dev)
    ps.fill_input(p, sx, x, c_logical=64)
    ps.fill_filter(p, sw, w, c_logical=64)
    ref_plan = ps.ConvPlan(p, mode="3xtf32", device=0, recipe="gpu=bn:128,box:4x4x8,cl:1")
    plan = ps.ConvPlan(p, mode="3xtf32", device=0, recipe="gpu=bn:128,box:4x4x8,cl:1,os:8")
    assert "os:8" in plan.recipe
    y0 = torch.zeros(p.output_elems(), device=dev)
    y1 = torch.zeros(p.output_elems(), device=dev)
    ref_plan.forward(x, w, y0, img_begin=7, img_count=80)
    plan.forward(x, w, y1, img_begin=7, img_count=80)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1), "os:8 changes the result of an image sub-range"
    hy = torch.zeros(p.output_elems()).pin_memory()
    plan.forward_host(x.cpu().pin_memory(), w.cpu().pin_memory(), hy, img_begin=7, img_count=80)
    torch.cuda.synchronize()
    assert torch.equal(hy, y0.cpu()), "os:8 host path differs from the device path"
    y2 = torch.zeros(p.output_elems(), device=dev)
    plan.prepack(w)
    g = plan.graph(x, None, y2)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    plan.forward(x, w, y0)
    torch.cuda.synchronize()
    assert torch.equal(y2, y0), "os:8 graph replay differs from the eager call"


@pytest.mark.gpu
@pytest.mark.parametrize("accumulate", [False, True])
def test_forward_host(accumulate):
    """conv_fwd_host: host buffers streamed through the device in double-buffered chunks
    (more chunks than slots), same result as the device path; `+=` reads the host output."""
    conv = "conv:200,32,32,56,56,3,3,1,1,16,1,1,56,56"  # 401 KB/image: 81-image chunks, 3 chunks
    p = ps.ConvPreset.parse(conv)
    sx, sw = seeds(11)
    dev = torch.device("cuda:0")
    x = torch.empty(p.input_elems(), device=dev)
    w = torch.empty(p.filter_elems(), device=dev)
    ps.fill_input(p, sx, x, c_logical=32)
    ps.fill_filter(p, sw, w, c_logical=32)
    y = torch.zeros(p.output_elems(), device=dev)
    base = torch.randn(p.output_elems()) if accumulate else torch.zeros(p.output_elems())
    y.copy_(base.to(dev))
    plan = ps.ConvPlan(p, mode="3xtf32", device=0)
    plan.forward(x, w, y, img_begin=5, img_count=190, accumulate=accumulate)
    hx = x.cpu().pin_memory()
    hw = w.cpu().pin_memory()
    hy = base.clone().pin_memory()
    plan.forward_host(hx, hw, hy, img_begin=5, img_count=190, accumulate=accumulate)
    torch.cuda.synchronize()
    yd = y.cpu()
    assert torch.equal(hy[: 5 * p.output_elems(1)], base[: 5 * p.output_elems(1)])
    assert torch.equal(hy, yd), "host-pipelined result differs from the device path"
    # unpinned numpy buffers work too (copies then serialise)
    hy2 = base.numpy().copy()
    plan.forward_host(hx.numpy(), hw.numpy(), hy2, img_begin=5, img_count=190, accumulate=accumulate)
    torch.cuda.synchronize()
    assert np.array_equal(hy2, yd.numpy())


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
@pytest.mark.parametrize("relu", [False, True])
@pytest.mark.parametrize("recipe", [None, "gpu=bn:64,halo:1", "gpu=bn:64,box:4x4x8,os:8"])
def test_fused_bias_relu(mode, relu, recipe):
    """fused epilogue out = max(conv + bias, 0) against the oracle conv
    with the same bias / ReLU applied on the host (3xTF32 uses several accumulation chunks)."""
    p = ps.ConvPreset.parse("conv:3,64,64,20,20,3,3,1,1,16,1,1,20,20")
    sx, sw = seeds(12)
    dev = torch.device("cuda:0")
    x = torch.empty(p.input_elems(), device=dev)
    w = torch.empty(p.filter_elems(), device=dev)
    ps.fill_input(p, sx, x, c_logical=64)
    ps.fill_filter(p, sw, w, c_logical=64)
    bias = torch.linspace(-3.0, 3.0, p.nOfm, device=dev)
    y = torch.full((p.output_elems(),), float("nan"), device=dev)
    plan = ps.ConvPlan(p, mode=mode, device=0, recipe=recipe)
    plan.forward(x, w, y, bias=bias, relu=relu)
    torch.cuda.synchronize()
    ref = oracle.conv(p, oracle.fill_input(p, sx, 64), oracle.fill_filter(p, sw, 64))
    ref = ref.reshape(p.nImg, p.nOfm // 16, p.ofh, p.ofw, 16)
    ref = ref + bias.cpu().numpy().reshape(1, p.nOfm // 16, 1, 1, 16)
    if relu:
        ref = np.maximum(ref, 0)
    err = oracle.rel_l2(y.cpu().numpy(), ref.ravel())
    assert err <= TOL[mode], f"relL2 {err:.3e} ({plan.recipe})"
    if relu:
        assert (y >= 0).all()


@pytest.mark.gpu
def test_relu_with_accumulate_rejected():
    p = ps.ConvPreset.parse("conv:1,16,16,4,4,1,1,1,1,16")
    plan = ps.ConvPlan(p, mode="tf32", device=0)
    t = torch.zeros(4096, device="cuda:0")
    with pytest.raises(ps.ConfigRejectedError):
        plan.forward(t, t, t, accumulate=True, relu=True)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32", "f16x2"])
def test_gemm_from_nest_document(mode):
    """a matmul nest document runs on the conv kernel as a 1x1 conv."""
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "nests", "gemm_96.nest")) as f:
        info = ps.parse_nest(f.read())
    g = ps.GemmPlan(info.M, info.N, info.K, mode=mode)
    rng = np.random.default_rng(5)
    a = rng.uniform(-1, 1, (info.M, info.K)).astype(np.float32)
    b = rng.uniform(-1, 1, (info.K, info.N)).astype(np.float32)
    c = torch.full((info.M, info.N), float("nan"), device="cuda:0")
    g.forward(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), c)
    torch.cuda.synchronize()
    ref = a.astype(np.float64) @ b.astype(np.float64)
    err = oracle.rel_l2(c.cpu().numpy(), ref)
    assert err <= TOL[mode], f"GEMM relL2 {err:.3e} ({g.recipe})"


@pytest.mark.gpu
def test_conv_from_nest_document():
    """A permuted, renamed conv document -> descriptor + recipe -> GPU parity."""
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "nests", "conv_cfg3_perm.nest")) as f:
        info = ps.parse_nest(f.read())
    conv = "conv:" + ",".join(str(info.preset).split(":")[1].split(","))
    _check("nest-conv", conv, 128, 13, "3xtf32", info.preset.nImg, info.recipe)


@pytest.mark.gpu
@pytest.mark.parametrize("recipe", ["gpu=bn:64,box:2x2x32,cl:1,gm:5", "gpu=bn:64,box:2x2x32,cl:2,gm:3",
                                    "gpu=bn:128,box:2x2x32,cl:1,gm:1"])
def test_grouped_raster(recipe):
    """Grouped (M-block x N-tile) rasterisation covers every tile exactly once, including
    the partial last block."""
    mode = "tf32" if "cl:2" in recipe else "3xtf32"
    _check("gm", BASELINE["cfg5"][0], 256, 5, mode, 23, recipe)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
@pytest.mark.parametrize("conv,c_log,recipe", [
    # the ResNet-50 stem (7x7/s2/p3, C = 3 of 16): 5 taps per folded block, 2 tap groups
    ("conv:2,64,16,112,112,7,7,2,2,16,3,3,224,224", 3, "gpu=bn:64,fold:3"),
    ("conv:2,64,16,20,20,7,7,2,2,16,3,3,40,40", 3, "gpu=bn:32,box:20x6x1,fold:3"),
    # 3x3 stride 1 with C = 5 (G = 3: one tap group), and C = 8 (G = 2) 5x5 unpadded
    ("conv:3,32,16,17,19,3,3,1,1,16,1,1,17,19", 5, "gpu=bn:32,fold:5"),
    ("conv:2,32,16,12,12,5,5,1,1,16,0,0,16,16", 8, "gpu=bn:32,fold:8"),
])
def test_cs_fold(conv, c_log, recipe, mode):
    """(c,s)-folded input (SURVEY §8d stem note): G = 16 / C kw taps share one 16-channel
    block; same result as the unfolded conv on inputs whose channels >= C are zero."""
    n = ps.ConvPreset.parse(conv).nImg
    _check("fold", conv, c_log, 14, mode, n, recipe)
    if mode == "tf32":
        _check("fold-pair", conv, c_log, 14, mode, n, recipe + ",cl:2")


@pytest.mark.gpu
@pytest.mark.parametrize("conv,c_log,recipe", [
    ("conv:3,64,64,20,20,3,3,1,1,16,1,1,20,20", 64, "gpu=bn:64,box:8x4x2,kg:1,ta:1"),
    ("conv:3,64,64,20,20,3,3,1,1,16,1,1,20,20", 64, "gpu=bn:64,box:7x3x2,kg:4,ta:1"),
    ("conv:2,128,128,14,14,3,3,1,1,16,1,1,14,14", 128, "gpu=bn:128,box:2x4x16,ta:1"),
    ("conv:2,128,128,14,14,3,3,1,1,16,1,1,14,14", 128, "gpu=bn:128,box:2x4x16,ta:0"),
    ("conv:2,32,48,9,9,3,3,1,1,16,1,1,9,9", 48, "gpu=bn:16,box:9x9x1,kg:4,ta:1"),
    ("conv:300,64,32,8,16,1,1,1,1,16,0,0,8,16", 32, "gpu=bn:64,box:16x8x1,ta:1,ch:1"),
])
def test_tmem_resident_a(conv, c_log, recipe):
    """3xTF32 with A_hi / A_lo in TMEM (splitter tcgen05.st, MMAs read A from TMEM): slot
    ring wrap-around, partial stages, unaligned boxes, many tiles, chunked sums."""
    n = ps.ConvPreset.parse(conv).nImg
    _check("tmem-a", conv, c_log, 15, "3xtf32", n, recipe)


def _bwd_data_ref(p, dy, w):
    """dX[n][c][h][w] = sum over (p, q, r, s) with h = p*sh + r - pad_h, w = q*sw + s - pad_w of
    dY[n][k][p][q] W[k][c][r][s] (float64, NCHW16c) -- the adjoint of the forward conv."""
    N, K, C = p.nImg, p.nOfm, p.nIfm
    P, Q, R, S, H, W_ = p.ofh, p.ofw, p.kh, p.kw, p.ifh, p.ifw
    sh, sw = p.stride_h, p.stride_w
    dyl = dy.reshape(N, K // 16, P, Q, 16).transpose(0, 1, 4, 2, 3).reshape(N, K, P, Q).astype(np.float64)
    wl = w.reshape(K // 16, C // 16, R, S, 16, 16).transpose(0, 5, 1, 4, 2, 3).reshape(K, C, R, S)
    dx = np.zeros((N, C, H, W_))
    for r in range(R):
        for s in range(S):
            ps_ = [pp for pp in range(P) if 0 <= pp * sh + r - p.pad_h < H]
            qs = [q for q in range(Q) if 0 <= q * sw + s - p.pad_w < W_]
            if not ps_ or not qs:
                continue
            hs = [pp * sh + r - p.pad_h for pp in ps_]
            ws = [q * sw + s - p.pad_w for q in qs]
            dx[:, :, np.ix_(hs, ws)[0], np.ix_(hs, ws)[1]] += np.einsum(
                "nkpq,kc->ncpq", dyl[:, :, ps_][:, :, :, qs], wl[:, :, r, s])
    return dx.reshape(N, C // 16, 16, H, W_).transpose(0, 1, 3, 4, 2).ravel()


BWD_DATA = ["conv:2,64,32,12,12,3,3,1,1,16,1,1,12,12",
            "conv:2,32,48,9,11,5,5,1,1,16,2,2,9,11",
            "conv:3,128,64,7,7,1,1,1,1,16",
            # strided: one stride-1 transposed conv per output phase (sh x sw of them)
            "conv:2,64,32,14,14,3,3,2,2,16,1,1,28,28",   # 3x3/s2 (ResNet-50 l2..l4 first 3x3)
            "conv:2,32,48,7,7,3,3,2,2,16,1,1,13,13",     # odd extent: phases of 7 and 6 rows
            "conv:2,64,32,7,7,1,1,2,2,16,0,0,14,14",     # 1x1/s2 downsample: 3 phases zero
            "conv:2,64,16,8,8,7,7,2,2,16,3,3,16,16",     # 7x7/s2 (stem-shaped)
            "conv:2,32,32,5,9,3,1,2,1,16,1,0,10,9"]      # stride only in h


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32", "f16x2"])
@pytest.mark.parametrize("conv", BWD_DATA)
def test_backward_data(conv, mode):
    """§8f row f4: dX as the transposed conv on the same kernel (strided layers: per phase)."""
    p = ps.ConvPreset.parse(conv)
    rng = np.random.default_rng(3)
    dy = rng.uniform(-1, 1, p.output_elems()).astype(np.float32)
    w = rng.uniform(-1, 1, p.filter_elems()).astype(np.float32)
    plan = ps.ConvPlan(p, mode=mode, device=0, bwd_data=True)
    dx = torch.full((p.input_elems(),), float("nan"), device="cuda:0")
    plan.forward(torch.from_numpy(dy).cuda(), torch.from_numpy(w).cuda(), dx)
    torch.cuda.synchronize()
    ref = _bwd_data_ref(p, dy, w)
    err = oracle.rel_l2(dx.cpu().numpy(), ref)
    assert err <= TOL[mode], f"bwd-data relL2 {err:.3e} ({plan.recipe})"


@pytest.mark.gpu
def test_backward_data_strided_paths():
    """Strided backward data through the other entry points: accumulate (+=, zero phases left
    alone), a prepacked filter, an image range, and the host-buffer path."""
    p = ps.ConvPreset.parse("conv:4,64,32,7,7,1,1,2,2,16,0,0,14,14")
    rng = np.random.default_rng(5)
    dy = rng.uniform(-1, 1, p.output_elems()).astype(np.float32)
    w = rng.uniform(-1, 1, p.filter_elems()).astype(np.float32)
    base = rng.uniform(-1, 1, p.input_elems()).astype(np.float32)
    ref = _bwd_data_ref(p, dy, w)
    plan = ps.ConvPlan(p, mode="3xtf32", device=0, bwd_data=True)
    assert plan.recipe.count("phase") == 4 and plan.launches == 3 + 3
    dyd, wd = torch.from_numpy(dy).cuda(), torch.from_numpy(w).cuda()
    dx = torch.from_numpy(base.copy()).cuda()
    plan.forward(dyd, wd, dx, accumulate=True)
    torch.cuda.synchronize()
    assert oracle.rel_l2(dx.cpu().numpy(), ref + base) <= 1e-5
    plan.prepack(wd)
    per = p.input_elems() // p.nImg
    dx = torch.full((p.input_elems(),), float("nan"), device="cuda:0")
    plan.forward(dyd, None, dx, img_begin=1, img_count=2, prepacked=True)
    torch.cuda.synchronize()
    got = dx.cpu().numpy()[per:3 * per]
    assert oracle.rel_l2(got, ref[per:3 * per]) <= 1e-5
    hx = np.full(p.input_elems(), np.nan, dtype=np.float32)
    plan.forward_host(dy, w, hx)
    torch.cuda.synchronize()
    assert oracle.rel_l2(hx, ref) <= 1e-5
    with pytest.raises(ps.ConfigRejectedError):
        plan.emit()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
def test_backward_data_cached_recipe(mode):
    """A stride-1 ResNet layer's backward data reuses the plan cache's recipe of its transposed
    (forward) shape; checked on an image range of the full N = 256 plan."""
    conv = R50["r50_l3_3x3_256_256"][0]
    p = ps.ConvPreset.parse(conv)
    plan = ps.ConvPlan(p, mode=mode, device=0, bwd_data=True)
    def items(r):
        perm, gpu = r.split(";gpu=")
        return perm, set(gpu.split(","))
    assert items(plan.recipe) == items(ps._cached_bwd_data_recipe(p, ps._MODES[mode]))
    rng = np.random.default_rng(7)
    sub = ps.ConvPreset.parse(conv.replace("conv:256,", "conv:2,", 1))
    dy = rng.uniform(-1, 1, sub.output_elems()).astype(np.float32)
    w = rng.uniform(-1, 1, sub.filter_elems()).astype(np.float32)
    dyd = torch.zeros(p.output_elems(), device="cuda:0")
    dyd[:dy.size] = torch.from_numpy(dy).cuda()
    dx = torch.full((p.input_elems(),), float("nan"), device="cuda:0")
    plan.forward(dyd, torch.from_numpy(w).cuda(), dx, img_begin=0, img_count=2)
    torch.cuda.synchronize()
    err = oracle.rel_l2(dx[:sub.input_elems()].cpu().numpy(), _bwd_data_ref(sub, dy, w))
    assert err <= TOL[mode], f"relL2 {err:.3e} ({plan.recipe})"


@pytest.mark.gpu
def test_backward_data_rejects_negative_phase_pad():
    # 2x2 / stride 2 / pad 1: phase 1's taps start one row past its first output row
    with pytest.raises(ps.ConfigRejectedError):
        ps.ConvPlan(ps.ConvPreset.parse("conv:1,16,16,4,4,2,2,2,2,16,1,1,6,6"), bwd_data=True)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
@pytest.mark.parametrize("conv,c_log,recipe", [
    ("conv:6,512,512,7,7,3,3,1,1,16,1,1,7,7", 512, "gpu=bn:256,box:7x1x18,ks:2"),
    ("conv:6,512,512,7,7,3,3,1,1,16,1,1,7,7", 512, "gpu=bn:128,box:1x7x18,ks:5"),
    ("conv:3,64,64,20,20,3,3,1,1,16,1,1,20,20", 64, "gpu=bn:64,box:8x4x2,kg:4,ks:3"),
    ("conv:2,32,48,9,9,3,3,1,1,16,1,1,9,9", 48, "gpu=bn:32,box:9x9x1,kg:4,ks:2"),
])
def test_split_k(conv, c_log, recipe, mode):
    """Split-K work units: each tile's reduction in ks stage ranges, the partials combined
    in split order by the tile's last unit (also with the pair, TMEM-A and partial-stage
    paths)."""
    n = ps.ConvPreset.parse(conv).nImg
    _check("ks", conv, c_log, 16, mode, n, recipe)
    if mode == "tf32":
        _check("ks-pair", conv, c_log, 16, mode, n, recipe + ",cl:2")


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
@pytest.mark.parametrize("conv,c_log,recipe", [
    # output-heavy 1x1 shapes: many tiles per CTA so the staging ring wraps many times
    ("conv:40,256,64,28,28,1,1,1,1,16,0,0,28,28", 64, "gpu=bn:256,box:4x4x8,cl:1,os:8"),
    ("conv:40,256,64,28,28,1,1,1,1,16,0,0,28,28", 64, "gpu=bn:256,box:4x4x8,cl:1,eg:2,os:8"),
    ("conv:40,256,64,28,28,1,1,1,1,16,0,0,28,28", 64, "gpu=bn:128,box:2x4x16,cl:1,os:8"),
    ("conv:40,128,64,28,28,1,1,1,1,16,0,0,28,28", 64, "gpu=bn:64,box:4x4x8,cl:1,os:8"),
    ("conv:40,128,64,28,28,1,1,1,1,16,0,0,28,28", 64, "gpu=bn:16,box:4x4x8,cl:1,os:8"),
    ("conv:40,128,64,28,28,1,1,1,1,16,0,0,28,28", 64, "gpu=bn:16,box:4x4x8,cl:1,os:16"),
    ("conv:40,256,64,28,28,1,1,1,1,16,0,0,28,28", 64, "gpu=bn:256,box:4x4x8,cl:1,os:12"),
    ("conv:40,256,64,28,28,1,1,1,1,16,0,0,28,28", 64, "gpu=bn:256,box:4x4x8,cl:1,eg:2,os:16"),
    ("conv:12,128,128,14,14,3,3,1,1,16,1,1,14,14", 128, "gpu=bn:128,box:2x2x32,cl:1,ks:3,os:8"),
])
def test_deep_output_staging(conv, c_log, recipe, mode):
    """os:8 / 12 / 16 staging blocks; the store warp hands a slot back only once half the
    slots' TMA stores are still reading shared memory (deferred, in order)."""
    n = ps.ConvPreset.parse(conv).nImg
    _check("os8", conv, c_log, 21, mode, n, recipe)
    if mode == "tf32" and "bn:16" not in recipe:
        _check("os8-pair", conv, c_log, 21, mode, n, recipe.replace("cl:1", "cl:2"))


@pytest.mark.gpu
def test_deep_output_staging_accumulate():
    """os:8 with `+=` (TMA reduce-add stores) on a pre-filled output."""
    conv = "conv:24,256,64,14,14,1,1,1,1,16,0,0,14,14"
    p = ps.ConvPreset.parse(conv)
    sx, sw = seeds(22)
    init = np.random.default_rng(5).uniform(-1, 1, p.output_elems()).astype(np.float32)
    _, _, yg, rec = _run_gpu(p, 64, sx, sw, "3xtf32", "gpu=bn:256,box:2x2x32,cl:1,os:8",
                             accumulate=True, out_init=init)
    ref = oracle.conv(p, oracle.fill_input(p, sx, 64), oracle.fill_filter(p, sw, 64)).ravel() + init
    assert oracle.rel_l2(yg, ref) <= 1e-5, rec


TAIL = "conv:8,64,64,56,56,3,3,1,1,16,1,1,56,56"  # 196 tiles of 8x8x2 px: 1 wave + 48


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
@pytest.mark.parametrize("recipe", [
    "gpu=bn:64,box:8x8x2,ks:3",   # 144 tail units after 148 whole tiles
    "gpu=bn:64,box:8x8x2,ks:4",   # 192 tail units: a second round of units
    "gpu=bn:64,box:8x8x2,ks:2,cl:2",  # pairs: 74 clusters, 98 groups
    "gpu=bn:64,box:8x8x2,ks:3,kt:1",  # every tile split: zeroed output, all partials added
])
def test_tail_split(recipe, mode):
    """Tail split-K: only the last partial wave's tiles are split; every unit writes its
    partial to the plan workspace and the last one adds them and stores (no output memset)."""
    if "cl:2" in recipe and mode == "3xtf32":
        pytest.skip("the CTA pair is TF32-only")
    _check("tail", TAIL, 64, 16, mode, 8, recipe)


@pytest.mark.gpu
def test_tail_split_relaunch():
    """The split tiles' ticket counters return to zero at the end of every launch: repeated
    launches of one plan on one stream stay correct (each overwrites a NaN-filled output)."""
    p = ps.ConvPreset.parse(TAIL)
    sx, sw = seeds(16)
    dev = torch.device("cuda:0")
    x = torch.empty(p.input_elems(), dtype=torch.float32, device=dev)
    w = torch.empty(p.filter_elems(), dtype=torch.float32, device=dev)
    ps.fill_input(p, sx, x, c_logical=64)
    ps.fill_filter(p, sw, w, c_logical=64)
    ref = oracle.conv(p, oracle.fill_input(p, sx, 64), oracle.fill_filter(p, sw, 64)).ravel()
    plan = ps.ConvPlan(p, mode="tf32", device=0, recipe="gpu=bn:64,box:8x8x2,ks:3")
    ys = [torch.full((p.output_elems(),), float("nan"), dtype=torch.float32, device=dev) for _ in range(11)]
    for y in ys:
        plan.forward(x, w, y)
    torch.cuda.synchronize()
    for i, y in enumerate(ys):
        err = oracle.rel_l2(y.cpu().numpy(), ref)
        assert err <= TOL["tf32"], f"launch {i}: relL2 {err:.3e}"


@pytest.mark.gpu
def test_tail_split_accumulate():
    p = ps.ConvPreset.parse(TAIL)
    sx, sw = seeds(16)
    base = np.random.default_rng(2).standard_normal(p.output_elems()).astype(np.float32)
    xg, wg, yg, rec = _run_gpu(p, 64, sx, sw, "3xtf32", recipe="gpu=bn:64,box:8x8x2,ks:3",
                               accumulate=True, out_init=base)
    ref = base + oracle.conv(p, oracle.fill_input(p, sx, 64), oracle.fill_filter(p, sw, 64)).ravel()
    assert oracle.rel_l2(yg, ref) <= 1e-5, rec


@pytest.mark.gpu
def test_split_k_accumulate():
    """+= with split-K: no zeroing, every unit adds into the existing output."""
    p = ps.ConvPreset.parse("conv:4,256,256,7,7,3,3,1,1,16,1,1,7,7")
    sx, sw = seeds(17)
    base = np.random.default_rng(1).standard_normal(p.output_elems()).astype(np.float32)
    xg, wg, yg, rec = _run_gpu(p, 256, sx, sw, "3xtf32", recipe="gpu=bn:128,box:7x1x18,ks:3",
                               accumulate=True, out_init=base)
    ref = base + oracle.conv(p, oracle.fill_input(p, sx, 256), oracle.fill_filter(p, sw, 256)).ravel()
    assert oracle.rel_l2(yg, ref) <= 1e-5, rec


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
@pytest.mark.parametrize("conv,c_log,recipe", [
    ("conv:3,64,64,20,20,3,3,1,1,16,1,1,20,20", 64, "gpu=bn:64,box:8x4x2,eg:2"),
    ("conv:2,256,128,14,14,3,3,1,1,16,1,1,14,14", 128, "gpu=bn:256,box:2x4x16,eg:2,ch:8"),
    ("conv:6,512,512,7,7,3,3,1,1,16,1,1,7,7", 512, "gpu=bn:256,box:7x1x18,ks:2,eg:2"),
    ("conv:6,512,512,7,7,3,3,1,1,16,1,1,7,7", 512, "gpu=bn:128,box:1x7x18,ks:3,kt:1,eg:2"),
    ("conv:300,128,32,8,16,1,1,1,1,16,0,0,8,16", 32, "gpu=bn:128,box:16x8x1,eg:2"),
    ("conv:3,64,64,20,20,3,3,1,1,16,1,1,20,20", 64, "gpu=bn:64,halo:1,eg:2"),
])
def test_two_epilogue_groups(conv, c_log, recipe, mode):
    """Recipe eg:2: two epilogue warp groups drain alternate 32-channel rounds (own staging
    blocks, bulk groups, named barriers); split-K flag release waits for both groups."""
    if mode == "tf32":
        recipe = recipe.replace(",ch:8", "")
        if "bn:128" in recipe and "ks" not in recipe:
            recipe += ",cl:2"
    n = ps.ConvPreset.parse(conv).nImg
    _check("eg2", conv, c_log, 16, mode, n, recipe)


@pytest.mark.gpu
def test_two_epilogue_groups_accumulate():
    p = ps.ConvPreset.parse("conv:4,128,64,12,12,3,3,1,1,16,1,1,12,12")
    sx, sw = seeds(17)
    init = np.random.default_rng(5).uniform(-1, 1, p.output_elems()).astype(np.float32)
    x = oracle.fill_input(p, sx, 64)
    w = oracle.fill_filter(p, sw, 64)
    ref = oracle.conv(p, x, w).ravel() + init
    _, _, yg, rec = _run_gpu(p, 64, sx, sw, "3xtf32", recipe="gpu=bn:128,eg:2", accumulate=True,
                             out_init=init)
    assert "eg:2" in rec
    assert oracle.rel_l2(yg, ref) <= TOL["3xtf32"]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
@pytest.mark.parametrize("conv,c_log,recipe", [
    # the ResNet-50 stem (7x7/s2/p3, C = 3 of 16): 4 parity planes, 25 tap-pair MMAs
    ("conv:2,64,16,112,112,7,7,2,2,16,3,3,224,224", 3, "gpu=pp:3"),
    # ragged tiles (P, Q not multiples of 16 / 8), 5x5/s2, bn 128 and two N tiles of 64
    ("conv:3,128,16,13,11,5,5,2,2,16,2,2,25,21", 2, "gpu=bn:128,pp:2"),
    ("conv:3,128,16,13,11,5,5,2,2,16,2,2,25,21", 2, "gpu=bn:64,pp:2"),
    # stride 1 (one plane), even tap count (3x4... 4x3), C = 4
    ("conv:2,64,16,20,19,4,3,1,1,16,1,1,21,19", 4, "gpu=pp:4"),
    ("conv:2,64,16,18,18,3,3,1,1,16,1,1,18,18", 1, "gpu=pp:1"),
])
def test_parity_plane_tap_pairs(conv, c_log, recipe, mode):
    """Few-channel kernel (recipe pp:C, conv_pp.cuh): tap pairs per K=8 MMA read straight
    from TMA-loaded input parity planes; same result as the plain conv on inputs whose
    channels >= C are zero."""
    n = ps.ConvPreset.parse(conv).nImg
    _check("pp", conv, c_log, 18, mode, n, recipe)


@pytest.mark.gpu
def test_parity_plane_f16x2_plan():
    """An f16x2 plan with pp:C runs the few-channel kernel in its 3xTF32 arithmetic."""
    _check("pp-f16x2", "conv:2,64,16,112,112,7,7,2,2,16,3,3,224,224", 3, 18, "f16x2", 2, "gpu=pp:3")


@pytest.mark.gpu
def test_parity_plane_accumulate_and_range():
    p = ps.ConvPreset.parse("conv:5,64,16,30,30,7,7,2,2,16,3,3,60,60")
    sx, sw = seeds(19)
    init = np.random.default_rng(7).uniform(-1, 1, p.output_elems()).astype(np.float32)
    x = oracle.fill_input(p, sx, 3)
    w = oracle.fill_filter(p, sw, 3)
    full = oracle.conv(p, x, w).ravel()
    per = full.size // p.nImg
    ref = init.copy()
    ref[per:4 * per] += full[per:4 * per]
    _, _, yg, rec = _run_gpu(p, 3, sx, sw, "3xtf32", recipe="gpu=pp:3", img_begin=1, img_count=3,
                             accumulate=True, out_init=init)
    assert "pp:3" in rec
    assert oracle.rel_l2(yg, ref) <= TOL["3xtf32"]


@pytest.mark.gpu
@pytest.mark.parametrize("mode,recipe", [
    ("tf32", "gpu=bn:64,box:8x8x2"),
    ("3xtf32", "gpu=bn:64,box:8x8x2,ks:3"),          # tail split-K: counters back at zero per replay
    ("tf32", "gpu=bn:64,box:8x8x2,ks:2,cl:2"),
])
def test_cuda_graph_replay(mode, recipe):
    """ConvPlan.graph(): the captured launch (PDL edge) replays to the same result as forward(),
    bit for bit, several times in a row (split-K combines partials in a fixed order)."""
    p = ps.ConvPreset.parse("conv:40,64,64,16,16,3,3,1,1,16,1,1,16,16")
    sx, sw = seeds(21)
    dev = torch.device("cuda:0")
    x = torch.empty(p.input_elems(), device=dev)
    w = torch.empty(p.filter_elems(), device=dev)
    ps.fill_input(p, sx, x, c_logical=64)
    ps.fill_filter(p, sw, w, c_logical=64)
    plan = ps.ConvPlan(p, mode=mode, device=0, recipe=recipe)
    plan.prepack(w)
    y0 = torch.empty(p.output_elems(), device=dev)
    plan.forward(x, None, y0, prepacked=True)
    y = torch.full((p.output_elems(),), float("nan"), device=dev)
    g = plan.graph(x, None, y)
    for _ in range(3):
        y.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert torch.isfinite(y).all()
        assert torch.equal(y, y0), "graph replay differs from forward()"


@pytest.mark.gpu
def test_parity_plane_forward_host():
    """The few-channel kernel behind the host-buffer entry (conv_fwd_host): chunked images,
    same result as its device path and within tolerance of the oracle."""
    p = ps.ConvPreset.parse("conv:24,64,16,28,28,7,7,2,2,16,3,3,56,56")
    sx, sw = seeds(22)
    x = oracle.fill_input(p, sx, 3)
    w = oracle.fill_filter(p, sw, 3)
    ref = oracle.conv(p, x, w).ravel()
    dev = torch.device("cuda:0")
    plan = ps.ConvPlan(p, mode="tf32", device=0, recipe="gpu=pp:3")
    yd = torch.empty(p.output_elems(), device=dev)
    plan.forward(torch.from_numpy(x.ravel()).to(dev), torch.from_numpy(w.ravel()).to(dev), yd)
    hy = np.full(p.output_elems(), np.nan, dtype=np.float32)
    plan.forward_host(x.ravel(), w.ravel(), hy)
    torch.cuda.synchronize()
    assert np.array_equal(hy, yd.cpu().numpy())
    assert oracle.rel_l2(hy, ref) <= TOL["tf32"]


@pytest.mark.gpu
@pytest.mark.parametrize("conv,c_log,recipe", [
    ("conv:2,64,64,14,14,3,3,1,1,16,1,1,14,14", 64, None),
    ("conv:2,256,256,14,14,3,3,1,1,16,1,1,14,14", 256, "gpu=bn:256,box:1x1x128"),
    ("conv:2,256,256,14,14,3,3,1,1,16,1,1,14,14", 256, "gpu=bn:128,box:2x2x32,kg:2"),   # b128 rows
    ("conv:6,512,512,7,7,3,3,1,1,16,1,1,7,7", 512, "gpu=bn:256,box:7x1x18,ks:2,eg:2"),
    ("conv:6,512,512,7,7,3,3,1,1,16,1,1,7,7", 512, "gpu=bn:128,box:1x7x18,ks:3,kt:1"),
    ("conv:3,128,128,28,28,3,3,2,2,16,1,1,56,56", 128, "gpu=bn:128,box:4x4x8,kg:1,ch:5"),
    ("conv:28,64,256,56,56,1,1,1,1,16,0,0,56,56", 256, "gpu=bn:64,box:8x8x2"),
    ("conv:300,64,32,8,16,1,1,1,1,16,0,0,8,16", 32, "gpu=bn:16,box:16x8x1"),
    ("conv:2,64,16,16,16,7,7,2,2,16,3,3,32,32", 3, "gpu=bn:64,fold:3"),
    # TMEM-resident fp16 A (default at bn <= 64; ta:1 at bn 128) and the smem path (ta:0)
    ("conv:3,64,64,20,20,3,3,1,1,16,1,1,20,20", 64, "gpu=bn:64,box:8x4x2,kg:4,ta:1"),
    ("conv:3,64,64,20,20,3,3,1,1,16,1,1,20,20", 64, "gpu=bn:64,box:8x4x2,ta:0"),
    ("conv:2,128,128,14,14,3,3,1,1,16,1,1,14,14", 128, "gpu=bn:128,box:2x4x16,ta:1"),
    ("conv:300,64,32,8,16,1,1,1,1,16,0,0,8,16", 32, "gpu=bn:64,box:16x8x1,ta:1,ch:1"),
])
def test_f16x2_mode(conv, c_log, recipe):
    """f16x2 (fp32-faithful): power-of-two scaled fp16 hi/lo split of both operands, three
    K=16 kind::f16 MMAs per 16-channel k-step; relative L2 <= 1e-5 like 3xTF32."""
    n = ps.ConvPreset.parse(conv).nImg
    _check("f16x2", conv, c_log, 23, "f16x2", n, recipe)


@pytest.mark.gpu
@pytest.mark.parametrize("xs,ws", [(1e-3, 1.0), (1.0, 1e4), (3e4, 2e-5), (1e-6, 1e-6)])
def test_f16x2_dynamic_range(xs, ws):
    """The operand scales follow the data: inputs / filters far from unit magnitude keep the
    1e-5 bound (hi/lo stay in fp16's normal range after scaling)."""
    p = ps.ConvPreset.parse("conv:3,128,64,12,12,3,3,1,1,16,1,1,12,12")
    sx, sw = seeds(24)
    x = (oracle.fill_input(p, sx, 64) * np.float32(xs)).astype(np.float32)
    w = (oracle.fill_filter(p, sw, 64) * np.float32(ws)).astype(np.float32)
    ref = oracle.conv(p, x, w).ravel()
    dev = torch.device("cuda:0")
    y = torch.full((p.output_elems(),), float("nan"), device=dev)
    plan = ps.ConvPlan(p, mode="f16x2", device=0)
    plan.forward(torch.from_numpy(x.ravel()).to(dev), torch.from_numpy(w.ravel()).to(dev), y)
    torch.cuda.synchronize()
    err = oracle.rel_l2(y.cpu().numpy(), ref)
    assert err <= TOL["f16x2"], f"relL2 {err:.3e} at scales {xs}, {ws}"


@pytest.mark.gpu
def test_f16x2_accumulate_bias_relu():
    p = ps.ConvPreset.parse("conv:4,128,64,12,12,3,3,1,1,16,1,1,12,12")
    sx, sw = seeds(25)
    x = oracle.fill_input(p, sx, 64)
    w = oracle.fill_filter(p, sw, 64)
    conv = oracle.conv(p, x, w).ravel()
    dev = torch.device("cuda:0")
    xd, wd = torch.from_numpy(x.ravel()).to(dev), torch.from_numpy(w.ravel()).to(dev)
    init = np.random.default_rng(8).uniform(-1, 1, p.output_elems()).astype(np.float32)
    y = torch.from_numpy(init.copy()).to(dev)
    plan = ps.ConvPlan(p, mode="f16x2", device=0)
    plan.forward(xd, wd, y, accumulate=True)
    torch.cuda.synchronize()
    assert oracle.rel_l2(y.cpu().numpy(), conv + init) <= TOL["f16x2"]
    bias = np.random.default_rng(9).uniform(-1, 1, p.nOfm).astype(np.float32)
    y2 = torch.empty(p.output_elems(), device=dev)
    plan.forward(xd, wd, y2, bias=torch.from_numpy(bias).to(dev), relu=True)
    torch.cuda.synchronize()
    ref = conv.reshape(p.nImg, p.nOfm // 16, p.ofh, p.ofw, 16) + bias.reshape(1, p.nOfm // 16, 1, 1, 16)
    ref = np.maximum(ref, 0).ravel()
    assert oracle.rel_l2(y2.cpu().numpy(), ref) <= TOL["f16x2"]


def _wgrad_ref(p, x, dy):
    """dW[k][c][r][s] = sum_{n,p,q} X[n][c][p*sh+r-pad][q*sw+s-pad] dY[n][k][p][q] in float64,
    returned in KCRS16c16k."""
    N, K, C = p.nImg, p.nOfm, p.nIfm
    P, Q, R, S, H, W_ = p.ofh, p.ofw, p.kh, p.kw, p.ifh, p.ifw
    sh, sw = p.stride_h, p.stride_w
    xl = x.reshape(N, C // 16, H, W_, 16).transpose(0, 1, 4, 2, 3).reshape(N, C, H, W_).astype(np.float64)
    dyl = dy.reshape(N, K // 16, P, Q, 16).transpose(0, 1, 4, 2, 3).reshape(N, K, P, Q).astype(np.float64)
    hp = max(H + 2 * p.pad_h, (P - 1) * sh + R)
    wp = max(W_ + 2 * p.pad_w, (Q - 1) * sw + S)
    xp = np.zeros((N, C, hp, wp))
    xp[:, :, p.pad_h:p.pad_h + H, p.pad_w:p.pad_w + W_] = xl
    dw = np.zeros((K, C, R, S))
    for r in range(R):
        for s in range(S):
            win = xp[:, :, r:r + (P - 1) * sh + 1:sh, s:s + (Q - 1) * sw + 1:sw]
            dw[:, :, r, s] = np.einsum("nkpq,ncpq->kc", dyl, win)
    return dw.reshape(K // 16, 16, C // 16, 16, R, S).transpose(0, 2, 4, 5, 3, 1).ravel()


WGRAD = [
    ("conv:16,48,32,10,10,3,3,1,1,16,1,1,10,10", None),            # K = 48: odd blocks, zero fill
    ("conv:32,64,16,12,12,1,1,1,1,16,0,0,12,12", None),            # C = 16: one block
    ("conv:16,16,16,9,9,5,5,1,1,16,2,2,9,9", None),                # K = C = 16
    ("conv:64,64,64,14,14,3,3,1,1,16,1,1,14,14", None),            # ResNet-style 3x3, K = 64
    ("conv:5,128,96,13,11,3,3,1,1,16,1,1,13,11", None),            # ragged N, C = 96, 13x11
    ("conv:4,256,128,7,7,3,3,2,2,16,1,1,14,14", None),             # 3x3 / stride 2
    ("conv:6,128,64,14,14,1,1,2,2,16,0,0,28,28", None),            # 1x1 / stride 2 (downsample)
    ("conv:2,64,16,16,16,7,7,2,2,16,3,3,32,32", None),             # 7x7 / stride 2 (stem-shaped)
    ("conv:8,128,64,10,10,3,3,1,1,16,1,1,10,10", "gpu=sw:0,kn:128,cn:64,nt:2,box:10x4,sp:5"),
    ("conv:8,64,64,10,10,3,3,1,1,16,1,1,10,10", "gpu=sw:1,kn:64,cn:64,nt:2,box:8x1,sp:3,st:3,ch:8"),
    ("conv:8,256,128,8,8,3,3,1,1,16,1,1,8,8", "gpu=sw:0,kn:128,cn:128,nt:1,box:8x2"),
    # CTA pairs (cta_group::2): two 128-channel output tiles, each CTA half of the input channels
    ("conv:6,512,256,7,7,3,3,1,1,16,1,1,7,7", "gpu=cl:2,sp:3"),
    ("conv:5,256,96,9,9,1,1,1,1,16,0,0,9,9", "gpu=cl:2,sw:0,kn:128,cn:64,tma:1"),   # C = 96: partial last pair
    ("conv:4,256,128,7,7,3,3,2,2,16,1,1,14,14", "gpu=cl:1,tma:1"),
]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
@pytest.mark.parametrize("conv,recipe", WGRAD)
def test_backward_weight(conv, recipe, mode):
    """dW = conv_bwd_weight(X, dY): the pixel-major wgrad kernel (MN-major tf32 operands,
    pixel-range splits added in split order), against float64."""
    p = ps.ConvPreset.parse(conv)
    rng = np.random.default_rng(26)
    x = rng.uniform(-1, 1, p.input_elems()).astype(np.float32)
    dy = rng.uniform(-1, 1, p.output_elems()).astype(np.float32)
    ref = _wgrad_ref(p, x, dy)
    dev = torch.device("cuda:0")
    dw = torch.full((p.filter_elems(),), float("nan"), device=dev)
    if recipe and mode == "tf32" and ",ch:" in recipe:
        recipe = recipe[:recipe.index(",ch:")]
    plan = ps.WgradPlan(p, mode=mode, device=0, recipe=recipe)
    plan.forward(torch.from_numpy(x).to(dev), torch.from_numpy(dy).to(dev), dw)
    torch.cuda.synchronize()
    got = dw.cpu().numpy()
    assert np.isfinite(got).all()
    err = oracle.rel_l2(got, ref)
    print(f"wgrad {conv} {mode} {plan.recipe} relL2={err:.2e}")
    assert err <= TOL[mode], f"relL2 {err:.3e} ({plan.recipe})"


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
def test_backward_weight_resnet_layer(mode):
    """ResNet-50 l1 3x3 shape at N = 32 (the K = 64 swapped-role tiles, 56x56 boxes) and
    bitwise run-to-run reproducibility (fixed split order)."""
    p = ps.ConvPreset.parse("conv:32,64,64,56,56,3,3,1,1,16,1,1,56,56")
    rng = np.random.default_rng(27)
    x = rng.uniform(-1, 1, p.input_elems()).astype(np.float32)
    dy = rng.uniform(-1, 1, p.output_elems()).astype(np.float32)
    ref = _wgrad_ref(p, x, dy)
    dev = torch.device("cuda:0")
    xd, dyd = torch.from_numpy(x).to(dev), torch.from_numpy(dy).to(dev)
    plan = ps.WgradPlan(p, mode=mode, device=0)
    outs = []
    for _ in range(2):
        dw = torch.full((p.filter_elems(),), float("nan"), device=dev)
        plan.forward(xd, dyd, dw)
        torch.cuda.synchronize()
        outs.append(dw.cpu().numpy())
    assert oracle.rel_l2(outs[0], ref) <= TOL[mode], plan.recipe
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32"])
@pytest.mark.parametrize("conv,c_log", [("conv:2,64,16,16,16,7,7,2,2,16,3,3,32,32", 3),   # stem-shaped
                                        ("conv:3,32,16,9,9,3,3,1,1,16,1,1,9,9", 5),
                                        ("conv:2,64,16,8,8,5,5,2,2,16,2,2,16,16", 16)])
def test_backward_weight_tap_fold(conv, c_log, mode):
    """Few-channel layers (pp:C): the 1x1 wgrad over the tap-folded input; the padded channels
    of X are zero and their dW is zero."""
    p = ps.ConvPreset.parse(conv)
    rng = np.random.default_rng(28)
    x = rng.uniform(-1, 1, p.input_elems()).astype(np.float32)
    x.reshape(p.nImg, 1, p.ifh, p.ifw, 16)[..., c_log:] = 0.0
    dy = rng.uniform(-1, 1, p.output_elems()).astype(np.float32)
    ref = _wgrad_ref(p, x, dy)
    dev = torch.device("cuda:0")
    dw = torch.full((p.filter_elems(),), float("nan"), device=dev)
    plan = ps.WgradPlan(p, mode=mode, device=0, recipe=f"gpu=pp:{c_log}")
    assert "pp:" in plan.recipe
    plan.forward(torch.from_numpy(x).to(dev), torch.from_numpy(dy).to(dev), dw)
    torch.cuda.synchronize()
    got = dw.cpu().numpy()
    err = oracle.rel_l2(got, ref)
    assert err <= TOL[mode], f"relL2 {err:.3e} ({plan.recipe})"


def test_backward_weight_rejects():
    with pytest.raises(ps.ConfigRejectedError):
        ps.WgradPlan(ps.ConvPreset.parse("conv:8,64,64,10,10,3,3,1,1,16,1,1,10,10"), mode="f16x2")
    with pytest.raises(ps.ConfigRejectedError):
        ps.WgradPlan(ps.ConvPreset.parse("conv:8,64,64,10,10,3,3,1,1,16,1,1,10,10"), recipe="gpu=box:7x1")
    with pytest.raises(ps.ConfigRejectedError):
        ps.WgradPlan(ps.ConvPreset.parse("conv:8,64,64,10,10,3,3,1,1,16,1,1,10,10"), recipe="gpu=zz:1")


@pytest.mark.gpu
def test_f16x2_forward_host_chunks():
    """f16x2 behind conv_fwd_host: every chunk launch runs its own input |max| pass (the two
    scale slots alternate per launch); result within the faithful bound of the oracle."""
    conv = "conv:200,32,32,56,56,3,3,1,1,16,1,1,56,56"
    p = ps.ConvPreset.parse(conv)
    sx, sw = seeds(27)
    x = oracle.fill_input(p, sx, 32)
    w = oracle.fill_filter(p, sw, 32)
    x[: x.size // 2] *= 1e-3  # the chunks see different input ranges
    plan = ps.ConvPlan(p, mode="f16x2", device=0)
    hy = np.full(p.output_elems(), np.nan, dtype=np.float32)
    plan.forward_host(x.ravel(), w.ravel(), hy, img_begin=0, img_count=p.nImg)
    torch.cuda.synchronize()
    ref = oracle.conv(p, x, w).ravel()
    per = p.output_elems(1)
    for lo, hi in ((0, 5), (195, 200)):  # images from early and late chunks
        assert oracle.rel_l2(hy[lo * per:hi * per], ref[lo * per:hi * per]) <= TOL["f16x2"]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["3xtf32", "tf32", "f16x2"])
def test_empty_image_range_is_a_noop(mode):
    """img_count = 0 launches nothing and leaves the output untouched (every mode)."""
    p = ps.ConvPreset.parse("conv:4,64,64,10,10,3,3,1,1,16,1,1,10,10")
    dev = torch.device("cuda:0")
    x = torch.ones(p.input_elems(), device=dev)
    w = torch.ones(p.filter_elems(), device=dev)
    y = torch.full((p.output_elems(),), 7.0, device=dev)
    plan = ps.ConvPlan(p, mode=mode, device=0)
    plan.forward(x, w, y, img_begin=2, img_count=0)
    torch.cuda.synchronize()
    assert bool((y == 7.0).all())


@pytest.mark.gpu
@pytest.mark.parametrize("conv,c_log,recipe", [
    # cfg1's shape (2 column tiles of 30, 4-row tiles), resident filter, single CTA and pair
    ("conv:4,64,64,56,56,3,3,1,1,16,1,1,56,56", 64, "gpu=bn:64,tc:1,cl:1"),
    ("conv:4,64,64,56,56,3,3,1,1,16,1,1,56,56", 64, "gpu=bn:64,tc:1,cl:2"),
    ("conv:4,64,64,56,56,3,3,1,1,16,1,1,56,56", 64, "gpu=bn:64,tc:1,cl:2,kg:1"),
    # B ring instead of the resident filter, two epilogue groups
    ("conv:4,64,64,56,56,3,3,1,1,16,1,1,56,56", 64, "gpu=bn:64,tc:1,cl:1,br:0"),
    ("conv:4,64,64,56,56,3,3,1,1,16,1,1,56,56", 64, "gpu=bn:64,tc:1,cl:1,eg:2"),
    # ragged tiles (21 rows = 5 x 4 + 1, 19 < 30 columns), Cb = 3, bn 32 / 16, unpadded
    ("conv:3,32,48,21,19,3,3,1,1,16,1,1,21,19", 48, "gpu=bn:32,tc:1"),
    ("conv:2,16,32,9,40,3,3,1,1,16,1,1,9,40", 32, "gpu=bn:16,tc:1,br:0"),
    ("conv:2,64,32,10,33,3,3,1,1,16,0,0,12,35", 32, "gpu=bn:64,tc:1,cl:2"),
])
def test_tap_concat(conv, c_log, recipe):
    """TF32 tap concat (recipe tc:1): per filter row one N = 3 bn MMA over shared halo rows
    pitched at 32 pixels; the epilogue adds D_ki shifted by ki rows with warp shuffles."""
    n = ps.ConvPreset.parse(conv).nImg
    _check("tc", conv, c_log, 23, "tf32", n, recipe)


@pytest.mark.gpu
def test_tap_concat_rejected_outside_its_domain():
    for conv, mode, recipe in [
        ("conv:2,64,64,8,8,3,3,1,1,16,1,1,8,8", "3xtf32", "gpu=bn:64,tc:1"),   # TF32 only
        ("conv:2,128,64,8,8,3,3,1,1,16,1,1,8,8", "tf32", "gpu=bn:128,tc:1"),  # N = 3 bn > 192
        ("conv:2,128,64,8,8,3,3,1,1,16,1,1,8,8", "tf32", "gpu=bn:64,tc:1"),   # two N tiles
        ("conv:2,64,64,8,8,3,3,2,2,16,1,1,16,16", "tf32", "gpu=bn:64,tc:1"),  # stride 2
        ("conv:2,64,64,8,8,5,5,1,1,16,2,2,8,8", "tf32", "gpu=bn:64,tc:1"),    # 5x5
    ]:
        with pytest.raises(ps.ConfigRejectedError):
            ps.ConvPlan(ps.ConvPreset.parse(conv), mode=mode, device=0, recipe=recipe)
