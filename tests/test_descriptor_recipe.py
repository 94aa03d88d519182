"""Host logic (CPU): conv-layer descriptor and recipe grammar, mirroring the reference's
ConvPreset (presets.hpp:26-58), the `conv:` loader (cli.hpp:54-66) and VariantRecipe /
plan_recipe (variants.hpp:16-65, 186-228), with the reference's error classes (status 2)."""
import os

import pytest

import paper_2002_02145_b200 as ps
from paper_2002_02145_b200 import ConfigRejectedError, ConvPreset

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_default_preset_fields():
    p = ConvPreset.parse("conv:2,32,32,4,4,3,3,1,1,16")
    assert (p.nImg, p.nOfm, p.nIfm, p.ofh, p.ofw, p.kh, p.kw, p.stride_h, p.stride_w,
            p.gemm_block) == (2, 32, 32, 4, 4, 3, 3, 1, 1, 16)
    assert (p.pad_h, p.pad_w, p.ifh, p.ifw) == (0, 0, 6, 6)  # implied extent (presets.hpp:88-91)
    assert str(p) == "conv:2,32,32,4,4,3,3,1,1,16"


@pytest.mark.parametrize("bad", [
    "conv:1,2,3",                               # tests/test_cli.cpp:295 (not 10 ints)
    "conv:2,33,32,4,4,3,3,1,1,16",              # tests/test_cli.cpp:296 (33 % 16)
    "conv:2,32,32,4,4,3,3,1,0,16",              # non-positive
    "conv:2,32,32,4,4,3,3,1,1,16,1",            # 11 values
    "conv:2,32,32,4,4,x,3,1,1,16",              # bad value
    "gemm:2,32,32,4,4,3,3,1,1,16",              # unknown preset kind
    "conv:2,32,32,4,4,3,3,1,1,16,3,0,4,4",      # pad >= kh
    "conv:2,32,32,4,4,3,3,1,1,16,1,1,2,2",      # input too small for ofh
])
def test_rejected_descriptors(bad):
    with pytest.raises(ConfigRejectedError):
        ConvPreset.parse(bad)


def test_whitespace_and_empty_fields_like_reference():
    # presets.hpp:29-42: whitespace dropped, empty fields skipped
    p = ConvPreset.parse("conv: 2, 32,,32 ,4,4,3,3,1,1,16")
    assert (p.nImg, p.nOfm, p.nIfm) == (2, 32, 32)
    q = ConvPreset.parse("2,32,32,4,4,3,3,1,1,16")  # ConvPreset::parse form (no prefix)
    assert q == p


def test_extension_round_trip():
    s = "conv:56,128,128,28,28,3,3,2,2,16,1,1,56,56"
    p = ConvPreset.parse(s)
    assert str(p) == s and ConvPreset.parse(str(p)) == p
    assert p.flops() == 2 * 56 * 128 * 128 * 28 * 28 * 9


@pytest.mark.parametrize("i", range(7))
def test_emission_matches_reference_emitter(i):
    import json
    idx = json.load(open(os.path.join(GOLDEN, "index.json")))["emit"][i]
    want = open(os.path.join(GOLDEN, idx["file"])).read()
    got = ps.emit_driver(ConvPreset.parse(idx["conv"]), idx["recipe"])
    assert got == want


@pytest.mark.parametrize("recipe", [
    "perm=oi,ofm_tile",          # band loop permuted (InvalidPermutationError)
    "perm=ofm_tile,ofm_tile",    # listed twice
    "perm=foo",                  # unknown loop
    "tile=oj:0",                 # TileSizeNonPositiveError
    "tile=ifm:2",                # tiles band loop
    "tile=oj",                   # bad entry
    "order=ofm_tile",            # unknown clause
    "tile=oj:2,oj:4",            # tiled twice
])
def test_rejected_recipes(recipe):
    with pytest.raises(ConfigRejectedError):
        ps.emit_driver(ConvPreset(), recipe)


def test_select_topk_deterministic_and_resolvable():
    p = ConvPreset.parse("conv:2048,256,256,14,14,3,3,1,1,16,1,1,14,14")
    a = ps.select_topk(p, "3xtf32", 5)
    b = ps.select_topk(p, "3xtf32", 5)
    assert a == b and len(a) == 5
    us = [u for _, u in a]
    assert us == sorted(us)
    for rid, u in a:
        assert rid.startswith("perm=") and ";gpu=bn:" in rid
        assert abs(ps.model_us(p, rid, "3xtf32") - u) < 1e-6 * max(1.0, u)


def test_model_scales_with_work():
    small = ConvPreset.parse("conv:256,256,256,14,14,3,3,1,1,16,1,1,14,14")
    big = ConvPreset.parse("conv:2048,256,256,14,14,3,3,1,1,16,1,1,14,14")
    r = "perm=ofm_tile,ifm_tile,oj,kj,ki;gpu=bn:256,box:2x2x32"
    assert ps.model_us(big, r) > 4 * ps.model_us(small, r)
    assert ps.model_us(big, r, "tf32") < ps.model_us(big, r, "3xtf32")


def test_gpu_clause_validation():
    p = ConvPreset.parse("conv:8,64,64,8,8,3,3,1,1,16,1,1,8,8")
    with pytest.raises(ConfigRejectedError):
        ps.model_us(p, "gpu=bn:48")             # not a supported tile width
    with pytest.raises(ConfigRejectedError):
        ps.model_us(p, "gpu=bn:128")            # 64 % 128
    with pytest.raises(ConfigRejectedError):
        ps.model_us(p, "gpu=box:16x16x1")       # > 128 rows
    assert ps.model_us(p, "gpu=bn:32,box:8x8x2,ch:4") > 0


def test_split_k_recipe_keys():
    """Tail split-K (ks) and its scope (kt): ~1.3 waves of tiles -> the split of the
    partial wave is modelled faster; kt:1 (every tile split) is accepted, kt:2 is not."""
    p = ConvPreset.parse("conv:256,512,512,7,7,3,3,1,1,16,1,1,7,7")
    base = "gpu=bn:256,box:1x1x128,cl:1,ch:36"
    assert ps.model_us(p, base + ",ks:3", "3xtf32") < ps.model_us(p, base + ",ks:1", "3xtf32")
    assert ps.model_us(p, base + ",ks:3,kt:1", "3xtf32") > 0
    for bad in (",kt:2", ",ks:0", ",ks:65"):
        with pytest.raises(ConfigRejectedError):
            ps.model_us(p, base + bad, "3xtf32")


def test_epilogue_groups_recipe_key():
    """eg:2 (two epilogue warp groups) round-trips through the canonical recipe id;
    eg:1 is the default and is not shown; other values are rejected."""
    p = ConvPreset.parse("conv:8,128,64,8,8,3,3,1,1,16,1,1,8,8")
    top = ps.select_topk(p, "tf32", 1)[0][0]
    assert "eg:" not in top
    for bad in ("gpu=bn:64,eg:0", "gpu=bn:64,eg:3"):
        with pytest.raises(ConfigRejectedError):
            ps.model_us(p, bad, "tf32")
    assert ps.model_us(p, "gpu=bn:128,eg:2", "tf32") > 0
    with pytest.raises(ConfigRejectedError):  # accumulation chunks are 3xTF32-only
        ps.model_us(p, "gpu=bn:64,ch:4", "tf32")


def test_output_staging_recipe_key():
    """os:8 / 12 / 16 (8 KB output staging blocks, deferred hand-back in the store warp) is a
    non-halo option of the main kernel: 4 is the default and not shown, other values and
    halo / pp combinations are rejected."""
    p = ConvPreset.parse("conv:8,128,64,8,8,3,3,1,1,16,1,1,8,8")
    assert "os:" not in ps.select_topk(p, "tf32", 1)[0][0]
    assert ps.model_us(p, "gpu=bn:128,os:8", "tf32") > 0
    assert ps.model_us(p, "gpu=bn:128,os:4", "3xtf32") > 0
    assert ps.model_us(p, "gpu=bn:128,os:16", "tf32") > 0
    for bad in ("gpu=bn:64,os:2", "gpu=bn:64,os:32", "gpu=bn:64,halo:1,os:8", "gpu=bn:64,eg:2,os:12"):
        with pytest.raises(ConfigRejectedError):
            ps.model_us(p, bad, "tf32")


def test_select_topk_with_real_channel_count():
    """conv_select_topk_ex: with the caller's assertion that only 3 of the 16 input channels are
    real, the few-channel kernel's recipe joins the ranking (and wins on the ResNet stem);
    without it the descriptor alone never yields pp:."""
    stem = ConvPreset.parse("conv:256,64,16,112,112,7,7,2,2,16,3,3,224,224")
    for mode in ("3xtf32", "tf32"):
        assert all("pp:" not in r for r, _ in ps.select_topk(stem, mode, 8))
        top, us = ps.select_topk(stem, mode, 2, c_logical=3)[0]
        assert "pp:3" in top and us > 0
    # a 64-channel layer ignores the hint
    p = ConvPreset.parse("conv:8,64,64,8,8,3,3,1,1,16,1,1,8,8")
    assert ps.select_topk(p, "tf32", 3, c_logical=3) == ps.select_topk(p, "tf32", 3)


def test_parity_plane_recipe_key():
    """pp:C (few-channel kernel): accepted for C <= 4 real channels of one 16-channel block,
    stride 1 or 2, 2..64 taps; canonical id pins the 8x16 pixel tile; modelled far below the
    16-channel kernel on the stem."""
    stem = ConvPreset.parse("conv:256,64,16,112,112,7,7,2,2,16,3,3,224,224")
    pp = ps.model_us(stem, "gpu=pp:3", "tf32")
    assert 0 < pp < ps.model_us(stem, "gpu=bn:64", "tf32") / 3
    top = ps.select_topk(stem, "tf32", 1)[0][0]
    assert "pp:" not in top  # opt-in: the selector cannot know the real channel count
    bad = [("gpu=pp:5", stem), ("gpu=pp:3,fold:3", stem), ("gpu=bn:256,pp:3", stem),
           ("gpu=pp:3", ConvPreset.parse("conv:2,64,32,8,8,3,3,1,1,16,1,1,8,8")),   # nIfm 32
           ("gpu=pp:3", ConvPreset.parse("conv:2,64,16,8,8,1,1,1,1,16,0,0,8,8")),   # 1 tap
           ("gpu=pp:3", ConvPreset.parse("conv:2,64,16,8,8,3,3,3,3,16,1,1,24,24"))]  # stride 3
    for rid, p in bad:
        with pytest.raises(ConfigRejectedError):
            ps.model_us(p, rid, "tf32")


def test_f16x2_mode_selection():
    """f16x2 plans through the same selector: half the 3xTF32 MMA work is modelled faster on a
    compute-bound layer; halo and the few-channel kernel are rejected for it."""
    cfg5 = ConvPreset.parse("conv:2048,256,256,14,14,3,3,1,1,16,1,1,14,14")
    top = ps.select_topk(cfg5, "f16x2", 2)
    assert len(top) == 2 and all("ch:" in r for r, _ in top)  # chunked sums as in 3xTF32
    assert ps.model_us(cfg5, top[0][0], "f16x2") < ps.model_us(cfg5, top[0][0], "3xtf32")
    with pytest.raises(ConfigRejectedError):
        ps.model_us(cfg5, "gpu=bn:256,halo:1", "f16x2")
    # the few-channel kernel has no fp16 variant: f16x2 pp plans run its 3xTF32 arithmetic
    stem = ConvPreset.parse("conv:2,64,16,16,16,7,7,2,2,16,3,3,32,32")
    assert ps.model_us(stem, "gpu=pp:3", "f16x2") == ps.model_us(stem, "gpu=pp:3", "3xtf32")
    with pytest.raises(ConfigRejectedError):
        ps.model_us(cfg5, "gpu=bn:256,cl:2", "f16x2")  # the CTA pair is TF32-only


def _random_recipes(n, seed=2024):
    import random
    rng = random.Random(seed)
    loops = ["img", "ofm_tile", "ifm_tile", "oj", "kj", "ki"]
    out = []
    for _ in range(n):
        perm = loops[1:] if rng.random() < 0.7 else loops[:]
        perm = perm[:]
        rng.shuffle(perm)
        k = rng.randint(1, len(perm))
        parts = ["perm=" + ",".join(perm[:k])]
        tiles = rng.sample(["oj", "ofm_tile", "ifm_tile", "kj", "img"], rng.randint(0, 3))
        if tiles:
            parts.append("tile=" + ",".join(f"{t}:{rng.randint(1, 5)}" for t in tiles))
        out.append(";".join(parts))
    return out


@pytest.mark.parametrize("conv", ["conv:3,48,32,7,5,3,3,1,1,16", "conv:5,32,64,9,4,3,2,2,1,16"])
def test_emission_matches_live_reference_emitter(conv):
    """Randomised recipes (several loops tiled, tiles that do not divide their trip counts,
    so nested partial-tile versions) vs the reference emitter itself (emit.hpp:60-134 via
    oracle/_ref, this container only): byte-identical text."""
    import oracle
    if not oracle.ref_available():
        pytest.skip("reference emitter not built here")
    csv10 = conv.split(":", 1)[1]
    n = 0
    for r in _random_recipes(120):
        try:
            want = oracle.ref_emit(csv10, r)
        except RuntimeError:  # the reference rejects it: so must we
            with pytest.raises(ConfigRejectedError):
                ps.emit_driver(ConvPreset.parse(conv), r)
            continue
        assert ps.emit_driver(ConvPreset.parse(conv), r) == want, r
        n += 1
    assert n >= 60


def test_wgrad_geometry_all_resnet_shapes():
    """Backward-weight geometry (conv_wgrad_describe, host only) for every bench layer in both
    modes: an M = 128 tile, a legal MMA N, whole K=8 steps per pixel box, and a ring that fits."""
    import re

    from paper_2002_02145_b200.workloads import ALL
    for name, (conv, _c, _i) in ALL.items():
        p = ps.ConvPreset.parse(conv)
        for mode in ("tf32", "3xtf32"):
            d = ps.WgradPlan.describe(p, mode)
            kv = dict(re.findall(r"(\w+):([\dx]+)", d))
            sw, kn, cn, nt = (int(kv[k]) for k in ("sw", "kn", "cn", "nt"))
            m = nt * cn if sw else kn
            bn = kn if sw else nt * cn
            assert m == 128, (name, mode, d)
            assert bn in (32, 64, 128, 192, 256) and (mode == "tf32" or bn <= 128), (name, mode, d)
            qb, pb = (int(v) for v in kv["box"].split("x"))
            assert (qb * pb) % 8 == 0 and qb * pb <= 256, (name, mode, d)
            assert int(kv["stage_bytes"]) * int(kv["st"]) <= 227 * 1024 - 6144, (name, mode, d)


def test_wgrad_recipe_override_and_errors():
    p = ps.ConvPreset.parse("conv:8,128,64,10,10,3,3,1,1,16,1,1,10,10")
    d = ps.WgradPlan.describe(p, "tf32", recipe="gpu=sw:0,kn:128,cn:64,nt:3,box:10x4,sp:5,st:3")
    assert d.startswith("gpu=sw:0,kn:128,cn:64,nt:3,box:10x4,sp:5,st:3")
    for bad in ("gpu=box:7x1", "gpu=zz:1", "gpu=nt:3,cn:64,sw:0", "sw:0"):
        with pytest.raises(ps.ConfigRejectedError):
            ps.WgradPlan.describe(p, "3xtf32", recipe=bad)
