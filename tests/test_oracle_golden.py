"""Oracle pinning (CPU): the C restatement of the reference nest vs goldens produced by the
reference's own IR executed numerically (tests/golden/make_golden.py)."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2002_02145_b200 import ConvPreset

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
INDEX = json.load(open(os.path.join(GOLDEN, "index.json")))


def _load(entry):
    f, key = entry["array"].split(":")
    z = np.load(os.path.join(GOLDEN, f))
    return z["input"], z["filter"], z[key]


@pytest.mark.parametrize("entry", INDEX["numeric"], ids=lambda e: f"{e['case']}-{e['recipe']}")
def test_generator_reproduces_golden_inputs(entry):
    p = ConvPreset.parse(entry["conv"])
    x, w, _ = _load(entry)
    sx, sw = entry["seeds"]
    assert np.array_equal(oracle.fill_input(p, sx), x)
    assert np.array_equal(oracle.fill_filter(p, sw), w)


@pytest.mark.parametrize("entry", [e for e in INDEX["numeric"] if e["recipe"] is None],
                         ids=lambda e: e["case"])
def test_fig5_oracle_bit_exact_vs_reference_ir(entry):
    """Identity order: same fp32 accumulation order as the reference program order."""
    p = ConvPreset.parse(entry["conv"])
    x, w, ref = _load(entry)
    got = oracle.conv(p, x, w)
    assert np.array_equal(got, ref)
    n_points = p.nImg * p.nOfm * p.nIfm * p.ofh * p.ofw * p.kh * p.kw
    assert entry["iterations"] == n_points  # execution count (oracle.hpp:45-74)


@pytest.mark.parametrize("entry", [e for e in INDEX["numeric"] if e["recipe"]],
                         ids=lambda e: f"{e['case']}-{e['recipe']}")
def test_recipe_variants_agree_within_fp32(entry):
    """apply_recipe reorders only the reduction order: results differ by fp32 rounding only."""
    p = ConvPreset.parse(entry["conv"])
    x, w, ref = _load(entry)
    got = oracle.conv(p, x, w)
    assert oracle.rel_l2(got, ref) < 1e-6


@pytest.mark.parametrize("entry", [e for e in INDEX["numeric"] if e["recipe"] is None],
                         ids=lambda e: e["case"])
def test_oracle_vs_float64(entry):
    p = ConvPreset.parse(entry["conv"])
    x, w, ref = _load(entry)
    assert oracle.rel_l2(ref, oracle.conv_f64(p, x, w)) < 1e-6


def test_padding_equivalence():
    """pad extension: conv over an unpadded input with pad=1 == reference nest over the
    explicitly zero-padded input (the reference's implied extent, presets.hpp:88-91)."""
    p = ConvPreset.parse("conv:2,32,32,6,6,3,3,1,1,16,1,1,6,6")
    x = oracle.fill_input(p, 5)
    w = oracle.fill_filter(p, 6)
    xp = oracle.pad_input(p, x)
    assert xp.shape[2:4] == (8, 8)
    assert np.all(xp[:, :, 0] == 0) and np.all(xp[:, :, :, 0] == 0)
    assert np.array_equal(xp[:, :, 1:7, 1:7], x)
    out = oracle.conv_fig5(p, xp, w)
    assert oracle.rel_l2(out, oracle.conv_f64(p, x, w)) < 1e-6


@pytest.mark.skipif(not oracle.ref_available(), reason="reference interpreter not built here")
@pytest.mark.parametrize("csv", ["3,32,48,5,6,3,2,2,1,16", "1,64,16,9,3,1,3,1,3,16"])
def test_live_reference_ir(csv):
    class P:
        pass
    p = ConvPreset.parse("conv:" + csv)
    x = oracle.fill_input(p, 123)
    w = oracle.fill_filter(p, 456)
    xp = oracle.pad_input(p, x)
    ref, _ = oracle.ref_interp(csv, xp, w, (p.nImg, p.nOfm // 16, p.ofh, p.ofw, 16))
    assert np.array_equal(oracle.conv_fig5(p, xp, w), ref)


def test_generator_values_exact_and_in_range():
    v = np.array([oracle.value(7, i) for i in range(4096)], np.float64)
    assert v.min() >= -1.0 and v.max() < 1.0
    k = (v + 1.0) * 2 ** 23
    assert np.all(k == np.round(k))  # k * 2^-23 - 1, exact in fp32
    assert abs(v.mean()) < 0.05


def test_generator_is_shard_independent():
    p = ConvPreset.parse("conv:6,16,32,4,4,3,3,1,1,16,1,1,4,4")
    full = oracle.fill_input(p, 99)
    part = oracle.fill_input(p, 99, img_begin=2, img_count=3)
    assert np.array_equal(full[2:5], part)


def test_stem_channel_padding_zero():
    p = ConvPreset.parse("conv:1,64,16,4,4,7,7,2,2,16,3,3,8,8")
    x = oracle.fill_input(p, 1, c_logical=3)
    w = oracle.fill_filter(p, 2, c_logical=3)
    assert np.all(x[..., 3:] == 0) and np.any(x[..., :3] != 0)
    assert np.all(w[:, :, :, :, 3:, :] == 0)


# ------------------------------------------------------- BASELINE-size pins (slices.json)
SLICES = json.load(open(os.path.join(GOLDEN, "slices.json")))


def _slice(entry):
    import importlib.util
    spec = importlib.util.spec_from_file_location("make_slices", os.path.join(GOLDEN, "make_slices.py"))
    mk = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mk)
    return mk, mk.slice_inputs(entry["conv"], entry["c_logical"], entry["cfg_id"], entry["image"],
                                entry["ofm_blocks"])


@pytest.mark.parametrize("entry", SLICES, ids=lambda e: e["name"])
def test_oracle_bit_exact_vs_reference_ir_at_baseline_size(entry):
    """One-image slices of cfg1/2/3/5 and the stem at full channel / spatial size: the oracle's
    output is bit-identical to the reference IR's (sha256 committed by make_slices.py from
    ConvPreset::build + for_each_iteration), and within 1e-6 of float64."""
    mk, (s, x, w) = _slice(entry)
    got = oracle.conv(s, x, w)
    assert mk.sha(got) == entry["sha256"], f"{entry['name']}: oracle differs from the reference IR"
    assert entry["iterations"] == s.nImg * s.nOfm * s.nIfm * s.ofh * s.ofw * s.kh * s.kw
    assert entry["rel_l2_vs_f64"] < 1e-6


@pytest.mark.slow
@pytest.mark.skipif(not oracle.ref_available(), reason="reference interpreter not built here")
@pytest.mark.parametrize("entry", SLICES, ids=lambda e: e["name"])
def test_live_reference_ir_at_baseline_size(entry):
    """Re-executes the reference IR live (this container only, ~5-9 s per slice)."""
    mk, (s, x, w) = _slice(entry)
    ref, n = oracle.ref_interp(entry["ref_csv10"], oracle.pad_input(s, x), w, (1, s.nOfm // 16, s.ofh, s.ofw, 16))
    assert n == entry["iterations"]
    assert np.array_equal(oracle.conv(s, x, w), ref)
