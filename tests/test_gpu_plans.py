"""Parity of every configuration bench.py times (VERDICT r1 "parity-test every config you
actually time"): each entry of the committed plan cache (paper_2002_02145_b200/plans_b200.json:
27 shapes x {3xTF32, TF32} + cfg5 and its 1/2/4/8-GPU shards x {3xTF32, TF32, f16x2}) runs
its tuned recipe at the descriptor's FULL image count -- so pixel boxes spanning 128 images
form whole tiles -- and one image per 128-image group plus the last is checked against the
CPU oracle (the identity-order Fig. 5 nest, pinned bit-exactly to the reference IR)."""
import functools
import json

import numpy as np
import pytest

import oracle
from paper_2002_02145_b200.tune import PLANS_PATH
from tests.cases import ALL, seeds, with_images

torch = pytest.importorskip("torch")
ps = pytest.importorskip("paper_2002_02145_b200")

TOL = {"3xtf32": 1e-5, "tf32": 5e-3, "f16x2": 1e-5}
PLANS = json.load(open(PLANS_PATH))


def _workload_of(conv):
    """(name, c_logical, cfg_id) of the named workload this descriptor is (a shard of): same
    descriptor up to the image count (the cache key is the canonical `conv:` string)."""
    from dataclasses import astuple
    key = astuple(ps.ConvPreset.parse(conv))[1:]
    for name, (c, c_log, cid) in ALL.items():
        if astuple(ps.ConvPreset.parse(c))[1:] == key:
            return name, c_log, cid
    raise KeyError(conv)


def _images(n):
    return sorted(set(range(0, n, 128)) | {n - 1})


@functools.lru_cache(maxsize=4)
def _oracle(conv, c_log, cid):
    p = ps.ConvPreset.parse(conv)
    sx, sw = seeds(cid)
    imgs = _images(p.nImg)
    w = oracle.fill_filter(p, sw, c_log)
    xs = np.concatenate([oracle.fill_input(p, sx, c_log, img_begin=i, img_count=1) for i in imgs])
    return imgs, oracle.conv(ps.ConvPreset.parse(with_images(conv, len(imgs))), xs, w)


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(PLANS), ids=lambda k: k.split(":", 1)[1].replace(",", "_"))
def test_tuned_plan_full_size(key):
    conv, mode = key.rsplit("|", 1)
    recipe = PLANS[key]["recipe"]
    name, c_log, cid = _workload_of(conv)
    p = ps.ConvPreset.parse(conv)
    sx, sw = seeds(cid)
    dev = torch.device("cuda:0")
    x = torch.empty(p.input_elems(), device=dev)
    w = torch.empty(p.filter_elems(), device=dev)
    y = torch.full((p.output_elems(),), float("nan"), device=dev)
    ps.fill_input(p, sx, x, c_logical=c_log)
    ps.fill_filter(p, sw, w, c_logical=c_log)
    plan = ps.ConvPlan(p, mode=mode, device=0, recipe=recipe)
    plan.forward(x, w, y)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(y).all()), f"{name} {mode}: unwritten outputs ({plan.recipe})"
    imgs, ref = _oracle(conv, c_log, cid)
    per = p.output_elems(n_img=1)
    worst = 0.0
    for k, i in enumerate(imgs):
        worst = max(worst, oracle.rel_l2(y[i * per:(i + 1) * per].cpu().numpy(), ref[k]))
    print(f"{name} N={p.nImg} {mode} {plan.recipe} images={imgs} relL2={worst:.3e}")
    assert worst <= TOL[mode], f"{name} {mode}: relL2 {worst:.3e} ({plan.recipe})"
    plan.close()
