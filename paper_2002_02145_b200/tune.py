"""Empirical top-k schedule selection (PolyScientist's last step: "run the
top-k variants and pick the best").

The closed-form model (csrc/select.cpp, conv_select_topk) ranks the recipe space; the top-k
plus the structural alternatives the model is least sure about (CTA pair on/off, BN one step
down) are timed on the device with the bench protocol (prepacked filter, L2 flushed, median of
repeats). Results go to a plan cache keyed by the descriptor and mode, and to a report in the
reference's tab-separated `rows` style (pipeline.hpp:232-278: one `ranked` row per variant).
"""
from __future__ import annotations

import json
import os
import statistics

from . import ConfigRejectedError, ConvPlan, ConvPreset, fill_filter, fill_input, select_topk
from .timing import L2Flush

CACHE_ENV = "PSCONV_PLAN_CACHE"
# The committed plan cache: the measured best recipe per (descriptor, mode) of every bench
# workload (BASELINE configs, the ResNet-50 sweep, cfg5's per-GPU shards), written by
# `bench.py --tune-plans K` on a B200. bench.py and the GPU parity tests run these recipes.
PLANS_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "plans_b200.json")


def lookup(preset: ConvPreset, mode: str, path: str | None = None) -> str | None:
    """The cached measured-best recipe of (preset, mode), or None."""
    path = path or PLANS_PATH
    try:
        with open(path) as fh:
            cache = json.load(fh)
    except (OSError, ValueError):
        return None
    e = cache.get(f"{preset}|{mode}")
    return e["recipe"] if e else None


def _variants(preset: ConvPreset, mode: str, k: int, c_logical: int = 0) -> list[str]:
    ranked = [r for r, _ in select_topk(preset, mode, k, c_logical=c_logical if 0 < c_logical < preset.nIfm else 0)]
    out = list(ranked)
    base = ranked[0]
    head, gpu = base.split(";gpu=")
    kv = dict(item.split(":") for item in gpu.split(","))
    alts = []
    if mode == "tf32":
        alts.append({**kv, "cl": "1" if kv.get("cl") == "2" else "2"})
    bn = int(kv["bn"])
    # two epilogue warp groups (alternate 32-channel rounds): faster on some
    # epilogue-heavy layers, slower on others
    if int(kv["bn"]) >= 64:
        alts.append({**kv, "eg": "2"})
    # deep output staging (os:8: 32 KB of the ring become four more staging blocks and the
    # store warp keeps two TMA stores in flight): output-heavy layers, mostly TF32
    if not any(key in kv for key in ("halo", "tc", "pp")):
        alts.append({**kv, "os": "8"})
        if "eg" not in kv:
            alts.append({**kv, "os": "12"})
        if bn >= 64 and "eg" not in kv:
            alts.append({**kv, "eg": "2", "os": "8"})
    if mode in ("3xtf32", "f16x2") and bn == 128:  # TMEM-resident A is opt-in at bn 128
        alts.append({**kv, "ta": "1"})
    widest = max(c for c in (16, 32, 64, 128, 256) if preset.nOfm % c == 0)
    for nb in (bn * 2, bn // 2, widest):
        if 16 <= nb <= 256 and preset.nOfm % nb == 0:
            alt = {**kv, "bn": str(nb)}
            alt.pop("ta", None)
            if mode in ("3xtf32", "f16x2"):
                alt["ch"] = "32" if nb == 256 else "16"
            alts.append(alt)
            if mode in ("3xtf32", "f16x2") and nb == 128:  # (l2 1x1 128->512: 183 -> 160 us)
                alts.append({**alt, "ta": "1"})
    # tail split-K: the model's split decision both ways
    # (kt:1 splits every tile instead of the tail wave: faster on some 3xTF32 layers)
    if "ks" in kv:
        alts += [{**kv, "ks": "1"}, {**kv, "kt": "1"}]
    else:
        alts += [{**kv, "ks": "2"}, {**kv, "ks": "3"}, {**kv, "ks": "3", "kt": "1"}]
    # (c,s) fold when the caller knows only c_logical <= 8 of the 16 input channels are
    # real (the stem): the same top candidates over the folded input
    if 0 < c_logical <= 8 and preset.nIfm == 16 and preset.kw > 1:
        for rid in ranked[:2]:
            h2, g2 = rid.split(";gpu=")
            kv2 = dict(item.split(":") for item in g2.split(","))
            kv2.pop("box", None)  # the folded layer has its own box candidates
            kv2.pop("ch", None)
            alts.append({**kv2, "fold": str(c_logical)})
    # 3xTF32 halo mode with the N-concat filter rows and ONE accumulation chunk (the lean
    # 3x3 issuer needs it; <= 40 k-steps keeps the chunk error ~5e-6): the model ranks it
    # low, measured best on the K = 64 3x3 layers
    ksteps = preset.nIfm // 16 * preset.kh * preset.kw
    if (mode == "3xtf32" and preset.stride_h == preset.stride_w == 1 and preset.kh * preset.kw > 1
            and bn <= 64 and ksteps <= 40):
        alts.append({"bn": str(bn), "halo": "1", "ch": str(ksteps), "eg": "2"})
    # TF32 tap concat (halo rows pitched at 32 px, one N = 3 bn MMA per filter row): the
    # K <= 64 3x3 layers, where N = 64 MMAs run at 2/3 of the tensor rate
    if (mode == "tf32" and preset.kh == preset.kw == 3 and preset.stride_h == preset.stride_w == 1
            and preset.nOfm <= 64 and preset.nOfm % 16 == 0):
        for extra in ({}, {"eg": "2"}, {"br": "0"}):
            alts.append({"bn": str(preset.nOfm), "tc": "1", "cl": "1", **extra})
    # few-channel kernel (conv_pp.cuh) when at most 4 input channels are real: tap pairs
    # straight from the input's parity planes, no folded copy
    if (0 < c_logical <= 4 and preset.nIfm == 16 and preset.stride_h == preset.stride_w <= 2
            and 2 <= preset.kh * preset.kw <= 64):
        for pbn in (64, 128):
            if preset.nOfm % pbn == 0:
                alts.append({"bn": str(pbn), "pp": str(c_logical)})
    for a in alts:
        rid = head + ";gpu=" + ",".join(f"{key}:{val}" for key, val in a.items())
        if rid not in out:
            out.append(rid)
    return out


def time_recipe(preset, mode, recipe, x, w, y, flush, stream, reps=5, warm=2) -> float:
    import torch
    plan = ConvPlan(preset, mode=mode, device=x.device.index or 0, recipe=recipe)
    plan.prepack(w, stream)
    f = lambda: plan.forward(x, None, y, stream=stream, prepacked=True)  # noqa: E731
    for _ in range(warm):
        f()
    ts = []
    for _ in range(reps):
        flush()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        f()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    plan.close()
    return statistics.median(ts)


def autotune(preset: ConvPreset, mode: str = "3xtf32", k: int = 4, device: int = 0,
             c_logical: int = 0, seeds=(1, 2), cache_path: str | None = None,
             report_path: str | None = None) -> tuple[str, list[tuple[str, float, float]]]:
    """Returns (best recipe id, [(recipe, model_us, measured_us), ...] best first)."""
    import torch
    from . import model_us
    cache_path = cache_path or os.environ.get(CACHE_ENV)
    key = f"{preset}|{mode}"
    if cache_path and os.path.exists(cache_path):
        with open(cache_path) as fh:
            cache = json.load(fh)
        if key in cache:
            return cache[key]["recipe"], [tuple(r) for r in cache[key]["ranked"]]
    dev = torch.device("cuda", device)
    stream = torch.cuda.current_stream(dev)
    x = torch.empty(preset.input_elems(), dtype=torch.float32, device=dev)
    w = torch.empty(preset.filter_elems(), dtype=torch.float32, device=dev)
    y = torch.empty(preset.output_elems(), dtype=torch.float32, device=dev)
    fill_input(preset, seeds[0], x, c_logical=c_logical)
    fill_filter(preset, seeds[1], w, c_logical=c_logical)
    flush = L2Flush(dev)
    rows = []
    for rid in _variants(preset, mode, k, c_logical):
        try:
            ms = time_recipe(preset, mode, rid, x, w, y, flush, stream)
        except ConfigRejectedError:
            continue
        rows.append((rid, model_us(preset, rid, mode), ms * 1e3))
    rows.sort(key=lambda r: (r[2], r[0]))
    best = rows[0][0]
    if cache_path:
        cache = {}
        if os.path.exists(cache_path):
            with open(cache_path) as fh:
                cache = json.load(fh)
        cache[key] = {"recipe": best, "ranked": rows}
        with open(cache_path, "w") as fh:
            json.dump(cache, fh, indent=1, sort_keys=True)
    if report_path:
        with open(report_path, "a") as fh:
            for i, (rid, mu, us) in enumerate(rows):
                fh.write(f"ranked\t{key}\t{i + 1}\t{rid}\tmodel_us={mu:.1f}\tmeasured_us={us:.1f}\n")
    return best, rows
