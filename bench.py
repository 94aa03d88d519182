#!/usr/bin/env python3
"""Bench: blocked fp32 direct-conv forward (the PolyScientist hot path) on B200.

Metric (BASELINE.json): "conv fwd GFLOP/s per layer & fraction of roofline at 1/2/4/8 B200
vs host-CPU ref". Default workload = BASELINE configs[4] ("cfg5", N=2048 3x3 256->256 14x14,
the config the metric is quoted on at 1/2/4/8 GPUs), fp32-faithful 3xTF32 mode; the TF32 fast
mode and the f16x2 faithful split are reported beside it. One step = one conv_fwd pass
(filter repack + conv kernel) over this rank's images [rank*N/W, (rank+1)*N/W) -- strong
scaling, no collective on the hot path. At N=1 the line also carries `layers`: the per-layer
metric (cfg1, cfg2, cfg3, the ResNet-50 stem and stride-2 downsample layers; `--layers all`
for the 27-shape sweep) in both modes, each with its own clock record, verification against
the CPU oracle and the reference CPU driver's time on the same layer.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg5] [--mode 3xtf32]
  python bench.py --impl reference ...   # the reference's own emitted CPU driver (oracle/_ref)
  python bench.py --layers all --no-headline --jsonl profiles/rNN_sweep.jsonl --md ...
  python bench.py --tune-plans 4 --layers all ...  # re-tune and rewrite the plan cache

Prints ONE JSON line on rank 0. Timing: CUDA events on the launching stream, L2 flushed
before every timed step (256 MiB write, then read back), barrier + synchronize around the
timed loop, max over ranks (paper_2002_02145_b200/measure.py describes both protocols).
"""
from __future__ import annotations

import argparse
import ctypes
import importlib.util
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "conv fwd GFLOP/s per layer & fraction of roofline at 1/2/4/8 B200 vs host-CPU ref"
DEFAULT_LAYERS = ("cfg1", "cfg2", "cfg3", "r50_stem", "r50_l2_ds_1x1s2_256_512",
                  "r50_l3_ds_1x1s2_512_1024", "r50_l4_ds_1x1s2_1024_2048")


def _workloads():
    """paper_2002_02145_b200/workloads.py loaded by path: the reference arm must not load the
    product package (its __init__ maps libpsconv.so)."""
    spec = importlib.util.spec_from_file_location(
        "psconv_workloads", os.path.join(ROOT, "paper_2002_02145_b200", "workloads.py"))
    wl = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(wl)
    return wl


class Desc:
    """Pure-Python view of a `conv:` descriptor (reference ConvPreset fields, presets.hpp:13-23,
    + pad / input extent) for the CPU legs: no product library involved."""
    FIELDS = ("nImg", "nOfm", "nIfm", "ofh", "ofw", "kh", "kw", "stride_h", "stride_w",
              "gemm_block", "pad_h", "pad_w", "ifh", "ifw")

    def __init__(self, conv: str):
        v = [int(x) for x in conv.split(":", 1)[-1].split(",")]
        v += [0] * (14 - len(v))
        for k, x in zip(self.FIELDS, v):
            setattr(self, k, x)
        if not self.ifh:
            self.ifh = (self.ofh - 1) * self.stride_h + self.kh - 2 * self.pad_h
        if not self.ifw:
            self.ifw = (self.ofw - 1) * self.stride_w + self.kw - 2 * self.pad_w

    def with_images(self, n):
        d = Desc("conv:" + ",".join(str(getattr(self, k)) for k in self.FIELDS))
        d.nImg = n
        return d

    def flops(self, c_logical=None, n_img=None):
        c = c_logical or self.nIfm
        n = self.nImg if n_img is None else n_img
        return 2 * n * self.nOfm * c * self.ofh * self.ofw * self.kh * self.kw


def run_config(name, conv, c_logical, n_img):
    """The `config` object of both arms (identical keys and values for the same workload)."""
    return {"workload": f"{name} {conv}", "images": n_img, "c_logical": c_logical}


# ----------------------------------------------------------------------------- CPU legs
def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _ref_driver_lib():
    """oracle/_ref/libref_driver_{v4,v3}.so (the reference's emitted driver) + manifest."""
    man = os.path.join(ROOT, "oracle", "_ref", "refdrv.json")
    if not os.path.exists(man):
        return None, None
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        flags = ""
    tag = "v4" if " avx512f" in flags else "v3"
    so = os.path.join(ROOT, "oracle", "_ref", f"libref_driver_{tag}.so")
    if not os.path.exists(so):
        return None, None
    with open(man) as fh:
        return ctypes.CDLL(so), json.load(fh)


class CpuLeg:
    """The reference's CPU path on the host cores: the reference emitter's own Fig. 5 driver for
    the WHOLE workload (oracle/_ref, emit.hpp:60-134, OpenMP over img as presets.hpp:125
    annotates, plain-C band microkernel) -- or, where it was not built, the oracle port."""

    def __init__(self, name, conv, c_logical, cfg_id):
        import numpy as np
        import oracle
        self.np, self.oracle = np, oracle
        self.name, self.conv, self.c_logical = name, conv, c_logical
        self.d = Desc(conv)
        lib, man = _ref_driver_lib()
        if lib is not None and name in man and man[name]["sample_img"] == self.d.nImg:
            self.kind = "reference"
            self.fn = getattr(lib, man[name]["symbol"])
            self.fn.restype = None
            self.fn.argtypes = [ctypes.c_void_p] * 3
        else:
            self.kind, self.fn = "port", None
        sx, sw = 1000 + cfg_id, 2000 + cfg_id
        self.xpad = oracle.pad_input(self.d, oracle.fill_input(self.d, sx, c_logical))
        self.w = oracle.fill_filter(self.d, sw, c_logical)
        self.out = np.zeros((self.d.nImg, self.d.nOfm // 16, self.d.ofh, self.d.ofw, 16), np.float32)

    def rep(self) -> float:
        self.out[...] = 0
        t = time.perf_counter()
        if self.fn is not None:
            self.fn(self.out.ctypes.data, self.w.ctypes.data, self.xpad.ctypes.data)
        else:
            self.oracle.conv_fig5(self.d, self.xpad, self.w, self.out)
        return time.perf_counter() - t

    def run(self, reps, warmup):
        for _ in range(warmup):
            self.rep()
        times = [self.rep() for _ in range(reps)]
        f = self.d.flops(self.c_logical)
        mean = statistics.mean(times)
        what = ("reference emitted Fig.5 driver (oracle/_ref, emit.hpp:60-134) + plain-C band microkernel"
                if self.kind == "reference" else "oracle port (oracle/oracle.c Fig.5 restatement)")
        return {"value": round(f / mean / 1e9, 3), "unit": "GFLOP/s", "cores": self.oracle.threads(),
                "kind": self.kind, "best_value": round(f / min(times) / 1e9, 3),
                "ms_per_rep": round(mean * 1e3, 3),
                "sample": f"all {self.d.nImg} images of {self.name} ({f / 1e9:.2f} GFLOP), {reps} reps after "
                          f"{warmup} warm-up, gcc -O3 OpenMP over img; {what}",
                "cpu_model": _cpu_model()}


# ----------------------------------------------------------------------------- verification
def verify_images(conv, c_logical, cfg_id, images, got: dict):
    """Untimed: the given global images vs the CPU oracle (the identity-order Fig. 5 nest,
    pinned bit-exactly to the reference IR, tests/test_oracle_golden.py). got: img -> array."""
    import numpy as np
    import oracle
    d = Desc(conv)
    sx, sw = 1000 + cfg_id, 2000 + cfg_id
    w = oracle.fill_filter(d, sw, c_logical)
    xs = np.concatenate([oracle.fill_input(d, sx, c_logical, img_begin=i, img_count=1) for i in images])
    ref = oracle.conv(d.with_images(len(images)), xs, w)
    worst_l2, worst_abs = 0.0, 0.0
    for k, i in enumerate(images):
        worst_l2 = max(worst_l2, oracle.rel_l2(got[i], ref[k]))
        worst_abs = max(worst_abs, oracle.max_abs(got[i], ref[k]))
    return {"images": list(images), "max_rel_l2_vs_oracle": float(f"{worst_l2:.3g}"),
            "max_abs_vs_oracle": float(f"{worst_abs:.3g}")}


def sample_images(n, n_box=128):
    """One image per n_box-image group (a TMA box spans up to 128 images) plus the last."""
    return sorted(set(range(0, n, n_box)) | {n - 1})


TOL = {"3xtf32": 1e-5, "tf32": 5e-3, "f16x2": 1e-5}


# ----------------------------------------------------------------------------- GPU arm
def choose_recipe(ps, preset, mode, args, c_logical, seeds, device):
    """Committed plan cache (measured best per descriptor and mode), else the tuner."""
    from paper_2002_02145_b200 import tune
    if args.recipe and mode == args.mode:
        return args.recipe, "command line"
    if args.tune_plans:
        rid, _ = tune.autotune(preset, mode, k=args.tune_plans, device=device, c_logical=c_logical,
                               seeds=seeds, cache_path=args.plans_out or tune.PLANS_PATH,
                               report_path=args.rows)
        return rid, f"tuned now (top-{args.tune_plans} + alternatives)"
    rid = tune.lookup(preset, mode)
    if rid is not None:
        return rid, "plan cache (paper_2002_02145_b200/plans_b200.json)"
    rid, _ = tune.autotune(preset, mode, k=4, device=device, c_logical=c_logical, seeds=seeds)
    return rid, "tuned now (not in the plan cache)"


def measure_layer(ps, meas, name, args, flush, device, hbm, bf16, modes, cpu=True):
    """Per-layer record: both modes, single-launch + steady-state, clocks, verification,
    reference CPU driver on the same layer."""
    wl = _workloads()
    conv, c_log, cid = wl.ALL[name]
    p = ps.ConvPreset.parse(conv)
    seeds = wl.seeds(cid)
    lb = meas.LayerBench(ps, p, c_log, seeds, device)
    imgs = sample_images(p.nImg)
    rec = {"layer": name, "conv": conv, "gflop": round(meas.flops(p, c_log) / 1e9, 3),
           "mb_compulsory": round(meas.compulsory_bytes(p, c_log) / 1e6, 1), "modes": {}}
    outs = {}
    for mode in modes:
        recipe, src = choose_recipe(ps, p, mode, args, c_log, seeds, device)
        plan = ps.ConvPlan(p, mode=mode, device=device, recipe=recipe)
        roof = meas.roofline(p, c_log, mode, hbm, bf16)
        step_ms, kern_ms = lb.single(plan, flush, args.steps, args.warmup)
        with meas.ClockSampler(device) as clk:
            steady_ms, launches, sets = lb.steady(plan, min_seconds=args.layer_seconds)
        clocks = clk.summary()
        # the verified output is the timed plan's (steady state ran on the rotating copies)
        plan.forward(lb.x, lb.w, lb.y, stream=lb.stream)
        import torch
        torch.cuda.synchronize()
        outs[mode] = lb.output_images(imgs)
        km, sm = statistics.mean(kern_ms), statistics.mean(step_ms)
        tr = roof["t_roof_s"] * 1e3
        rec["modes"][mode] = {
            "recipe": plan.recipe, "recipe_source": src, "bound": roof["bound"],
            "roofline_ms": round(tr, 5), "step_ms": round(sm, 5), "kernel_ms": round(km, 5),
            "steady_ms": round(steady_ms, 5),
            "gflops_step": round(roof["flops"] / sm / 1e6, 1),
            "gflops_steady": round(roof["flops"] / steady_ms / 1e6, 1),
            "frac_step": round(tr / sm, 4), "frac_kernel": round(tr / km, 4),
            "frac_steady": round(tr / steady_ms, 4),
            "roofline": meas.roofline_entry(roof, km, hbm),
            "roofline_steady": meas.roofline_entry(roof, steady_ms, hbm),
            "steady_protocol": f"{launches} back-to-back launches over {sets} rotating input/output "
                               f"sets ({sets} x {4 * (p.input_elems() + p.output_elems()) / 1e6:.0f} MB > 2x L2)",
            "clocks": clocks, "clocks_ok": meas.clocks_ok(clocks)}
        plan.close()
    lb.release()
    if not args.no_verify:
        for mode in modes:
            v = verify_images(conv, c_log, cid, imgs, outs[mode])
            v["pass"] = v["max_rel_l2_vs_oracle"] <= TOL[mode]
            rec["modes"][mode]["verified"] = v
    if cpu and not args.no_cpu:
        try:
            leg = CpuLeg(name, conv, c_log, cid)
            r = leg.run(reps=1, warmup=1)
            rec["cpu_reference"] = {k: r[k] for k in ("value", "unit", "cores", "kind", "ms_per_rep")}
        except Exception as e:  # noqa: BLE001
            rec["cpu_reference"] = {"error": str(e)}
    return rec


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2002_02145_b200 as ps
    from paper_2002_02145_b200 import measure as meas
    from paper_2002_02145_b200.dist import gather_shards, image_range
    from paper_2002_02145_b200.timing import L2Flush

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    # collectives: NCCL on the GPU tensors; gloo (CPU tests of the N>1 path on one GPU) on
    # host copies
    cdev = dev if args.dist_backend == "nccl" else torch.device("cpu")
    wl = _workloads()
    conv, c_logical, cfg_id = wl.ALL[args.workload]
    p = ps.ConvPreset.parse(conv)
    N = p.nImg
    b0, n_local = image_range(rank, world, N)
    b1 = b0 + n_local
    sx, sw = wl.seeds(cfg_id)
    # the schedule is chosen for THIS rank's shard: the descriptor of n_local images
    p_local = ps.ConvPreset.parse(wl.with_images(conv, n_local))
    hbm, bf16, peak_src = meas.peaks()
    flush = L2Flush(dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    result = {}
    if not args.no_headline:
        lb = meas.LayerBench(ps, p, c_logical, (sx, sw), local_rank, img_begin=b0, img_count=n_local)
        modes = [args.mode, "tf32" if args.mode != "tf32" else "3xtf32"]
        if args.mode == "3xtf32" and not args.no_f16x2:
            modes.append("f16x2")
        recipes = {}
        if rank == 0:
            for m in modes:
                recipes[m] = choose_recipe(ps, p_local, m, args, c_logical, (sx, sw), local_rank)
        if world > 1:
            obj = [recipes]
            dist.broadcast_object_list(obj, src=0)
            recipes = obj[0]
        legs = {}
        with meas.ClockSampler(local_rank) as clk:
            for m in modes:
                plan = ps.ConvPlan(p, mode=m, device=local_rank, recipe=recipes[m][0])
                barrier()
                torch.cuda.synchronize()
                step_ms, kern_ms = lb.single(plan, flush, args.steps, args.warmup)
                barrier()
                # (means are what the metric is computed from; the medians sit beside them so a
                # pass with a few slow launches -- clock dips under the power cap -- is visible)
                legs[m] = {"plan": plan, "step": max_over_ranks(statistics.mean(step_ms)),
                           "kern": max_over_ranks(statistics.mean(kern_ms)),
                           "step_med": max_over_ranks(statistics.median(step_ms)),
                           "kern_med": max_over_ranks(statistics.median(kern_ms))}
            # steady state of the headline mode (back-to-back, rotating sets)
            steady_ms, steady_n, steady_sets = lb.steady(legs[args.mode]["plan"], min_seconds=0.2)
            steady_ms = max_over_ranks(steady_ms)
            # outputs of each mode for verification / cross-mode checks
            outs = {}
            for m in modes:
                legs[m]["plan"].forward(lb.x, lb.w, lb.y, b0, n_local, stream)
                outs[m] = lb.y[b0 * lb.out_img:b1 * lb.out_img].clone()
            torch.cuda.synchronize()
            plan = legs[args.mode]["plan"]
            # end to end through the public host-buffer entry (C ABI conv_fwd_host)
            hx = torch.empty(n_local * lb.in_img, dtype=torch.float32).pin_memory()
            hw = torch.empty(p.filter_elems(), dtype=torch.float32).pin_memory()
            hy = torch.empty(n_local * lb.out_img, dtype=torch.float32).pin_memory()
            hx.copy_(lb.x[b0 * lb.in_img:b1 * lb.in_img])
            hw.copy_(lb.w)

            def e2e_step():
                plan.forward_host(hx, hw, hy, 0, n_local, stream)

            for _ in range(max(1, args.warmup)):
                e2e_step()
            torch.cuda.synchronize()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
            barrier()
            torch.cuda.synchronize()
            for e0, e1 in ev:
                flush()
                e0.record(stream)
                e2e_step()
                e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            e2e_ms = max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in ev))
            e2e_diff = float((hy.double() - outs[args.mode].cpu().double()).norm()
                             / outs[args.mode].cpu().double().norm().clamp_min(1e-30))
            # the e2e leg's own bound: the same bytes as two plain copies at once (duplex PCIe)
            s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
            xs = lb.x[b0 * lb.in_img:b1 * lb.in_img]
            pcie = []
            for _ in range(3):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                s_in.wait_stream(stream)
                s_out.wait_stream(stream)
                with torch.cuda.stream(s_in):
                    xs.copy_(hx, non_blocking=True)
                with torch.cuda.stream(s_out):
                    hy.copy_(outs[args.mode], non_blocking=True)
                stream.wait_stream(s_in)
                stream.wait_stream(s_out)
                e1.record(stream)
                torch.cuda.synchronize()
                pcie.append(e0.elapsed_time(e1))
            pcie_ms = max_over_ranks(min(pcie))
        clocks = clk.summary()

        # ---- verification (untimed): all-gather the shards (NCCL), sampled images on rank 0
        full = {}
        for m in modes:
            full[m] = gather_shards(outs[m].to(cdev), N, lb.out_img) if world > 1 else outs[m]
        verified = None
        cross = {}
        if rank == 0:
            ref_m = full[args.mode]
            for m in modes:
                if m != args.mode:
                    cross[m] = float(torch.linalg.vector_norm((full[m] - ref_m).double())
                                     / torch.linalg.vector_norm(ref_m.double()))
            if not args.no_verify:
                imgs = sample_images(N)
                host = full[args.mode].cpu().numpy()
                got = {i: host[i * lb.out_img:(i + 1) * lb.out_img] for i in imgs}
                verified = verify_images(conv, c_logical, cfg_id, imgs, got)
                verified["pass"] = verified["max_rel_l2_vs_oracle"] <= TOL[args.mode]
                verified["gather"] = (f"{args.dist_backend} all-gather of variable-size image shards"
                                      if world > 1 else "single GPU")
        if rank == 0:
            total_flops = meas.flops(p, c_logical)
            roof = meas.roofline(p, c_logical, args.mode, hbm, bf16, n_img=n_local)
            hl = legs[args.mode]
            roof_obj = meas.roofline_entry(roof, hl["kern"], hbm)
            tf32_gemm = meas.tf32_gemm_tflops(local_rank)
            roof_obj.update({
                "traffic": ncu_traffic(args.workload, args.mode),
                "kernel_ms": round(hl["kern"], 4), "kernel_ms_median": round(hl["kern_med"], 4),
                "step_ms_median": round(hl["step_med"], 4), "steady_kernel_ms": round(steady_ms, 4),
                "frac_steady": meas.roofline_entry(roof, steady_ms, hbm)["frac"],
                "roofline_ms": round(roof["t_roof_s"] * 1e3, 4),
                "step_frac": round(roof["t_roof_s"] * 1e3 / hl["step"], 4),
                "peak_source": f"{peak_src}: bf16 {bf16} TFLOP/s /2 (tf32 rate)"
                               + (" /3 (3xTF32: three tf32 MMAs per MAC)" if args.mode == "3xtf32" else "")
                               + f"; HBM {hbm} GB/s",
                "tf32_gemm_tflops_measured": round(tf32_gemm, 1),
                "frac_vs_measured_tf32_gemm": round(roof["flops"] / (hl["kern"] * 1e-3) / 1e12 /
                                                    (tf32_gemm / (3 if args.mode == "3xtf32" else 1)), 4)
                if roof["bound"] == "tensor" and args.mode != "f16x2" else None,
                "algorithmic": f"{roof['flops'] / 1e9:.3f} GFLOP and {roof['bytes'] / 1e6:.1f} MB compulsory "
                               f"per launch ({n_local} images x 2*K*C*P*Q*R*S)"})
            bi = 4 * (n_local * lb.in_img + p.filter_elems())
            bo = 4 * n_local * lb.out_img
            others = {}
            for m in modes:
                if m == args.mode:
                    continue
                lg = legs[m]
                rm = meas.roofline(p, c_logical, m, hbm, bf16, n_img=n_local)
                others[f"{m}_mode"] = {
                    "mode": m, "value": round(total_flops / (lg["step"] * 1e-3) / 1e9, 1),
                    "ms_per_step": round(lg["step"], 4), "kernel_ms": round(lg["kern"], 4),
                    "kernel_ms_median": round(lg["kern_med"], 4),
                    "kernel_tflops": round(rm["flops"] / (lg["kern"] * 1e-3) / 1e12, 2),
                    "frac_of_peak": round(rm["t_roof_s"] * 1e3 / lg["kern"], 4),
                    "peak": f"{rm['peak_tflops']:.1f} TFLOP/s ({m})", "recipe": lg["plan"].recipe,
                    "rel_l2_vs_" + args.mode: float(f"{cross[m]:.3g}")}
            result = {
                "metric": METRIC,
                "value": round(total_flops / (hl["step"] * 1e-3) / 1e9, 1), "unit": "GFLOP/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(hl["step"], 4), "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None,
                "dtype": {"3xtf32": "f32 (3xtf32 tensor-core split, fp32 in/out)",
                          "tf32": "f32 in/out, tf32 tensor-core",
                          "f16x2": "f32 (scaled fp16 hi/lo tensor-core split, fp32 in/out)"}[args.mode],
                "data": "synthetic: seeded uniform[-1,1) by logical NCHW/KCRS index (BASELINE configs)",
                "config": run_config(args.workload, conv, c_logical, N),
                "run": {"mode": args.mode, "recipe": hl["plan"].recipe, "recipe_source": recipes[args.mode][1],
                        "images_per_gpu": n_local, "parallelism": f"dp{world} (img split)",
                        "l2": "flushed before every timed step (256 MiB write, then read back so the "
                              "write-back completes outside the timed region)",
                        "steady_state": f"{steady_n} back-to-back launches over {steady_sets} rotating sets"},
                "roofline": roof_obj,
                "e2e": {"value": round(total_flops / (e2e_ms * 1e-3) / 1e9, 1), "unit": "GFLOP/s",
                        "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo, "ms_per_step": round(e2e_ms, 3),
                        "matches_device_path": e2e_diff <= 1e-5, "rel_l2_vs_device_path": float(f"{e2e_diff:.3g}"),
                        "copy_bound_ms": round(pcie_ms, 3), "frac_of_copy_bound": round(pcie_ms / e2e_ms, 4),
                        "path": "ConvPlan.forward_host (C ABI conv_fwd_host): pinned host -> device -> pinned "
                                "host, chunked and overlapped"},
                "gpu_launches": args.steps * plan.launches,
                "clocks": clocks, "clocks_ok": meas.clocks_ok(clocks),
                **others,
                "verified": verified,
            }
        for m in modes:
            legs[m]["plan"].close()
        lb.release()
        del outs, full
        torch.cuda.empty_cache()

    # ---- per-layer metric (1 GPU)
    if world == 1 and args.layers != "none":
        names = (list(wl.ALL) if args.layers == "all" else
                 list(DEFAULT_LAYERS) if args.layers == "default" else args.layers.split(","))
        modes = args.layer_modes.split(",")
        recs = []
        for name in names:
            rec = measure_layer(ps, meas, name, args, flush, local_rank, hbm, bf16, modes)
            recs.append(rec)
            if args.jsonl:
                with open(args.jsonl, "a") as fh:
                    fh.write(json.dumps(rec) + "\n")
            print(f"# layer {name}: " + ", ".join(
                f"{m} step {r['step_ms'] * 1e3:.1f} us ({r['frac_step']:.2f}) steady {r['steady_ms'] * 1e3:.1f} us "
                f"({r['frac_steady']:.2f})" for m, r in rec["modes"].items()), file=sys.stderr, flush=True)
            torch.cuda.empty_cache()
        result["layers"] = recs
        result["layers_summary"] = layer_summary(recs, modes)
        if args.md:
            write_md(args.md, recs, modes, meas.peaks()[2])
    return result


def layer_summary(recs, modes):
    out = {}
    for m in modes:
        rows = [r["modes"][m] for r in recs if m in r["modes"]]
        if not rows:
            continue
        g = lambda k: math.exp(sum(math.log(r[k]) for r in rows) / len(rows))  # noqa: E731
        out[m] = {"layers": len(rows), "geomean_frac_step": round(g("frac_step"), 4),
                  "geomean_frac_steady": round(g("frac_steady"), 4),
                  "ge_0p6_step": sum(r["frac_step"] >= 0.6 for r in rows),
                  "ge_0p6_steady": sum(r["frac_steady"] >= 0.6 for r in rows),
                  "all_verified": all(r.get("verified", {}).get("pass", False) for r in rows),
                  "all_clocks_ok": all(r["clocks_ok"] for r in rows)}
    return out


def write_md(path, recs, modes, src):
    with open(path, "w") as fh:
        fh.write(f"# Per-layer conv fwd on 1 B200 (bench.py; peaks: {src}; tf32 = bf16/2, 3xtf32 = tf32/3, "
                 "f16x2 = bf16/3)\n\n")
        fh.write("step = repack + conv, one launch after an L2 flush; steady = back-to-back launches over "
                 "rotating input/output sets > 2x L2. frac = roofline time / measured time.\n\n")
        fh.write("| layer | mode | bound | roofline us | step us | kernel us | steady us | frac step | "
                 "frac steady | SM MHz | relL2 | CPU ref GFLOP/s | recipe |\n")
        fh.write("|---|---|---|---|---|---|---|---|---|---|---|---|---|\n")
        for r in recs:
            cpu = r.get("cpu_reference", {}).get("value", "")
            for m, x in r["modes"].items():
                fh.write(f"| {r['layer']} | {m} | {x['bound']} | {x['roofline_ms'] * 1e3:.1f} | "
                         f"{x['step_ms'] * 1e3:.1f} | {x['kernel_ms'] * 1e3:.1f} | {x['steady_ms'] * 1e3:.1f} | "
                         f"{x['frac_step']:.3f} | {x['frac_steady']:.3f} | {x['clocks'].get('sm_mhz')} | "
                         f"{x.get('verified', {}).get('max_rel_l2_vs_oracle', '')} | {cpu} | `{x['recipe']}` |\n")
        for m, s in layer_summary(recs, modes).items():
            fh.write(f"\n{m}: geomean frac {s['geomean_frac_step']:.3f} (step) / {s['geomean_frac_steady']:.3f} "
                     f"(steady) over {s['layers']} layers; >= 0.6: {s['ge_0p6_step']} (step) / "
                     f"{s['ge_0p6_steady']} (steady); verified {s['all_verified']}; clocks ok {s['all_clocks_ok']}\n")


def ncu_traffic(workload, mode):
    """dram bytes per launch of the conv kernel from the committed ncu capture, or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(f"{workload}/{mode}")
    except (OSError, ValueError):
        return None


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """The reference's CPU path (its own emitted driver) on the box's host cores, on the SAME
    configuration as the GPU arm (all N images). Loads nothing from paper_2002_02145_b200."""
    if rank != 0:
        return None
    wl = _workloads()
    conv, c_logical, cfg_id = wl.ALL[args.workload]
    leg = CpuLeg(args.workload, conv, c_logical, cfg_id).run(args.steps, args.warmup)
    v = leg["value"]
    return {
        "metric": METRIC, "value": v, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": leg["ms_per_rep"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "impl": "reference",
        "data": "synthetic: seeded uniform[-1,1) by logical NCHW/KCRS index (BASELINE configs)",
        "config": run_config(args.workload, conv, c_logical, Desc(conv).nImg),
        "run": {"step": "one pass of the reference driver over all images of the workload",
                "threads": leg["cores"]},
        "cpu_baseline": {k: leg[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cpu_model": leg["cpu_model"],
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg5")
    ap.add_argument("--mode", default="3xtf32", choices=["3xtf32", "tf32", "f16x2"])
    ap.add_argument("--no-f16x2", action="store_true", help="skip the f16x2 leg beside 3xTF32")
    ap.add_argument("--recipe", default=None, help="headline recipe (overrides the plan cache)")
    ap.add_argument("--no-headline", action="store_true", help="per-layer records only")
    ap.add_argument("--layers", default="default", help="default | all | none | comma list")
    ap.add_argument("--layer-modes", default="3xtf32,tf32")
    ap.add_argument("--layer-seconds", type=float, default=0.3, help="steady-state time per layer/mode")
    ap.add_argument("--jsonl", default=None, help="append per-layer records here")
    ap.add_argument("--md", default=None, help="write the per-layer table here")
    ap.add_argument("--tune-plans", type=int, default=0,
                    help="re-tune every timed (descriptor, mode) with the model's top-k and write the cache")
    ap.add_argument("--plans-out", default=None, help="plan cache written by --tune-plans")
    ap.add_argument("--rows", default=None, help="append the tuner's `ranked` rows here")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline / per-layer CPU legs")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: run the N>1 path with every rank on the visible GPU(s) (tests)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        res = run_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return

    import torch
    import torch.distributed as dist
    device = local_rank
    if world > 1:
        if args.dist_backend == "nccl":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:  # ranks may share a GPU (one process per rank, independent kernels)
            device = local_rank % torch.cuda.device_count()
            dist.init_process_group("gloo")
    res = run_ours(args, rank, world, device)
    if rank == 0:
        if not args.no_cpu and not args.no_headline:
            wl = _workloads()
            conv, c_logical, cfg_id = wl.ALL[args.workload]
            leg = CpuLeg(args.workload, conv, c_logical, cfg_id).run(reps=3, warmup=1)
            res["cpu_baseline"] = {k: leg[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")}
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
