"""The conv work of one ResNet-50 training step at N = 256 on this framework: all 53 forward
convolutions, then the backward pass in reverse layer order -- backward data (dX; not for the
stem, whose input is the image) and backward weight (dW) for every conv -- back to back on one
stream (PDL-chained launches; buffers per distinct shape, reused by its repeats; L2 flushed once
before each pass). Forward recipes from the committed plan cache, backward plans from the
selectors. Reports ms, TFLOP/s and the sum of per-conv rooflines per pass.
  python tools/resnet50_train_pass.py [modes...]        (default: tf32 3xtf32)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import paper_2002_02145_b200 as ps  # noqa: E402
from paper_2002_02145_b200 import measure, tune  # noqa: E402
from paper_2002_02145_b200.timing import L2Flush  # noqa: E402
from paper_2002_02145_b200.workloads import R50, seeds  # noqa: E402
from resnet50_pass import COUNT  # noqa: E402


def main():
    modes = sys.argv[1:] or ["tf32", "3xtf32"]
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream()
    flush = L2Flush(dev)
    hbm, bf16, _ = measure.peaks()
    for mode in modes:
        layers = []
        for name, (conv, c_log, cid) in R50.items():
            p = ps.ConvPreset.parse(conv)
            x = torch.empty(p.input_elems(), device=dev)
            w = torch.empty(p.filter_elems(), device=dev)
            y = torch.empty(p.output_elems(), device=dev)
            sx, sw = seeds(cid)
            ps.fill_input(p, sx, x, c_logical=c_log)
            ps.fill_filter(p, sw, w, c_logical=c_log)
            dy = torch.rand(p.output_elems(), device=dev) - 0.5
            dx = torch.empty(p.input_elems(), device=dev) if name != "r50_stem" else None
            dw = torch.empty(p.filter_elems(), device=dev)
            fwd = ps.ConvPlan(p, mode=mode, recipe=tune.lookup(p, mode))
            fwd.prepack(w)
            bwd = ps.ConvPlan(p, mode=mode, bwd_data=True) if dx is not None else None
            if bwd is not None:
                bwd.prepack(w)
            wg = ps.WgradPlan(p, mode=mode, c_logical=c_log)  # (the stem: tap-folded, 3 channels)
            roof = measure.roofline(p, c_log, mode, hbm, bf16)
            layers.append(dict(name=name, p=p, x=x, w=w, y=y, dy=dy, dx=dx, dw=dw, fwd=fwd, bwd=bwd, wg=wg,
                               flops=p.flops(c_log), roof_ms=roof["t_roof_s"] * 1e3, c_log=c_log))

        def fwd_pass():
            for L in layers:
                for _ in range(COUNT[L["name"]]):
                    L["fwd"].forward(L["x"], None, L["y"], stream=st, prepacked=True)

        def dgrad_pass():
            for L in reversed(layers):
                if L["bwd"] is not None:
                    for _ in range(COUNT[L["name"]]):
                        L["bwd"].forward(L["dy"], None, L["dx"], stream=st, prepacked=True)

        def wgrad_pass():
            for L in reversed(layers):
                for _ in range(COUNT[L["name"]]):
                    L["wg"].forward(L["x"], L["dy"], L["dw"], stream=st)

        def timed(fn, reps=3):
            fn()
            torch.cuda.synchronize()
            ts = []
            for _ in range(reps):
                flush()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                fn()
                e1.record(st)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            return min(ts)

        res = {"mode": mode, "n": 256, "convs": 53}
        for key, fn, sel in (("forward", fwd_pass, lambda L: True), ("backward_data", dgrad_pass,
                                                                     lambda L: L["bwd"] is not None),
                             ("backward_weight", wgrad_pass, lambda L: True)):
            ms = timed(fn)
            fl = sum(COUNT[L["name"]] * L["flops"] for L in layers if sel(L))
            rf = sum(COUNT[L["name"]] * L["roof_ms"] for L in layers if sel(L))
            res[key] = {"ms": round(ms, 3), "tflops": round(fl / ms / 1e9, 1), "sum_roofline_ms": round(rf, 3),
                        "frac_of_summed_roofline": round(rf / ms, 3)}
        res["step_conv_ms"] = round(sum(res[k]["ms"] for k in ("forward", "backward_data", "backward_weight")), 3)
        print(json.dumps(res), flush=True)
        for L in layers:
            for k in ("fwd", "bwd", "wg"):
                if L[k] is not None:
                    L[k].close()
        del layers
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
