"""Backward-data (ConvPlan(bwd_data=True)) timings on the ResNet-50 layer shapes at N = 256: prepacked
filter, L2 flushed before each call, CUDA events, median of 5; roofline = the forward layer's
(same FLOPs; dY + W + dX bytes).
  python tools/dgrad_times.py [mode ...]"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2002_02145_b200 as ps  # noqa: E402
from paper_2002_02145_b200 import measure  # noqa: E402
from paper_2002_02145_b200.timing import L2Flush  # noqa: E402
from paper_2002_02145_b200.workloads import R50  # noqa: E402


def main():
    modes = sys.argv[1:] or ["tf32", "3xtf32"]
    dev = torch.device("cuda:0")
    flush = L2Flush(dev)
    hbm, bf16, _ = measure.peaks()
    for name, (conv, c_log, _) in R50.items():
        if name == "r50_stem":
            continue
        p = ps.ConvPreset.parse(conv)
        dy = torch.rand(p.output_elems(), device=dev) - 0.5
        w = torch.rand(p.filter_elems(), device=dev) - 0.5
        dx = torch.empty(p.input_elems(), device=dev)
        flops = measure.flops(p)
        nbytes = 4 * (p.input_elems() + p.output_elems() + p.filter_elems())
        for mode in modes:
            plan = ps.ConvPlan(p, mode=mode, bwd_data=True)
            plan.prepack(w)
            for _ in range(2):
                plan.forward(dy, None, dx, prepacked=True)
            ts = []
            for _ in range(5):
                flush()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                plan.forward(dy, None, dx, prepacked=True)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            roof = max(flops / (measure.mode_peak_tflops(mode, bf16) * 1e12), nbytes / (hbm * 1e9)) * 1e3
            print(json.dumps({"layer": name, "mode": mode, "ms": round(ms, 4), "roofline_ms": round(roof, 4),
                              "frac": round(roof / ms, 3), "launches": plan.launches,
                              "recipe": plan.recipe[:160]}), flush=True)
            plan.close()
        del dy, w, dx
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
