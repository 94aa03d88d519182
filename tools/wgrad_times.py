"""Backward-weight (conv_bwd_weight) timings on ResNet-50 stride-1 layer shapes: the whole call
(X transpose, dY -> filter layout, role-swapped conv with split-K, dW layout), L2 flushed.
  python tools/wgrad_times.py [mode ...]"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2002_02145_b200 as ps  # noqa: E402
from paper_2002_02145_b200.timing import L2Flush  # noqa: E402
from paper_2002_02145_b200.workloads import ALL  # noqa: E402

LAYERS = ["cfg1", "r50_l1_3x3_64_64", "r50_l2_3x3_128_128", "r50_l3_3x3_256_256", "r50_l4_3x3_512_512",
          "r50_l3_1x1_1024_256", "cfg5"]


def main():
    modes = sys.argv[1:] or ["3xtf32", "tf32"]
    dev = torch.device("cuda:0")
    flush = L2Flush(dev)
    for name in LAYERS:
        conv = ALL[name][0]
        p = ps.ConvPreset.parse(conv)
        if p.nImg % 16:
            continue
        x = torch.rand(p.input_elems(), device=dev) * 2 - 1
        dy = torch.rand(p.output_elems(), device=dev) * 2 - 1
        dw = torch.empty(p.filter_elems(), device=dev)
        for mode in modes:
            plan = ps.WgradPlan(p, mode=mode)
            for _ in range(2):
                plan.forward(x, dy, dw)
            ts = []
            for _ in range(5):
                flush()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                plan.forward(x, dy, dw)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            print(json.dumps({"layer": name, "mode": mode, "ms": round(ms, 4),
                              "tflops": round(p.flops() / ms / 1e9, 1), "recipe": plan.recipe}), flush=True)
            plan.close()
        del x, dy, dw
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
