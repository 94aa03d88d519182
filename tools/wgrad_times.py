"""Backward-weight (conv_bwd_weight) timings on ResNet-50 layer shapes at N = 256: the whole call
(pixel-major wgrad kernel + split reduction), L2 flushed before each call, CUDA events, median of 5;
roofline = max(FLOPs at the mode's tensor peak, (X + dY + dW) bytes at the HBM peak).
  python tools/wgrad_times.py [mode ...]"""
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
from paper_2002_02145_b200.workloads import ALL  # noqa: E402

LAYERS = ["cfg1", "r50_stem", "r50_l1_1x1_64_64", "r50_l1_3x3_64_64", "r50_l1_1x1_64_256", "r50_l1_1x1_256_64",
          "r50_l2_3x3s2_128_128", "r50_l2_3x3_128_128", "r50_l2_ds_1x1s2_256_512", "r50_l3_3x3_256_256",
          "r50_l3_1x1_1024_256", "r50_l4_3x3s2_512_512", "r50_l4_3x3_512_512", "r50_l4_1x1_2048_512", "cfg5"]


def main():
    modes = sys.argv[1:] or ["3xtf32", "tf32"]
    dev = torch.device("cuda:0")
    flush = L2Flush(dev)
    hbm, bf16, _ = measure.peaks()
    for name in LAYERS:
        conv, c_log, _ = ALL[name]
        p = ps.ConvPreset.parse(conv)
        x = torch.rand(p.input_elems(), device=dev) * 2 - 1
        dy = torch.rand(p.output_elems(), device=dev) * 2 - 1
        dw = torch.empty(p.filter_elems(), device=dev)
        flops = measure.flops(p)
        nbytes = 4 * (p.input_elems() + p.output_elems() + p.filter_elems())
        for mode in modes:
            plan = ps.WgradPlan(p, mode=mode, c_logical=c_log)
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
            roof = max(flops / (measure.mode_peak_tflops(mode, bf16) * 1e12), nbytes / (hbm * 1e9)) * 1e3
            print(json.dumps({"layer": name, "mode": mode, "ms": round(ms, 4),
                              "tflops": round(flops / ms / 1e9, 1), "roofline_ms": round(roof, 4),
                              "frac": round(roof / ms, 3), "recipe": plan.recipe}), flush=True)
            plan.close()
        del x, dy, dw
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
