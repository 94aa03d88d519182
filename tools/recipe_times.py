"""Time a list of recipes for one workload (kernel only, prepacked filter, L2 flushed).
  python tools/recipe_times.py cfg5 3xtf32 "gpu=bn:256,ch:16" "gpu=bn:128,ch:16" ...
  python tools/recipe_times.py cfg5 3xtf32 --topk 8     # the selector's top-k
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2002_02145_b200 import measure as bench  # noqa: E402
import paper_2002_02145_b200 as ps  # noqa: E402
from paper_2002_02145_b200.timing import L2Flush  # noqa: E402
from paper_2002_02145_b200.workloads import ALL, seeds  # noqa: E402


def main():
    name, mode = sys.argv[1], sys.argv[2]
    recipes = sys.argv[3:]
    conv, c_log, cid = ALL[name]
    p = ps.ConvPreset.parse(conv)
    if recipes and recipes[0] == "--topk":
        recipes = [r for r, _ in ps.select_topk(p, mode, int(recipes[1]))]
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream()
    x = torch.empty(p.input_elems(), device=dev)
    w = torch.empty(p.filter_elems(), device=dev)
    y = torch.empty(p.output_elems(), device=dev)
    sx, sw = seeds(cid)
    ps.fill_input(p, sx, x, c_logical=c_log)
    ps.fill_filter(p, sw, w, c_logical=c_log)
    flush = L2Flush(dev)
    hbm, bf16, _ = bench.peaks()
    peak = (bf16 / 3 if mode == "f16x2" else bf16 / 2 / (3 if mode == "3xtf32" else 1))
    flops = p.flops(c_log)
    t_roof = max(flops / (peak * 1e12), bench.compulsory_bytes(p, c_log) / (hbm * 1e9)) * 1e3
    for r in recipes:
        plan = ps.ConvPlan(p, mode=mode, recipe=r)
        plan.prepack(w, st)
        f = lambda: plan.forward(x, None, y, stream=st, prepacked=True)  # noqa: E731
        for _ in range(3):
            f()
        ts = []
        for _ in range(10):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            f()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        print(f"{name} {mode} {ms:8.4f} ms  frac={t_roof / ms:.3f}  model={ps.model_us(p, plan.recipe, mode):8.1f}us  {plan.recipe}",
              flush=True)
        plan.close()


if __name__ == "__main__":
    main()
