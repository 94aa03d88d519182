"""Back-to-back per-call time of direct forward() calls vs CUDA-graph replays (ConvPlan.graph)
for the small BASELINE layers and a few ResNet-50 layers (prepacked filter, tuned recipes from
the committed sweep; no L2 flush: a serving loop over resident buffers).
  python tools/graph_times.py [profiles/r01_sweep.jsonl]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2002_02145_b200 as ps  # noqa: E402
from paper_2002_02145_b200.workloads import ALL, seeds  # noqa: E402

LAYERS = ["cfg1", "cfg2", "cfg3", "r50_l3_3x3_256_256", "r50_l4_1x1_2048_512"]


def per_call(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    sweep = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r01_sweep.jsonl")
    recs = {(r["layer"], r["mode"]): r for r in map(json.loads, open(sweep))}
    dev = torch.device("cuda:0")
    for name in LAYERS:
        conv, c_log, cid = ALL[name]
        p = ps.ConvPreset.parse(conv)
        x = torch.empty(p.input_elems(), device=dev)
        w = torch.empty(p.filter_elems(), device=dev)
        y = torch.empty(p.output_elems(), device=dev)
        sx, sw = seeds(cid)
        ps.fill_input(p, sx, x, c_logical=c_log)
        ps.fill_filter(p, sw, w, c_logical=c_log)
        for mode in ("tf32", "3xtf32"):
            plan = ps.ConvPlan(p, mode=mode, recipe=recs[(name, mode)]["recipe"])
            plan.prepack(w)
            direct = per_call(lambda: plan.forward(x, None, y, prepacked=True))
            g = plan.graph(x, None, y)
            graphed = per_call(g.replay)
            print(json.dumps({"layer": name, "mode": mode, "direct_us": round(direct, 2),
                              "graph_us": round(graphed, 2), "recipe": plan.recipe}), flush=True)
            plan.close()


if __name__ == "__main__":
    main()
