"""Measured training data for the pairwise ranker: for every BASELINE
and ResNet-50 shape and both modes, the cost model's top-k candidates are timed on the GPU
(kernel only, prepacked filter, L2 flushed, median of 5) next to their model statistics.
  python tools/collect_ranker_data.py --k 16 --out profiles/r01_ranker_data.jsonl"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2002_02145_b200 as ps  # noqa: E402
from paper_2002_02145_b200.timing import L2Flush  # noqa: E402
from paper_2002_02145_b200.workloads import ALL, seeds  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=16)
    ap.add_argument("--out", default="profiles/r01_ranker_data.jsonl")
    ap.add_argument("--only", default=None)
    ap.add_argument("--modes", default="3xtf32,tf32,f16x2")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream()
    flush = L2Flush(dev)
    names = args.only.split(",") if args.only else list(ALL)
    with open(args.out, "w") as fo:
        for name in names:
            conv, c_log, cid = ALL[name]
            p = ps.ConvPreset.parse(conv)
            sx, sw = seeds(cid)
            x = torch.empty(p.input_elems(), device=dev)
            w = torch.empty(p.filter_elems(), device=dev)
            y = torch.empty(p.output_elems(), device=dev)
            ps.fill_input(p, sx, x, c_logical=c_log)
            ps.fill_filter(p, sw, w, c_logical=c_log)
            for mode in args.modes.split(","):
                for rid, mus in ps.select_topk(p, mode, k=args.k):
                    plan = ps.ConvPlan(p, mode=mode, recipe=rid)
                    plan.prepack(w, st)
                    f = lambda: plan.forward(x, None, y, stream=st, prepacked=True)  # noqa: E731
                    f()
                    f()
                    ts = []
                    for _ in range(5):
                        flush()
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(st)
                        f()
                        e1.record(st)
                        torch.cuda.synchronize()
                        ts.append(e0.elapsed_time(e1) * 1e3)
                    rec = {"layer": name, "mode": mode, "recipe": plan.recipe, "model_us": round(mus, 2),
                           "stats": [round(v, 4) for v in ps.model_stats(p, rid, mode)],
                           "measured_us": round(statistics.median(ts), 2)}
                    fo.write(json.dumps(rec) + "\n")
                    fo.flush()
                    plan.close()
            print(name, flush=True)


if __name__ == "__main__":
    main()
