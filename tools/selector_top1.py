"""Selector quality: the closed-form model's own top-1 recipe (select_topk, no tuning) timed against
the plan cache's measured best on every bench workload and mode (the stem with the caller's
assertion of 3 real input channels, select_topk(c_logical=3)), interleaved on one box
(prepacked filter, L2 flushed, median of 7).  python tools/selector_top1.py > profiles/r02_selector_top1.md"""
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2002_02145_b200 as ps  # noqa: E402
from paper_2002_02145_b200 import tune, workloads  # noqa: E402
from paper_2002_02145_b200.timing import L2Flush  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream(dev)
    flush = L2Flush(dev)
    print("# Selector model top-1 vs the measured-best cached plan (1 B200, same box, interleaved)\n")
    print("| layer | mode | model top-1 us | cached best us | ratio | model top-1 recipe | cached recipe |")
    print("|---|---|---|---|---|---|---|")
    ratios = {"3xtf32": [], "tf32": []}
    for name, (conv, c_log, cid) in workloads.ALL.items():
        p = ps.ConvPreset.parse(conv)
        x = torch.empty(p.input_elems(), dtype=torch.float32, device=dev)
        w = torch.empty(p.filter_elems(), dtype=torch.float32, device=dev)
        y = torch.empty(p.output_elems(), dtype=torch.float32, device=dev)
        sx, sw = workloads.seeds(cid)
        ps.fill_input(p, sx, x, c_logical=c_log)
        ps.fill_filter(p, sw, w, c_logical=c_log)
        for mode in ("3xtf32", "tf32"):
            top = ps.select_topk(p, mode, 1, c_logical=c_log if c_log < p.nIfm else 0)[0][0]
            best = tune.lookup(p, mode) or top
            plans = []
            for rid in (top, best):
                pl = ps.ConvPlan(p, mode=mode, device=0, recipe=rid)
                pl.prepack(w, st)
                for _ in range(2):
                    pl.forward(x, None, y, stream=st, prepacked=True)
                plans.append((pl, []))
            for _ in range(7):
                for pl, ts in plans:
                    flush()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    pl.forward(x, None, y, stream=st, prepacked=True)
                    e1.record(st)
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e3)
            t_top, t_best = (statistics.median(ts) for _, ts in plans)
            recs = [pl.recipe.split("gpu=")[1] for pl, _ in plans]
            for pl, _ in plans:
                pl.close()
            ratios[mode].append(t_top / t_best)
            print(f"| {name} | {mode} | {t_top:.1f} | {t_best:.1f} | {t_top / t_best:.3f} | `{recs[0]}` | `{recs[1]}` |",
                  flush=True)
        del x, w, y
    print()
    for mode, r in ratios.items():
        g = math.exp(sum(math.log(v) for v in r) / len(r))
        print(f"{mode}: geomean ratio {g:.3f}; within 1.05x of the cached best on {sum(v <= 1.05 for v in r)} of {len(r)}; "
              f"within 1.10x on {sum(v <= 1.10 for v in r)}; worst {max(r):.2f}x")


if __name__ == "__main__":
    main()
