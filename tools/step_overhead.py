"""Where does the single-launch step's overhead over the conv kernel go? (profiling tool)

For the small BASELINE layers, times after an L2 flush (CUDA events, median of 30):
  a  e0 | prepack | e1 | conv | e2   (bench.py's step = a0..a2, kernel = a1..a2)
  b  e0 | prepack | conv | e2        (no event between the two launches: PDL can overlap them)
  c  e0 | conv (prepacked) | e2      (conv alone)
  d  e0 | empty-ish torch kernel | e2 (the launch floor after the flush)
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_02145_b200 as ps  # noqa: E402
from paper_2002_02145_b200 import tune, workloads as wl  # noqa: E402
from paper_2002_02145_b200.timing import L2Flush  # noqa: E402

dev = torch.device("cuda", 0)
flush = L2Flush(dev)
st = torch.cuda.current_stream(dev)
reps = 30
names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3"]
for name in names:
    conv, c_log, cid = wl.ALL[name]
    p = ps.ConvPreset.parse(conv)
    x = torch.empty(p.input_elems(), device=dev)
    w = torch.empty(p.filter_elems(), device=dev)
    y = torch.empty(p.output_elems(), device=dev)
    ps.fill_input(p, 1, x, c_logical=c_log)
    ps.fill_filter(p, 2, w, c_logical=c_log)
    for mode in ("tf32", "3xtf32"):
        plan = ps.ConvPlan(p, mode=mode, device=0, recipe=tune.lookup(p, mode))
        plan.prepack(w, st)
        for _ in range(3):
            plan.forward(x, w, y, stream=st)
        res = {}
        for kind in "abcd":
            t01, t12, t02 = [], [], []
            for _ in range(reps):
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                flush()
                e[0].record(st)
                if kind == "a":
                    plan.prepack(w, st)
                    e[1].record(st)
                    plan.forward(x, None, y, stream=st, prepacked=True)
                elif kind == "b":
                    plan.prepack(w, st)
                    plan.forward(x, None, y, stream=st, prepacked=True)
                elif kind == "c":
                    plan.forward(x, None, y, stream=st, prepacked=True)
                else:
                    y[:4].zero_()
                e[2].record(st)
                torch.cuda.synchronize()
                t02.append(e[0].elapsed_time(e[2]) * 1e3)
                if kind == "a":
                    t01.append(e[0].elapsed_time(e[1]) * 1e3)
                    t12.append(e[1].elapsed_time(e[2]) * 1e3)
            res[kind] = statistics.median(t02)
            if kind == "a":
                res["a01"], res["a12"] = statistics.median(t01), statistics.median(t12)
        print(f"{name:5s} {mode:6s} a(step)={res['a']:6.1f} [prepack {res['a01']:5.1f} | conv {res['a12']:6.1f}]  "
              f"b(no mid event)={res['b']:6.1f}  c(conv only)={res['c']:6.1f}  d(launch floor)={res['d']:5.1f} us",
              flush=True)
        plan.close()
