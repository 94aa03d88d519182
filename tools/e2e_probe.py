"""Where does conv_fwd_host's time go? cfg5 through the host-buffer entry: full call,
prepacked filter, CPU enqueue time. python tools/e2e_probe.py [mode]"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2002_02145_b200 as ps  # noqa: E402
from paper_2002_02145_b200.workloads import ALL  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "3xtf32"
p = ps.ConvPreset.parse(ALL["cfg5"][0])
plan = ps.ConvPlan(p, mode=mode, device=0, recipe="gpu=bn:256,box:1x1x128,cl:1,ks:2,ch:36")
hx = torch.randn(p.input_elems()).pin_memory()
hw = torch.randn(p.filter_elems()).pin_memory()
hy = torch.empty(p.output_elems()).pin_memory()
st = torch.cuda.current_stream()


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        fn()
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        out.append((e0.elapsed_time(e1), (t1 - t0) * 1e3))
    return min(o[0] for o in out), min(o[1] for o in out)


print("full      gpu %.3f ms  enqueue %.3f ms" % timeit(lambda: plan.forward_host(hx, hw, hy, stream=st)))
dw = hw.cuda()
plan.prepack(dw, st)
print("prepacked gpu %.3f ms  enqueue %.3f ms" % timeit(lambda: plan.forward_host(hx, None, hy, stream=st,
                                                                                  prepacked=True)))
dx = torch.empty(p.input_elems(), device="cuda")
dy = torch.empty(p.output_elems(), device="cuda")
print("device    gpu %.3f ms  enqueue %.3f ms" % timeit(lambda: plan.forward(dx, None, dy, stream=st,
                                                                             prepacked=True)))
