"""Time arbitrary conv descriptors x recipes (kernel only, prepacked, L2 flushed).
  python tools/conv_times.py "conv:28,64,64,56,56,3,3,1,1,16,1,1,56,56" tf32 "gpu=bn:64" ...
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2002_02145_b200 as ps  # noqa: E402
from paper_2002_02145_b200.timing import L2Flush  # noqa: E402


def main():
    conv, mode = sys.argv[1], sys.argv[2]
    p = ps.ConvPreset.parse(conv)
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream()
    x = torch.empty(p.input_elems(), device=dev)
    w = torch.empty(p.filter_elems(), device=dev)
    y = torch.empty(p.output_elems(), device=dev)
    ps.fill_input(p, 1, x)
    ps.fill_filter(p, 2, w)
    flush = L2Flush(dev)
    for r in sys.argv[3:] or [None]:
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
        print(f"{conv} {mode} {ms * 1e3:8.1f} us {p.flops() / ms / 1e9:8.1f} TFLOP/s  {plan.recipe}",
              flush=True)
        if os.environ.get("CT_DIAG"):
            import time
            torch.cuda.synchronize()
            h0 = time.perf_counter()
            for _ in range(50):
                f()
            h1 = time.perf_counter()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(50):
                f()
            e1.record(st)
            torch.cuda.synchronize()
            print(f"   host {1e6 * (h1 - h0) / 50:.1f} us/call; back-to-back {e0.elapsed_time(e1) * 20:.1f} us/call")
        plan.close()


if __name__ == "__main__":
    main()
