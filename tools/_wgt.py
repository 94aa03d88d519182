"""Backward-weight timing of one layer for a list of recipes ('-' = selector); profiling helper.
    PSCONV_DEBUG=0|1|2|3 python tools/_wgt.py conv:... tf32|3xtf32 - gpu=..."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_02145_b200 as ps  # noqa: E402
from paper_2002_02145_b200.timing import L2Flush  # noqa: E402

conv, mode = sys.argv[1], sys.argv[2]
p = ps.ConvPreset.parse(conv)
x = torch.rand(p.input_elems(), device="cuda") - 0.5
dy = torch.rand(p.output_elems(), device="cuda") - 0.5
dw = torch.empty(p.filter_elems(), device="cuda")
fl = L2Flush(torch.device("cuda"))
for r in sys.argv[3:]:
    try:
        plan = ps.WgradPlan(p, mode=mode, recipe=None if r == "-" else r)
    except ps.Error as e:
        print(f"{r}: {e}")
        continue
    plan.forward(x, dy, dw)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        fl()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.forward(x, dy, dw)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"dbg={os.environ.get('PSCONV_DEBUG', '0')} {conv} {mode} {statistics.median(ts) * 1e3:9.1f} us  {plan.recipe}",
          flush=True)
