import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import paper_2002_02145_b200 as ps
conv, mode = sys.argv[1], sys.argv[2]
rec = sys.argv[3] if len(sys.argv) > 3 else None
p = ps.ConvPreset.parse(conv)
x = torch.rand(p.input_elems(), device="cuda") - 0.5
dy = torch.rand(p.output_elems(), device="cuda") - 0.5
dw = torch.zeros(p.filter_elems(), device="cuda")
plan = ps.WgradPlan(p, mode=mode, recipe=rec)
print(plan.recipe, flush=True)
plan.forward(x, dy, dw)
torch.cuda.synchronize()
print("ok", dw.abs().sum().item())
