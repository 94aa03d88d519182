import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, paper_2002_02145_b200 as ps
from tests.cases import ALL, seeds, with_images
for name, n in [("cfg5", 8), ("r50_l4_3x3_512_512", 16)]:
    conv, cl, cid = ALL[name]
    p = ps.ConvPreset.parse(with_images(conv, n)); sx, sw = seeds(cid)
    x = oracle.fill_input(p, sx, cl); w = oracle.fill_filter(p, sw, cl)
    ref64 = oracle.conv_f64(p, x, w)
    xd = torch.from_numpy(x.ravel()).cuda(); wd = torch.from_numpy(w.ravel()).cuda()
    for ch in [1, 2, 4, 8, 16, 32, 64, 10000]:
        yd = torch.empty(p.output_elems(), device='cuda')
        plan = ps.ConvPlan(p, mode="3xtf32", recipe=f"gpu=bn:128,ch:{ch}")
        plan.forward(xd, wd, yd); torch.cuda.synchronize()
        print(f"{name:22s} ch={ch:5d} relL2-vs-f64={oracle.rel_l2(yd.cpu().numpy(), ref64):.2e} {plan.recipe}")
