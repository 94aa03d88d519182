import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, paper_2002_02145_b200 as ps
from tests.cases import ALL, seeds, with_images
for name, n in [("cfg5", 8), ("r50_l4_3x3_512_512", 16), ("r50_l4_1x1_2048_512", 16), ("cfg1", 2)]:
    conv, cl, cid = ALL[name]
    p = ps.ConvPreset.parse(with_images(conv, n)); sx, sw = seeds(cid)
    x = oracle.fill_input(p, sx, cl); w = oracle.fill_filter(p, sw, cl)
    ref32 = oracle.conv(p, x, w); ref64 = oracle.conv_f64(p, x, w)
    out = {}
    for mode in ["3xtf32", "tf32"]:
        xd = torch.from_numpy(x.ravel()).cuda(); wd = torch.from_numpy(w.ravel()).cuda()
        yd = torch.empty(p.output_elems(), device='cuda')
        ps.ConvPlan(p, mode=mode).forward(xd, wd, yd); torch.cuda.synchronize()
        out[mode] = yd.cpu().numpy()
    print(f"{name:24s} CRS={p.nIfm*p.kh*p.kw:5d} oracle32-vs-f64={oracle.rel_l2(ref32, ref64):.2e} "
          f"gpu3x-vs-f64={oracle.rel_l2(out['3xtf32'], ref64):.2e} gpu3x-vs-oracle32={oracle.rel_l2(out['3xtf32'], ref32):.2e} "
          f"gputf32-vs-f64={oracle.rel_l2(out['tf32'], ref64):.2e}")
