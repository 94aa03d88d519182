"""Layout probe: 1x1 conv with a single k-step, inspect the effective operand mapping."""
import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2002_02145_b200 as ps
import oracle

def run(csv, mode, recipe=None):
    p = ps.ConvPreset.parse(csv)
    x = oracle.fill_input(p, 5); w = oracle.fill_filter(p, 6)
    xd = torch.from_numpy(x.ravel()).cuda(); wd = torch.from_numpy(w.ravel()).cuda()
    yd = torch.full((p.output_elems(),), 777.0, device='cuda')
    plan = ps.ConvPlan(p, mode=mode, recipe=recipe)
    plan.forward(xd, wd, yd); torch.cuda.synchronize()
    y = yd.cpu().numpy()
    ref = oracle.conv(p, x, w).ravel()
    print(csv, mode, plan.recipe, "relL2", oracle.rel_l2(y, ref), "n777", int((y == 777).sum()), "nzero", int((y == 0).sum()), "of", y.size)
    return p, x, w, y, ref

for mode in ["tf32", "3xtf32"]:
    p, x, w, y, ref = run("conv:1,16,16,8,16,1,1,1,1,16", mode, "gpu=bn:16,box:16x8x1")
    X = x.reshape(128, 16); Y = y.reshape(128, 16); W = w.reshape(16, 16)
    Weff, res, rk, sv = np.linalg.lstsq(X.astype(np.float64), Y.astype(np.float64), rcond=None)
    print(" lstsq residual", res.sum() if res.size else None, "rank", rk)
    print(" Weff vs W", np.abs(Weff - W).max(), " vs W.T", np.abs(Weff - W.T).max())
    print(" Y[:2]", Y[:2, :6]); print(" R[:2]", (X @ W)[:2, :6])
    # row permutation check: for each GPU row find best matching ref row
    R = X @ W
    d = ((Y[:, None, :] - R[None, :, :]) ** 2).sum(-1)
    print(" best rows", d.argmin(1)[:32])
