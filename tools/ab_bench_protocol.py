"""A/B of recipes under bench.py's own per-layer protocol (LayerBench.single: step = repack + conv
after an L2 flush, queued back to back; then the conv-only pass) on one box, alternating A and B
three times.  python tools/ab_bench_protocol.py LAYER MODE RECIPE_A RECIPE_B [...]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2002_02145_b200 as ps  # noqa: E402
from paper_2002_02145_b200 import measure as meas, workloads  # noqa: E402
from paper_2002_02145_b200.timing import L2Flush  # noqa: E402


def main():
    name, mode, recipes = sys.argv[1], sys.argv[2], sys.argv[3:]
    conv, c_log, cid = workloads.ALL[name]
    p = ps.ConvPreset.parse(conv)
    lb = meas.LayerBench(ps, p, c_log, workloads.seeds(cid), 0)
    flush = L2Flush(torch.device("cuda:0"))
    res = {r: ([], []) for r in recipes}
    for _ in range(3):
        for r in recipes:
            plan = ps.ConvPlan(p, mode=mode, device=0, recipe=r)
            step, kern = lb.single(plan, flush, 20, 5)
            res[r][0].append(statistics.mean(step) * 1e3)
            res[r][1].append(statistics.mean(kern) * 1e3)
            plan.close()
    for r in recipes:
        s, k = res[r]
        print(f"{name} {mode} step {statistics.median(s):7.1f} us (runs {' '.join(f'{v:.1f}' for v in s)})  "
              f"kernel {statistics.median(k):7.1f} us  {r.split('gpu=')[1]}", flush=True)


if __name__ == "__main__":
    main()
