"""Re-time the recipes recorded in a sweep file with the current library (A/B of kernel changes).
  python tools/ab_sweep.py profiles/r01_sweep.jsonl [--only cfg1,cfg2] [--modes tf32]
Select the library with PSCONV_LIB_NAME (tools/build_variant.sh builds variants). Kernel only,
prepacked filter, L2 flushed before every timed launch, mean of --steps launches.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

from paper_2002_02145_b200 import measure as bench  # noqa: E402
import paper_2002_02145_b200 as ps  # noqa: E402
from paper_2002_02145_b200.timing import L2Flush  # noqa: E402
from paper_2002_02145_b200.workloads import ALL, seeds  # noqa: E402


def time_it(fn, flush, steps, warm, stream):
    """Mean event time (ms) of fn with the L2 flushed before every launch."""
    import statistics
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for e0, e1 in ev:
        flush()
        e0.record(stream)
        fn()
        e1.record(stream)
    torch.cuda.synchronize()
    return statistics.mean(e0.elapsed_time(e1) for e0, e1 in ev)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sweep")
    ap.add_argument("--only", default=None)
    ap.add_argument("--modes", default="3xtf32,tf32")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--extra", default="", help="appended to every recipe's gpu clause, e.g. eg:2")
    args = ap.parse_args()
    only = set(args.only.split(",")) if args.only else None
    modes = set(args.modes.split(","))
    hbm, bf16, _ = bench.peaks()
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream()
    flush = L2Flush(dev)
    recs = []
    for line in open(args.sweep):
        if not line.strip():
            continue
        r = json.loads(line)
        if "modes" in r:  # bench.py per-layer records (one per layer, nested modes)
            for m, x in r["modes"].items():
                recs.append({"layer": r["layer"], "mode": m, "recipe": x["recipe"], "kernel_ms": x["kernel_ms"]})
        else:
            recs.append(r)
    fr = []
    for r in recs:
        if (only and r["layer"] not in only) or r["mode"] not in modes:
            continue
        conv, c_log, cid = ALL[r["layer"]]
        p = ps.ConvPreset.parse(conv)
        x = torch.empty(p.input_elems(), device=dev)
        w = torch.empty(p.filter_elems(), device=dev)
        y = torch.empty(p.output_elems(), device=dev)
        sx, sw = seeds(cid)
        ps.fill_input(p, sx, x, c_logical=c_log)
        ps.fill_filter(p, sw, w, c_logical=c_log)
        rid = r["recipe"] + ("," + args.extra if args.extra else "")
        plan = ps.ConvPlan(p, mode=r["mode"], recipe=rid)
        plan.prepack(w, st)
        ms = time_it(lambda: plan.forward(x, None, y, stream=st, prepacked=True), flush, args.steps, 3, st)
        peak = (bf16 / 3 if r["mode"] == "f16x2" else bf16 / 2 / (3 if r["mode"] == "3xtf32" else 1))
        t_roof = max(p.flops(c_log) / (peak * 1e12), bench.compulsory_bytes(p, c_log) / (hbm * 1e9)) * 1e3
        fr.append(t_roof / ms)
        print(f"{r['layer']:28s} {r['mode']:6s} {ms * 1e3:8.1f} us (was {r['kernel_ms'] * 1e3:8.1f})"
              f"  frac {t_roof / ms:.3f}  {plan.recipe}", flush=True)
        plan.close()
        del x, w, y
    if fr:
        import math
        print(f"geomean frac {math.exp(sum(map(math.log, fr)) / len(fr)):.4f} over {len(fr)}")


if __name__ == "__main__":
    main()
