"""Per-layer sweep: every BASELINE config + the ResNet-50 layer shapes, both modes, on cuda:0.

Same protocol as bench.py (CUDA events, L2 flushed before each timed step, warm-up first).
Writes one JSON record per (layer, mode) to --out and a markdown table to --md.
  python tools/sweep.py --out profiles/r01_sweep.jsonl --md profiles/r01_sweep.md
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2002_02145_b200 as ps  # noqa: E402
from paper_2002_02145_b200.timing import L2Flush  # noqa: E402
from paper_2002_02145_b200.workloads import ALL, seeds  # noqa: E402


def time_it(fn, flush, steps, warm, stream):
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
    ap.add_argument("--out", default="profiles/sweep.jsonl")
    ap.add_argument("--md", default=None)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only", default=None, help="comma list of workload names")
    ap.add_argument("--modes", default="3xtf32,tf32,f16x2")
    ap.add_argument("--recipe", default=None)
    ap.add_argument("--tune", type=int, default=0, help="time the model's top-k per layer")
    ap.add_argument("--rows", default=None, help="append tuner `ranked` rows here")
    args = ap.parse_args()
    hbm, bf16, src = bench.peaks()
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream()
    flush = L2Flush(dev)  # write + read 256 MiB (> 126 MB L2)
    names = args.only.split(",") if args.only else list(ALL)
    recs = []
    for name in names:
        conv, c_log, cid = ALL[name]
        p = ps.ConvPreset.parse(conv)
        sx, sw = seeds(cid)
        x = torch.empty(p.input_elems(), dtype=torch.float32, device=dev)
        w = torch.empty(p.filter_elems(), dtype=torch.float32, device=dev)
        y = torch.empty(p.output_elems(), dtype=torch.float32, device=dev)
        ps.fill_input(p, sx, x, c_logical=c_log)
        ps.fill_filter(p, sw, w, c_logical=c_log)
        flops = p.flops(c_log)
        bytes_c = bench.compulsory_bytes(p, c_log)
        for mode in args.modes.split(","):
            recipe = args.recipe
            if args.tune and recipe is None:
                from paper_2002_02145_b200.tune import autotune
                recipe, _ = autotune(p, mode, k=args.tune, c_logical=c_log, seeds=(sx, sw),
                                     report_path=args.rows)
            plan = ps.ConvPlan(p, mode=mode, recipe=recipe)
            step = time_it(lambda: plan.forward(x, w, y, stream=stream), flush, args.steps, args.warmup, stream)
            plan.prepack(w, stream)
            kern = time_it(lambda: plan.forward(x, None, y, stream=stream, prepacked=True), flush,
                           args.steps, args.warmup, stream)
            peak = (bf16 / 3 if mode == "f16x2" else bf16 / 2 / (3 if mode == "3xtf32" else 1))
            t_roof = max(flops / (peak * 1e12), bytes_c / (hbm * 1e9)) * 1e3
            rec = {"layer": name, "conv": conv, "mode": mode, "recipe": plan.recipe,
                   "gflop": round(flops / 1e9, 3), "mb_compulsory": round(bytes_c / 1e6, 1),
                   "bound": "tensor" if flops / (peak * 1e12) >= bytes_c / (hbm * 1e9) else "hbm",
                   "roofline_ms": round(t_roof, 4), "step_ms": round(step, 4), "kernel_ms": round(kern, 4),
                   "gflops_step": round(flops / step / 1e6, 1), "frac_step": round(t_roof / step, 4),
                   "frac_kernel": round(t_roof / kern, 4), "model_us": round(ps.model_us(p, plan.recipe, mode), 1)}
            recs.append(rec)
            print(json.dumps(rec), flush=True)
            plan.close()
        del x, w, y
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    with open(args.out, "w") as fh:
        for r in recs:
            fh.write(json.dumps(r) + "\n")
    if args.md:
        write_md(args.md, recs, src)


def write_md(path, recs, src):
    import math
    with open(path, "w") as fh:
        fh.write(f"# Per-layer sweep (1 B200, peaks: {src}; tf32 = bf16/2, 3xtf32 = tf32/3, f16x2 = bf16/3)\n\n")
        fh.write("| layer | mode | GFLOP | bound | roofline ms | step ms | kernel ms | GFLOP/s (step) | frac (step) | frac (kernel) | recipe |\n")
        fh.write("|---|---|---|---|---|---|---|---|---|---|---|\n")
        for r in recs:
            fh.write(f"| {r['layer']} | {r['mode']} | {r['gflop']} | {r['bound']} | {r['roofline_ms']} | "
                     f"{r['step_ms']} | {r['kernel_ms']} | {r['gflops_step']} | {r['frac_step']} | "
                     f"{r['frac_kernel']} | `{r['recipe']}` |\n")
        for mode in ("3xtf32", "tf32", "f16x2"):
            fr = [r["frac_step"] for r in recs if r["mode"] == mode]
            if fr:
                g = math.exp(sum(map(math.log, fr)) / len(fr))
                fh.write(f"\nGeomean roofline fraction (step), {mode}: {g:.3f} over {len(fr)} layers; "
                         f"layers >= 0.6: {sum(f >= 0.6 for f in fr)}/{len(fr)}\n")


def merge(main_path, part_path, md_path):
    """Replace the (layer, mode) records of main_path with those of part_path; rewrite the md."""
    recs = [json.loads(l) for l in open(main_path) if l.strip()]
    new = {(r["layer"], r["mode"]): r for r in (json.loads(l) for l in open(part_path) if l.strip())}
    recs = [new.pop((r["layer"], r["mode"]), r) for r in recs] + list(new.values())
    with open(main_path, "w") as fh:
        for r in recs:
            fh.write(json.dumps(r) + "\n")
    write_md(md_path, recs, bench.peaks()[2])


if __name__ == "__main__":
    if len(sys.argv) == 5 and sys.argv[1] == "--merge":  # sweep.py --merge main.jsonl part.jsonl main.md
        merge(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        main()
