"""All 53 convolutions of a ResNet-50 forward pass at N=256 (BASELINE.json configs[3]) run back
to back on one stream -- direct PDL-chained calls and one CUDA graph of the 53 launches -- with
the per-layer recipes of a sweep file (prepacked filters; buffers per distinct shape, reused by
its repeats; the L2 is flushed once before the pass, not between layers, as in a real network).
Reports total ms, TFLOP/s and the fraction of the summed per-layer rooflines.
  python tools/resnet50_pass.py [profiles/r01_sweep.jsonl] [modes...]
Mode "faithful" takes, per layer, the faster of 3xtf32 / f16x2 in the sweep file."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2002_02145_b200 as ps  # noqa: E402
from paper_2002_02145_b200.timing import L2Flush  # noqa: E402
from paper_2002_02145_b200.workloads import R50, seeds  # noqa: E402

# multiplicity of each distinct shape in ResNet-50 (3 / 4 / 6 / 3 bottleneck blocks)
COUNT = {
    "r50_stem": 1, "r50_l1_1x1_64_64": 1, "r50_l1_3x3_64_64": 3, "r50_l1_1x1_64_256": 4,
    "r50_l1_1x1_256_64": 2, "r50_l2_1x1_256_128": 1, "r50_l2_3x3s2_128_128": 1,
    "r50_l2_1x1_128_512": 4, "r50_l2_ds_1x1s2_256_512": 1, "r50_l2_1x1_512_128": 3,
    "r50_l2_3x3_128_128": 3, "r50_l3_1x1_512_256": 1, "r50_l3_3x3s2_256_256": 1,
    "r50_l3_1x1_256_1024": 6, "r50_l3_ds_1x1s2_512_1024": 1, "r50_l3_1x1_1024_256": 5,
    "r50_l3_3x3_256_256": 5, "r50_l4_1x1_1024_512": 1, "r50_l4_3x3s2_512_512": 1,
    "r50_l4_1x1_512_2048": 3, "r50_l4_ds_1x1s2_1024_2048": 1, "r50_l4_1x1_2048_512": 2,
    "r50_l4_3x3_512_512": 2,
}
assert sum(COUNT.values()) == 53 and set(COUNT) == set(R50)


def main():
    sweep = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r01_sweep.jsonl")
    modes = sys.argv[2:] or ["tf32", "3xtf32", "faithful"]
    recs = {}
    for r in map(json.loads, open(sweep)):
        if "modes" in r:  # r02 sweep rows: one per layer with a "modes" map
            for m, v in r["modes"].items():
                recs[(r["layer"], m)] = {**v, "mode": m}
        else:             # r01 rows: one per (layer, mode)
            recs[(r["layer"], r["mode"])] = r
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream()
    flush = L2Flush(dev)
    for mode in modes:
        plans, bufs, flops, roof = [], [], 0.0, 0.0
        for name, (conv, c_log, cid) in R50.items():
            if mode == "faithful":
                a, b = recs[(name, "3xtf32")], recs[(name, "f16x2")]
                r = a if a["step_ms"] <= b["step_ms"] else b
            else:
                r = recs[(name, mode)]
            p = ps.ConvPreset.parse(conv)
            x = torch.empty(p.input_elems(), device=dev)
            w = torch.empty(p.filter_elems(), device=dev)
            y = torch.empty(p.output_elems(), device=dev)
            sx, sw = seeds(cid)
            ps.fill_input(p, sx, x, c_logical=c_log)
            ps.fill_filter(p, sw, w, c_logical=c_log)
            plan = ps.ConvPlan(p, mode=r["mode"], recipe=r["recipe"])
            plan.prepack(w)
            plans.append((name, plan))
            bufs.append((x, y))
            flops += COUNT[name] * p.flops(c_log)
            roof += COUNT[name] * r["roofline_ms"]

        def run_pass():
            for (name, plan), (x, y) in zip(plans, bufs):
                for _ in range(COUNT[name]):
                    plan.forward(x, None, y, stream=st, prepacked=True)

        def timed(fn, reps=5):
            ts = []
            for _ in range(reps):
                flush()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                fn()
                e1.record(st)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            return min(ts)

        run_pass()
        torch.cuda.synchronize()
        direct = timed(run_pass)
        side = torch.cuda.Stream(dev)
        g = torch.cuda.CUDAGraph()
        side.wait_stream(st)
        with torch.cuda.graph(g, stream=side):
            for (name, plan), (x, y) in zip(plans, bufs):
                for _ in range(COUNT[name]):
                    plan.forward(x, None, y, stream=side, prepacked=True)
        graphed = timed(g.replay)
        print(json.dumps({"mode": mode, "convs": 53, "gflop": round(flops / 1e9, 1),
                          "direct_ms": round(direct, 3), "graph_ms": round(graphed, 3),
                          "tflops": round(flops / min(direct, graphed) / 1e9, 1),
                          "sum_roofline_ms": round(roof, 3),
                          "frac_of_summed_roofline": round(roof / min(direct, graphed), 4)}), flush=True)
        del g, plans, bufs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
