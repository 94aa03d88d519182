"""Per-layer ncu metrics (north star: tensor-pipe utilisation and achieved HBM bandwidth for each
layer): runs every (layer, mode) of a sweep file once with its tuned recipe (prepacked filter),
in order, so that one ncu session can attribute the conv kernel launches to layers.

  ncu --metrics <M> --clock-control none -k regex:"conv_(fwd|pp)_sm100" --csv \\
      --log-file gpurun_out/ncu_layers.csv python tools/ncu_layers.py run profiles/r02_sweep.jsonl
  python tools/ncu_layers.py table profiles/r02_sweep.jsonl gpurun_out/ncu_layers.csv > profiles/r02_ncu_layers.md
(M: see METRICS; cold caches and serialised launches, so absolute times run above the bench's)
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
           "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_sectors_srcunit_tex_op_read.sum"]


def records(sweep):
    """(layer, mode) records of a sweep file: r01 rows are per (layer, mode); r02 rows per layer
    with a "modes" map."""
    out = []
    for r in map(json.loads, open(sweep)):
        if "modes" in r:
            for mode, m in r["modes"].items():
                out.append({"layer": r["layer"], "mode": mode, "recipe": m["recipe"],
                            "mb_compulsory": r["mb_compulsory"]})
        else:
            out.append(r)
    return out


def run(sweep):
    import torch
    import paper_2002_02145_b200 as ps
    from paper_2002_02145_b200.workloads import ALL, seeds
    dev = torch.device("cuda:0")
    for r in records(sweep):
        conv, c_log, cid = ALL[r["layer"]]
        p = ps.ConvPreset.parse(conv)
        x = torch.empty(p.input_elems(), device=dev)
        w = torch.empty(p.filter_elems(), device=dev)
        y = torch.empty(p.output_elems(), device=dev)
        sx, sw = seeds(cid)
        ps.fill_input(p, sx, x, c_logical=c_log)
        ps.fill_filter(p, sw, w, c_logical=c_log)
        plan = ps.ConvPlan(p, mode=r["mode"], recipe=r["recipe"])
        plan.prepack(w)
        plan.forward(x, None, y, prepacked=True)  # exactly one conv kernel launch
        torch.cuda.synchronize()
        plan.close()
        del x, w, y
        torch.cuda.empty_cache()


def table(sweep, ncu_csv):
    recs = records(sweep)
    rows = [r for r in csv.reader(open(ncu_csv)) if len(r) > 10 and r[0].isdigit()]
    # long format: one row per (launch id, metric)
    by_id = {}
    for r in rows:
        by_id.setdefault(int(r[0]), {})[r[-3]] = (float(r[-1].replace(",", "")), r[-2])
    ids = sorted(by_id)
    if len(ids) != len(recs):
        raise SystemExit(f"{len(ids)} profiled launches for {len(recs)} sweep records")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "hz": 1,
             "msecond": 1e-3, "Hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "%": 1}
    print("# Per-layer ncu (1 B200, `tools/ncu_layers.py`; cold caches, serialised launches, clock-control none)\n")
    print("| layer | mode | kernel us | SM GHz | tensor pipe % | DRAM MB | DRAM / compulsory | DRAM GB/s | DRAM % of peak "
          "| compulsory MB | L2->SM MB |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for i, r in zip(ids, recs):
        m = by_id[i]
        v = {k: m[k][0] * scale.get(m[k][1], 1) for k in m}
        t = v["gpu__time_duration.sum"]
        mb = (v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]) / 1e6
        l2 = v.get("lts__t_sectors_srcunit_tex_op_read.sum", 0.0) * 32 / 1e6
        print(f"| {r['layer']} | {r['mode']} | {t * 1e6:.1f} | {v['sm__cycles_elapsed.avg.per_second'] / 1e9:.2f} | "
              f"{v['sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed']:.1f} | {mb:.1f} | "
              f"{mb / r['mb_compulsory']:.3f} | {mb / 1e3 / t:.0f} | "
              f"{v['dram__throughput.avg.pct_of_peak_sustained_elapsed']:.1f} | {r['mb_compulsory']} | {l2:.0f} |")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        table(sys.argv[2], sys.argv[3])
