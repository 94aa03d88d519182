"""Top stalled SASS instructions from an `ncu --page source --csv` export.
  python tools/ncu_hot.py file_source.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print("total samples", tot)
agg = {s: sum(float(r[ix[s]] or 0) for r in data) for s in stalls}
print("by reason:", ", ".join(f"{k[6:]}={v / tot:.1%}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
data.sort(key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
for r in data[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    top = sorted(((float(r[ix[k]] or 0), k[6:]) for k in stalls), reverse=True)[:2]
    print(f"{s / tot:6.1%} {r[ix['Address']]:>6} {r[ix['Source']][:70]:70} " + " ".join(f"{k}:{v / tot:.1%}" for v, k in top))
