"""Offline check of the selector's closed-form model against measured tuner rows (CPU only).
For every (descriptor, mode) group of a `ranked` rows file (bench.py --tune-plans / tune.py),
re-evaluates the CURRENT model on every timed candidate and reports the measured time of the
model's pick relative to the measured best (the VERDICT r1 bar: <= 1.05 on every group).
  python tools/model_fit.py profiles/r02_tune_rows.tsv [--show 20]
"""
import argparse
import collections
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2002_02145_b200 as ps  # noqa: E402


def load(path):
    rows = collections.defaultdict(dict)
    for line in open(path):
        f = line.rstrip("\n").split("\t")
        if f[0] != "ranked":
            continue
        conv, mode = f[1].rsplit("|", 1)
        us = float(f[5].split("=")[1])
        rid = f[3]
        rows[(conv, mode)][rid] = min(us, rows[(conv, mode)].get(rid, 1e30))
    return rows


def evaluate(rows):
    out = []
    for (conv, mode), cands in rows.items():
        p = ps.ConvPreset.parse(conv)
        best = min(cands.values())
        scored = []
        for rid, us in cands.items():
            try:
                scored.append((ps.model_us(p, rid, mode), rid, us))
            except ps.ConfigRejectedError:
                continue
        pick = min(scored)
        out.append((pick[2] / best, conv, mode, pick[1], min(cands, key=cands.get)))
    return sorted(out, reverse=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rows")
    ap.add_argument("--show", type=int, default=20)
    a = ap.parse_args()
    res = evaluate(load(a.rows))
    g = math.exp(sum(math.log(r[0]) for r in res) / len(res))
    print(f"groups {len(res)}  geomean(pick/best) {g:.4f}  within 1.05: {sum(r[0] <= 1.05 for r in res)}  "
          f"max {res[0][0]:.3f}")
    for r in res[:a.show]:
        print(f"{r[0]:.3f} {r[1][:44]:44s} {r[2]:6s} pick {r[3].split('gpu=')[1]:42s} best {r[4].split('gpu=')[1]}")


if __name__ == "__main__":
    main()
