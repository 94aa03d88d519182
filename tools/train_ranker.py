"""Trains the B200 pairwise ranker on measured candidate timings and
evaluates it the way the paper does (Table 1): pairwise accuracy, and the
slowdown of the top-1 pick versus the measured best, next to the cost model's top-1.

  python tools/train_ranker.py profiles/r01_ranker_data.jsonl \
      --weights paper_2002_02145_b200/ranker_b200.pairnet --report profiles/r01_ranker.md

Evaluation is leave-layers-out: the layers are split into 5 folds; each fold's layers are
ranked by a net trained on the other folds' pairs. The shipped weights are trained on all.
"""
import argparse
import collections
import itertools
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2002_02145_b200 as ps  # noqa: E402

TIE = 1.03  # pairs within 3% of each other are not labelled


def pairs_text(groups):
    rows = []
    for recs in groups:
        for a, b in itertools.combinations(recs, 2):
            ta, tb = a["measured_us"], b["measured_us"]
            if max(ta, tb) / min(ta, tb) < TIE:
                continue
            lab = "A" if ta < tb else "B"
            rows.append(" ".join(f"{v:.6g}" for v in a["stats"] + b["stats"]) + " " + lab)
    return "\n".join(rows) + "\n", len(rows)


def top1_dnn(weights, recs):
    """Tournament among the measured candidates (wins desc, model cost, id)."""
    wins = collections.Counter()
    for i, j in itertools.combinations(range(len(recs)), 2):
        r, _, _ = ps.ranker_compare(weights, recs[i]["stats"], recs[j]["stats"])
        if r == 0:
            wins[i] += 1
        elif r == 1:
            wins[j] += 1
    return min(range(len(recs)), key=lambda i: (-wins[i], recs[i]["model_us"], recs[i]["recipe"]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("data")
    ap.add_argument("--weights", default=None)
    ap.add_argument("--report", default=None)
    ap.add_argument("--epochs", type=int, default=300)
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    recs = [json.loads(l) for l in open(args.data)]
    groups = collections.defaultdict(list)
    for r in recs:
        groups[(r["layer"], r["mode"])].append(r)
    layers = sorted({k[0] for k in groups})
    folds = [layers[i::5] for i in range(5)]
    lines = []
    regret_dnn, regret_cost, acc_fold = [], [], []
    for f, held in enumerate(folds):
        train = [g for k, g in groups.items() if k[0] not in held]
        test = [(k, g) for k, g in groups.items() if k[0] in held]
        txt, n = pairs_text(train)
        w, tr_acc, _ = ps.ranker_train(txt, epochs=args.epochs, learning_rate=args.lr, seed=args.seed,
                                       split=1.0)
        ttxt, tn = pairs_text([g for _, g in test])
        # held-out pairwise accuracy
        good = 0
        for row in ttxt.strip().split("\n") if tn else []:
            v = row.split()
            a, b, lab = [float(x) for x in v[:4]], [float(x) for x in v[4:8]], v[8]
            _, pa, pb = ps.ranker_compare(w, a, b)
            good += (pa >= pb) == (lab == "A")
        acc_fold.append(good / tn if tn else float("nan"))
        for (layer, mode), g in test:
            best = min(r["measured_us"] for r in g)
            d = g[top1_dnn(w, g)]["measured_us"] / best
            c = min(g, key=lambda r: (r["model_us"], r["recipe"]))["measured_us"] / best
            regret_dnn.append(d)
            regret_cost.append(c)
            lines.append(f"| {layer} | {mode} | {len(g)} | {c:.3f} | {d:.3f} |")
        print(f"fold {f}: train pairs {n} (acc {tr_acc:.3f}), held-out pairs {tn} (acc {acc_fold[-1]:.3f})",
              flush=True)
    gm = statistics.geometric_mean
    summary = (f"leave-layers-out (5 folds): held-out pairwise accuracy {statistics.mean(acc_fold):.3f}; "
               f"top-1 slowdown vs the measured best, geomean: cost model {gm(regret_cost):.3f}, "
               f"pairwise net {gm(regret_dnn):.3f}")
    print(summary)
    txt, n = pairs_text(list(groups.values()))
    w, tr_acc, _ = ps.ranker_train(txt, epochs=args.epochs, learning_rate=args.lr, seed=args.seed, split=1.0)
    if args.weights:
        open(args.weights, "w").write(w)
    if args.report:
        with open(args.report, "w") as fo:
            fo.write("# Pairwise ranker (PolyScientist-DNN on B200), round 1\n\n")
            fo.write(f"Data: `{os.path.basename(args.data)}` — {len(recs)} measured candidates "
                     f"({len(groups)} layer x mode groups, the cost model's top-k each; kernel only, "
                     f"prepacked, L2 flushed). Pairs labelled by measured time (ties < {TIE:.2f}x "
                     f"dropped): {n}. Net 8-64-32-16-8-2, {args.epochs} epochs, lr {args.lr}, seed "
                     f"{args.seed}; shipped weights train accuracy {tr_acc:.3f}.\n\n{summary}.\n\n")
            fo.write("| layer | mode | candidates | cost-model top-1 / best | net top-1 / best |\n"
                     "|---|---|---|---|---|\n" + "\n".join(sorted(lines)) + "\n")


if __name__ == "__main__":
    main()
