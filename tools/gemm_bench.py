"""GEMM through the nest front end's path (C = A @ B as a 1x1 conv on the sm_100a kernel):
GFLOP/s and fraction of the mode's tensor peak, kernel-only (B blocked outside the timed
region), L2 flushed, tuned top-4.   python tools/gemm_bench.py [--out profiles/r01_gemm.md]"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2002_02145_b200 import measure as bench  # noqa: E402
import paper_2002_02145_b200 as ps  # noqa: E402
from paper_2002_02145_b200.timing import L2Flush  # noqa: E402
from paper_2002_02145_b200.tune import autotune  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    _, bf16, _ = bench.peaks()
    dev = torch.device("cuda:0")
    flush = L2Flush(dev)
    rows = ["| M x N x K | mode | recipe | ms | TFLOP/s | frac of peak |", "|---|---|---|---|---|---|"]
    for (m, n, k) in [(8192, 8192, 8192), (16384, 4096, 4096), (4096, 1024, 4096)]:
        a = torch.rand(m, k, device=dev) - 0.5
        b = torch.rand(k, n, device=dev) - 0.5
        c = torch.empty(m, n, device=dev)
        for mode in ("3xtf32", "tf32"):
            preset = ps.ConvPreset.parse(f"conv:{m},{n},{k},1,1,1,1,1,1,16")
            recipe, _ = autotune(preset, mode, k=4)
            g = ps.GemmPlan(m, n, k, mode=mode, recipe=recipe)
            g.forward(a, b, c)  # blocks B once
            f = lambda: g.conv.forward(a, g._bblk, c)  # noqa: E731
            for _ in range(3):
                f()
            ts = []
            for _ in range(10):
                flush()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                f()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            tf = 2.0 * m * n * k / ms / 1e9
            peak = bf16 / 2 / (3 if mode == "3xtf32" else 1)
            ref = (a.double() @ b.double()).float()
            err = ((c - ref).norm() / ref.norm()).item()
            rows.append(f"| {m}x{n}x{k} | {mode} | `{g.recipe}` | {ms:.3f} | {tf:.1f} | {tf / peak:.3f} (relL2 {err:.1e}) |")
            print(rows[-1], flush=True)
    if args.out:
        with open(args.out, "w") as fo:
            fo.write("# GEMM via the conv kernel (nest front end path, 1 B200, L2 flushed, kernel only)\n\n")
            fo.write("\n".join(rows) + "\n")


if __name__ == "__main__":
    main()
