# Re-tune every (descriptor, mode) of the plan cache + the per-layer sweep with the current kernels
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/plans_b200.json gpurun_out/tune_rows.tsv gpurun_out/sweep.jsonl
python bench.py --tune-plans 4 --plans-out gpurun_out/plans_b200.json --rows gpurun_out/tune_rows.tsv \
  --layers all --no-headline --no-cpu --jsonl gpurun_out/sweep.jsonl --md gpurun_out/sweep.md \
  > gpurun_out/sweep.json 2> gpurun_out/sweep.err
echo "sweep rc=$?"
python - <<'PY' > gpurun_out/tune_cfg5.log 2>&1
import sys; sys.path.insert(0, ".")
import paper_2002_02145_b200 as ps
from paper_2002_02145_b200 import tune
from paper_2002_02145_b200.workloads import ALL, with_images, seeds
conv, c, cid = ALL["cfg5"]
for n in (2048, 1024, 512, 256):
    p = ps.ConvPreset.parse(with_images(conv, n))
    for m in ("3xtf32", "tf32", "f16x2"):
        r, rows = tune.autotune(p, m, k=4, c_logical=c, seeds=seeds(cid), cache_path="gpurun_out/plans_b200.json",
                                report_path="gpurun_out/tune_rows.tsv")
        print(n, m, r, rows[0][2], flush=True)
PY
echo "cfg5 rc=$?"
tail -4 gpurun_out/sweep.md
