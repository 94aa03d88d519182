cd $GRAFT_REPO_ROOT
python - <<'PY' > /tmp/layers.txt
import sys; sys.path.insert(0,'.')
from paper_2002_02145_b200.workloads import R50
for n,(c,_,_) in R50.items(): print(n, c)
PY
while read n c; do for m in tf32 3xtf32; do timeout 120 python tools/_wgt.py $c $m "gpu=tma:0" "gpu=tma:1" - 2>&1 | sed "s/^/$n /"; done; done < /tmp/layers.txt > gpurun_out/wg_tma_ab.txt
timeout 1200 python tools/resnet50_train_pass.py 2>&1 | tail -3 | tee gpurun_out/r50_train.jsonl
