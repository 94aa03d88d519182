cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py --layers all --no-headline --no-cpu --jsonl gpurun_out/r02b_sweep.jsonl --md gpurun_out/r02b_sweep.md > gpurun_out/r02b_sweep.json 2> gpurun_out/r02b_sweep.err
echo sweep rc=$?
timeout 900 python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err
echo bench rc=$?
