cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_plans.py -q -x -p no:cacheprovider > gpurun_out/r02c_plans_tests.log 2>&1; echo "plans rc=$?"; tail -2 gpurun_out/r02c_plans_tests.log
timeout 1500 python bench.py --layers all --no-headline --no-cpu --jsonl gpurun_out/r02c_sweep.jsonl --md gpurun_out/r02c_sweep.md > gpurun_out/r02c_sweep.json 2> gpurun_out/r02c_sweep.err
echo sweep rc=$?
tail -4 gpurun_out/r02c_sweep.md
