cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_plans.py tests/test_dist_gpu.py tests/test_gpu_contract.py -m gpu -q -p no:cacheprovider -s > gpurun_out/pytest_gpu2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
tail -5 gpurun_out/pytest_gpu2.log
