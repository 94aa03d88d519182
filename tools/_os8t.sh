cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "deep_output or split or tail" -p no:cacheprovider > gpurun_out/os8_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/os8_tests.log
