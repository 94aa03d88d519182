cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_final.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --steps 2 --warmup 1 --layers none --no-f16x2 --no-cpu --no-verify > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_fwd_sm100" -s 3 -c 1 -o gpurun_out/r02_ncu_full_cfg5_3xtf32 python bench.py --steps 2 --warmup 2 --layers none --no-f16x2 --no-cpu --no-verify > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
