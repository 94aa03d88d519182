# Round-2 closing run: smoke, GPU tests, default bench, reference arm, all-layer sweep, then the
# ncu launch list and one --set full capture of the same bench command (numbers under ncu are
# never bench values).
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/f_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err; echo "ref rc=$?"
timeout 1500 python bench.py --layers all --no-headline --no-cpu --jsonl gpurun_out/f_sweep.jsonl --md gpurun_out/f_sweep.md > gpurun_out/f_sweep.json 2> gpurun_out/f_sweep.err; echo "sweep rc=$?"; tail -4 gpurun_out/f_sweep.md
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --layers none --no-cpu --no-f16x2 > gpurun_out/f_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_fwd_sm100 -s 4 -c 1 -o gpurun_out/f_cfg5_full -f python bench.py --steps 2 --warmup 3 --layers none --no-cpu --no-f16x2 > gpurun_out/f_ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:"conv_(fwd|pp)_sm100" --csv --log-file gpurun_out/f_ncu_layers.csv python tools/ncu_layers.py run gpurun_out/f_sweep.jsonl > gpurun_out/f_ncu_layers.log 2>&1; echo "ncu layers rc=$?"
python tools/ncu_layers.py table gpurun_out/f_sweep.jsonl gpurun_out/f_ncu_layers.csv > gpurun_out/f_ncu_layers.md 2>&1; echo "table rc=$?"
