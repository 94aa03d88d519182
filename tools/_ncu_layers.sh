cd $GRAFT_REPO_ROOT
timeout 1500 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:"conv_(fwd|pp)_sm100" --csv --log-file gpurun_out/ncu_layers.csv python tools/ncu_layers.py run profiles/r02_sweep.jsonl > gpurun_out/ncu_layers.log 2>&1
echo rc=$?
python tools/ncu_layers.py table profiles/r02_sweep.jsonl gpurun_out/ncu_layers.csv > gpurun_out/r02_ncu_layers.md 2>&1; echo rc2=$?
