cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_sw.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_sw.log
for lib in libpsconv_base.so libpsconv.so; do
  echo "== $lib"
  PSCONV_LIB_NAME=$lib python tools/ab_sweep.py profiles/r02_sweep_first.jsonl --steps 10
done > gpurun_out/ab_sw.log 2>&1
python tools/ab_cmp.py gpurun_out/ab_sw.log
grep geomean gpurun_out/ab_sw.log
C1="conv:28,64,64,56,56,3,3,1,1,16,1,1,56,56"
echo "== trace"
PSCONV_LIB_NAME=libpsconv_trace.so PSCONV_DEBUG=8 python tools/conv_times.py $C1 tf32 "gpu=bn:64,tc:1,cl:1" 2>&1 | tail -24 | grep -v "^conv:"
