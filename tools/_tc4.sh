cd $GRAFT_REPO_ROOT
C1="conv:28,64,64,56,56,3,3,1,1,16,1,1,56,56"
for dbg in 8 10; do echo "== trace dbg $dbg"
PSCONV_LIB_NAME=libpsconv_trace.so PSCONV_DEBUG=$dbg python tools/conv_times.py $C1 tf32 "gpu=bn:64,tc:1,cl:1" 2>&1 | tail -24 | grep -v "^conv:"
done
