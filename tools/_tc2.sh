cd $GRAFT_REPO_ROOT
C1="conv:28,64,64,56,56,3,3,1,1,16,1,1,56,56"
L1="conv:256,64,64,56,56,3,3,1,1,16,1,1,56,56"
for dbg in 0 1 2 4 6 7; do echo "== dbg $dbg"; PSCONV_DEBUG=$dbg python tools/conv_times.py $L1 tf32 "gpu=bn:64,tc:1,cl:1" "gpu=bn:64,tc:1,cl:1,eg:2"; done
echo "== trace"
PSCONV_LIB_NAME=libpsconv_trace.so PSCONV_DEBUG=8 python tools/conv_times.py $C1 tf32 "gpu=bn:64,tc:1,cl:1" 2>&1 | tail -60 | grep -v "^conv:"
