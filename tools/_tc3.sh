cd $GRAFT_REPO_ROOT
L1="conv:256,64,64,56,56,3,3,1,1,16,1,1,56,56"
for dbg in 0 1 2 4 6 7; do echo "== dbg $dbg"; PSCONV_DEBUG=$dbg python tools/conv_times.py $L1 tf32 "gpu=bn:64,tc:1,cl:1" "gpu=bn:64,tc:1,cl:1,eg:2" "gpu=bn:64,box:56x2x1,cl:2,halo:1,eg:2" "gpu=bn:64,box:56x2x1,cl:2,halo:1"; done > gpurun_out/tc3.txt 2>&1
cat gpurun_out/tc3.txt
