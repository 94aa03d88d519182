cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "backward_weight" 2>&1 | tail -4
L3=conv:256,256,256,14,14,3,3,1,1,16,1,1,14,14
L1=conv:256,64,64,56,56,3,3,1,1,16,1,1,56,56
L4=conv:256,512,512,7,7,3,3,1,1,16,1,1,7,7
for L in $L3 $L1 $L4; do for m in tf32 3xtf32; do
timeout 120 python tools/_wgt.py $L $m - "gpu=tma:0"
done; done
PSCONV_DEBUG=2 timeout 120 python tools/_wgt.py $L3 tf32 -
PSCONV_DEBUG=1 timeout 120 python tools/_wgt.py $L3 tf32 -
