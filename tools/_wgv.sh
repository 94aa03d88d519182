cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "backward_weight" 2>&1 | tail -1
L3=conv:256,256,256,14,14,3,3,1,1,16,1,1,14,14
L4=conv:256,512,512,7,7,3,3,1,1,16,1,1,7,7
for d in 0 1; do for L in $L3 $L4; do PSCONV_DEBUG=$d timeout 120 python tools/_wgt.py $L tf32 -; done; done
timeout 120 python tools/_wgt.py $L3 3xtf32 -
