cd $GRAFT_REPO_ROOT
L3=conv:256,256,256,14,14,3,3,1,1,16,1,1,14,14
L1=conv:256,64,64,56,56,3,3,1,1,16,1,1,56,56
L4=conv:256,512,512,7,7,3,3,1,1,16,1,1,7,7
for d in 0 2; do
PSCONV_DEBUG=$d timeout 120 python tools/_wgt.py $L3 tf32 - 
PSCONV_DEBUG=$d timeout 120 python tools/_wgt.py $L1 tf32 - 
PSCONV_DEBUG=$d timeout 120 python tools/_wgt.py $L4 tf32 - 
done
timeout 120 python tools/_wgt.py $L3 3xtf32 -
timeout 120 python tools/_wgt.py $L4 tf32 "gpu=box:8x8" "gpu=box:8x7,sp:4" 
