cd $GRAFT_REPO_ROOT
L3=conv:256,256,256,14,14,3,3,1,1,16,1,1,14,14
L4=conv:256,512,512,7,7,3,3,1,1,16,1,1,7,7
L31=conv:256,256,512,28,28,1,1,1,1,16,0,0,28,28
C5=conv:2048,256,256,14,14,3,3,1,1,16,1,1,14,14
timeout 300 python tools/_wgt.py $L3 tf32 - gpu=box:16x4,st:3 gpu=box:14x4,st:3 gpu=box:14x4,st:4 gpu=box:16x8,st:2 gpu=box:14x8,st:2
timeout 300 python tools/_wgt.py $L3 3xtf32 - gpu=box:16x4,st:2 gpu=box:14x4,st:2 gpu=box:14x4,st:3
timeout 300 python tools/_wgt.py $L4 tf32 - gpu=box:8x8,st:3 gpu=box:7x8,st:3 gpu=box:8x7,st:3 gpu=box:8x7,st:4
timeout 300 python tools/_wgt.py $L31 tf32 - gpu=box:28x2,st:3 gpu=box:8x8,st:3 gpu=box:4x16,st:3 gpu=box:28x2,st:4
timeout 300 python tools/_wgt.py $C5 tf32 - gpu=box:14x4,st:3 gpu=box:14x4,st:4
