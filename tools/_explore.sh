cd $GRAFT_REPO_ROOT
R=""
for box in 4x4x8 2x2x32 4x8x4 8x4x4 2x4x16 4x2x16 8x8x2 8x2x8 2x8x8 14x2x4 7x4x4 28x1x4; do for cl in 1 2; do for ks in 1 2 3; do
R="$R gpu=bn:128,box:$box,cl:$cl,ks:$ks"; done; done; done
timeout 600 python tools/recipe_times.py cfg3 tf32 $R 2>&1 | sort -k3 -n | head -12
R=""
for box in 4x4x8 2x2x32 4x8x4 8x4x4 2x4x16 4x2x16 8x2x8 14x2x4; do for ks in 1 3; do for x in "" ",eg:2" ",ta:1"; do
R="$R gpu=bn:128,box:$box,cl:1,ks:$ks$x"; done; done; done
for box in 4x4x8 8x4x4 2x4x16; do R="$R gpu=bn:64,box:$box,cl:1 gpu=bn:64,box:$box,cl:1,ks:2"; done
timeout 600 python tools/recipe_times.py cfg3 3xtf32 $R 2>&1 | sort -k3 -n | head -12
