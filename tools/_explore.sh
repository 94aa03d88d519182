cd $GRAFT_REPO_ROOT
# cfg2 (1x1 256->64, 56x56, N=28) 3xTF32: boxes x kg x ta x ch x eg
R=""
for box in 4x8x4 8x4x4 8x8x2 8x16x1 4x4x8 2x8x8 8x2x8 14x8x1 28x4x1 56x2x1 7x8x2; do for x in "" ",ta:1" ",ks:2" ",kg:2" ",kg:8"; do
R="$R gpu=bn:64,box:$box,cl:1,ch:16$x"; done; done
timeout 600 python tools/recipe_times.py cfg2 3xtf32 $R 2>&1 | sort -k3 -n | head -8
# cfg1 (3x3 64->64, 56x56, N=28)
R=""
for box in 8x4x4 4x8x4 8x8x2 8x16x1 14x8x1 28x4x1 56x2x1 7x8x2; do for x in "" ",ta:1" ",ks:2" ",kg:2" ",ch:12"; do
R="$R gpu=bn:64,box:$box,cl:1,ch:36$x"; done; done
for h in "gpu=bn:64,box:56x2x1,cl:1,halo:1" "gpu=bn:64,box:28x4x1,cl:1,halo:1" "gpu=bn:64,box:30x4x1,cl:1,halo:1"; do R="$R $h"; done
timeout 600 python tools/recipe_times.py cfg1 3xtf32 $R 2>&1 | sort -k3 -n | head -8
R=""
for box in 30x4x1 56x2x1 28x4x1 14x8x1 30x2x1; do for x in ",tc:1" ",tc:1,cl:2" "" ",cl:2" ",tc:1,kg:2" ",tc:1,br:1"; do
R="$R gpu=bn:64,box:$box,halo:1$x"; done; done
for box in 8x4x4 8x8x2 8x16x1; do for cl in 1 2; do R="$R gpu=bn:64,box:$box,cl:$cl gpu=bn:64,box:$box,cl:$cl,ks:2"; done; done
timeout 600 python tools/recipe_times.py cfg1 tf32 $R 2>&1 | sort -k3 -n | head -8
