cd $GRAFT_REPO_ROOT
P="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu="
C2="conv:28,64,256,56,56,1,1,1,1,16,0,0,56,56"
C1="conv:28,64,64,56,56,3,3,1,1,16,1,1,56,56"
{
for b in 4x8x4 8x16x1 8x8x2 8x4x4 56x2x1 28x4x1 16x8x1 8x2x8 8x1x16; do
  python tools/conv_times.py $C2 3xtf32 "${P}bn:64,box:$b,cl:1,ch:16" "${P}bn:64,box:$b,cl:1,ch:16,ta:0" "${P}bn:64,box:$b,cl:1,ch:16,kg:2" "${P}bn:64,box:$b,cl:1,ch:16,eg:2,kg:2" "${P}bn:32,box:$b,cl:1,ch:16"
done
for b in 8x4x4 8x8x2 8x16x1 56x2x1 28x4x1 14x8x1; do
  python tools/conv_times.py $C1 3xtf32 "${P}bn:64,box:$b,cl:1,ch:36" "${P}bn:64,box:$b,cl:1,ch:36,kg:2" "${P}bn:64,box:$b,cl:1,ch:36,eg:2" "${P}bn:64,box:$b,cl:1,ch:36,ta:0"
done
} > gpurun_out/c2grid.txt 2>&1
