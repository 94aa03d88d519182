cd $GRAFT_REPO_ROOT
P="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu="
L43="conv:256,512,2048,7,7,1,1,1,1,16,0,0,7,7"
L42="conv:256,2048,512,7,7,1,1,1,1,16,0,0,7,7"
L31="conv:256,1024,256,14,14,1,1,1,1,16,0,0,14,14"
{
for b in 1x1x128 7x1x18 7x7x2 7x2x9 7x3x6; do
  python tools/conv_times.py $L43 tf32 "${P}bn:256,box:$b,cl:2,ks:3,eg:2" "${P}bn:256,box:$b,cl:2" "${P}bn:128,box:$b,cl:2"
  python tools/conv_times.py $L42 tf32 "${P}bn:256,box:$b,cl:2,os:8" "${P}bn:256,box:$b,cl:2" "perm=oj,ofm_tile,ifm_tile,kj,ki;gpu=bn:256,box:$b,cl:2,os:8"
done
for b in 1x1x128 14x1x9 14x9x1 14x3x3 14x2x4 2x1x64 2x2x32 14x4x2; do
  python tools/conv_times.py $L31 tf32 "${P}bn:256,box:$b,cl:2,os:8"
done
} > gpurun_out/l4box.txt 2>&1
