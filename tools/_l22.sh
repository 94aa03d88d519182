cd $GRAFT_REPO_ROOT
P="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu="
L22="conv:256,512,128,28,28,1,1,1,1,16,0,0,28,28"
L31="conv:256,1024,256,14,14,1,1,1,1,16,0,0,14,14"
L42="conv:256,2048,512,7,7,1,1,1,1,16,0,0,7,7"
{
python tools/conv_times.py $L22 3xtf32 "${P}bn:256,box:4x4x8,cl:1,os:8,ch:8" "${P}bn:128,box:4x4x8,cl:1,ch:8" "${P}bn:128,box:4x4x8,cl:1,ta:1,ch:8" "${P}bn:128,box:4x4x8,cl:1,ta:1,os:8,ch:8" "${P}bn:128,box:2x4x16,cl:1,ta:1,ch:8" "${P}bn:128,box:4x4x8,cl:1,ta:1,eg:2,ch:8" "${P}bn:64,box:4x4x8,cl:1,ch:8" "${P}bn:64,box:4x4x8,cl:1,os:8,ch:8" "${P}bn:128,box:4x4x8,cl:1,ta:1,kg:4,ch:8" "${P}bn:128,box:4x4x8,cl:1,ta:1,kg:2,ch:8"
python tools/conv_times.py $L31 3xtf32 "${P}bn:256,box:1x1x128,cl:1,ch:16" "${P}bn:128,box:1x1x128,cl:1,ta:1,ch:16" "${P}bn:128,box:1x1x128,cl:1,ta:1,os:8,ch:16" "${P}bn:128,box:1x1x128,cl:1,ch:16"
python tools/conv_times.py $L42 3xtf32 "${P}bn:256,box:1x1x128,cl:1,ch:32" "${P}bn:128,box:1x1x128,cl:1,ta:1,ch:16" "${P}bn:128,box:1x1x128,cl:1,ch:16"
python tools/conv_times.py $L31 tf32 "${P}bn:256,box:1x1x128,cl:2,os:8" "${P}bn:256,box:1x1x128,cl:1,os:8" "${P}bn:128,box:1x1x128,cl:2,os:8" "${P}bn:128,box:1x1x128,cl:1,os:8" "${P}bn:128,box:1x1x128,cl:1,os:12"  "${P}bn:256,box:1x1x128,cl:2,os:8,kg:4" "${P}bn:256,box:1x1x128,cl:2,os:8,kg:1"
python tools/conv_times.py $L42 tf32 "${P}bn:256,box:1x1x128,cl:2,os:8" "${P}bn:256,box:1x1x128,cl:2,os:8,kg:4" "${P}bn:256,box:1x1x128,cl:2,kg:8" "${P}bn:256,box:1x1x128,cl:1" "${P}bn:128,box:1x1x128,cl:2,os:8" "${P}bn:256,box:1x1x128,cl:2,ks:2" "${P}bn:256,box:1x1x128,cl:2,ks:3"
} > gpurun_out/l22.txt 2>&1
