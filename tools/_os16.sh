cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "deep_output" -p no:cacheprovider > gpurun_out/os8_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/os8_tests.log
P="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu="
L31="conv:256,1024,256,14,14,1,1,1,1,16,0,0,14,14"
L42="conv:256,2048,512,7,7,1,1,1,1,16,0,0,7,7"
L22="conv:256,512,128,28,28,1,1,1,1,16,0,0,28,28"
L13="conv:256,256,64,56,56,1,1,1,1,16,0,0,56,56"
L11="conv:256,64,64,56,56,1,1,1,1,16,0,0,56,56"
LDS="conv:256,512,256,28,28,1,1,2,2,16,0,0,56,56"
{
for x in ",os:8" ",os:12" ",os:16" ",eg:2,os:16"; do
  python tools/conv_times.py $L31 tf32 "${P}bn:256,box:1x1x128,cl:2$x"
  python tools/conv_times.py $L42 tf32 "perm=oj,ofm_tile,ifm_tile,kj,ki;gpu=bn:256,box:1x1x128,cl:2$x"
  python tools/conv_times.py $L22 tf32 "${P}bn:256,box:2x4x16,cl:2$x"
  python tools/conv_times.py $L22 3xtf32 "${P}bn:256,box:4x4x8,cl:1,ch:8$x"
  python tools/conv_times.py $L13 tf32 "${P}bn:256,box:8x1x16,cl:2$x"
  python tools/conv_times.py $L13 3xtf32 "${P}bn:256,box:8x1x16,cl:1,ch:4$x"
  python tools/conv_times.py $L11 tf32 "${P}bn:64,box:8x1x16,cl:1$x"
  python tools/conv_times.py $L11 3xtf32 "${P}bn:64,box:8x1x16,cl:1,ch:4$x"
  python tools/conv_times.py $LDS tf32 "${P}bn:256,box:2x4x16,cl:2$x"
done
} > gpurun_out/os16.txt 2>&1
echo done
