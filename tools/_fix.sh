cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -q -x -k "split or tail or reproduc or deep_output" -p no:cacheprovider > gpurun_out/fix_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fix_tests.log
P="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu="
{
python tools/conv_times.py "conv:256,512,2048,7,7,1,1,1,1,16,0,0,7,7" tf32 "${P}bn:256,box:1x1x128,cl:2,ks:3,eg:2" "${P}bn:256,box:1x1x128,cl:2,ks:3" "${P}bn:256,box:1x1x128,cl:2,ks:2" "${P}bn:256,box:1x1x128,cl:2,ks:4" "${P}bn:256,box:1x1x128,cl:2,ks:6" "${P}bn:256,box:1x1x128,cl:2,ks:1"
python tools/conv_times.py "conv:256,512,2048,7,7,1,1,1,1,16,0,0,7,7" 3xtf32 "${P}bn:256,box:1x1x128,cl:1,ks:3,eg:2,ch:32" "${P}bn:256,box:1x1x128,cl:1,ks:3,ch:32"
python tools/conv_times.py "conv:256,512,512,7,7,3,3,1,1,16,1,1,7,7" tf32 "${P}bn:256,box:1x1x128,cl:2,ks:3,eg:2" "${P}bn:256,box:1x1x128,cl:2,ks:3"
python tools/conv_times.py "conv:256,512,512,7,7,3,3,1,1,16,1,1,7,7" 3xtf32 "${P}bn:256,box:1x1x128,cl:1,ks:3,eg:2,ch:36" "${P}bn:256,box:1x1x128,cl:1,ks:3,ch:36"
python tools/conv_times.py "conv:256,512,512,7,7,3,3,2,2,16,1,1,14,14" tf32 "${P}bn:256,box:1x7x18,cl:2,ks:2,eg:2"
python tools/conv_times.py "conv:256,2048,1024,7,7,1,1,2,2,16,0,0,14,14" 3xtf32 "${P}bn:256,box:1x1x128,cl:1,ks:3,ch:32"
python tools/conv_times.py "conv:56,128,128,28,28,3,3,2,2,16,1,1,56,56" 3xtf32 "${P}bn:128,box:4x4x8,cl:1,ks:3,eg:2,ch:16"
python tools/conv_times.py "conv:56,128,128,28,28,3,3,2,2,16,1,1,56,56" tf32 "${P}bn:128,box:4x4x8,cl:2" "${P}bn:128,box:4x4x8,cl:2,ks:3" "${P}bn:128,box:4x4x8,cl:2,ks:2"
} > gpurun_out/fix_times.txt 2>&1
