cd $GRAFT_REPO_ROOT
for bp in 0 1; do
  export PSCONV_BPROD=$bp
  echo "== PSCONV_BPROD=$bp"
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "baseline_shapes or recipes or stage_geometry or split or tail or deep_output or tmem" -p no:cacheprovider 2>&1 | tail -1
  P="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu="
  python tools/conv_times.py "conv:256,2048,512,7,7,1,1,1,1,16,0,0,7,7" tf32 "perm=oj,ofm_tile,ifm_tile,kj,ki;gpu=bn:256,box:1x1x128,cl:2,os:8" "${P}bn:256,box:1x1x128,cl:2"
  python tools/conv_times.py "conv:256,512,2048,7,7,1,1,1,1,16,0,0,7,7" tf32 "${P}bn:256,box:1x1x128,cl:2,ks:3,eg:2"
  python tools/conv_times.py "conv:256,1024,256,14,14,1,1,1,1,16,0,0,14,14" tf32 "${P}bn:256,box:1x1x128,cl:2,os:8"
  python tools/conv_times.py "conv:256,512,1024,14,14,1,1,1,1,16,0,0,14,14" tf32 "${P}bn:256,box:2x2x32,cl:2"
  python tools/conv_times.py "conv:256,512,512,7,7,3,3,1,1,16,1,1,7,7" tf32 "${P}bn:256,box:1x1x128,cl:2,ks:3,eg:2"
  python tools/conv_times.py "conv:56,128,128,28,28,3,3,2,2,16,1,1,56,56" tf32 "${P}bn:128,box:4x4x8,cl:2"
  python tools/conv_times.py "conv:56,128,128,28,28,3,3,2,2,16,1,1,56,56" 3xtf32 "${P}bn:128,box:4x4x8,cl:1,ks:3,eg:2,ch:16"
  python tools/conv_times.py "conv:2048,256,256,14,14,3,3,1,1,16,1,1,14,14" tf32 "${P}bn:256,box:1x1x128,cl:2"
  python tools/conv_times.py "conv:2048,256,256,14,14,3,3,1,1,16,1,1,14,14" 3xtf32 "${P}bn:256,box:1x1x128,cl:1,eg:2,ch:36"
  python tools/conv_times.py "conv:28,64,64,56,56,3,3,1,1,16,1,1,56,56" 3xtf32 "${P}bn:64,box:8x4x4,cl:1,ch:36"
  python tools/conv_times.py "conv:28,64,256,56,56,1,1,1,1,16,0,0,56,56" 3xtf32 "${P}bn:64,box:4x8x4,cl:1,ch:16"
  python tools/conv_times.py "conv:256,256,256,14,14,3,3,2,2,16,1,1,28,28" tf32 "perm=kj,ki,oj,ofm_tile,ifm_tile;gpu=bn:256,box:2x2x32,cl:2"
done > gpurun_out/bprod.txt 2>&1
