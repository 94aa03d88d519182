# Ablation: what would a resident filter (no per-tile B loads) save? PSCONV_DEBUG bit 32 skips
# the B loads of the non-halo producer (results wrong); bits 1 / 2 / 4 as in _abl.sh.
cd $GRAFT_REPO_ROOT
P="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu="
L31="conv:256,1024,256,14,14,1,1,1,1,16,0,0,14,14"
L42="conv:256,2048,512,7,7,1,1,1,1,16,0,0,7,7"
L43="conv:256,512,2048,7,7,1,1,1,1,16,0,0,7,7"
L22="conv:256,512,128,28,28,1,1,1,1,16,0,0,28,28"
L13="conv:256,256,64,56,56,1,1,1,1,16,0,0,56,56"
C2="conv:28,64,256,56,56,1,1,1,1,16,0,0,56,56"
C3="conv:56,128,128,28,28,3,3,2,2,16,1,1,56,56"
for dbg in 0 32 36 33 4; do
  echo "== PSCONV_DEBUG=$dbg"
  export PSCONV_DEBUG=$dbg
  python tools/conv_times.py $L31 tf32 "${P}bn:256,box:1x1x128,cl:2" "${P}bn:128,box:1x1x128,cl:2" "${P}bn:128,box:1x1x128,cl:1"
  python tools/conv_times.py $L42 tf32 "perm=oj,ofm_tile,ifm_tile,kj,ki;gpu=bn:256,box:1x1x128,cl:2" "${P}bn:128,box:1x1x128,cl:2"
  python tools/conv_times.py $L43 tf32 "${P}bn:256,box:1x1x128,cl:2,ks:3,eg:2"
  python tools/conv_times.py $L22 tf32 "${P}bn:256,box:2x4x16,cl:2"
  python tools/conv_times.py $L22 3xtf32 "${P}bn:256,box:4x4x8,cl:1,ch:8" "${P}bn:128,box:4x4x8,cl:1,ch:8"
  python tools/conv_times.py $L13 tf32 "${P}bn:256,box:8x1x16,cl:2"
  python tools/conv_times.py $C2 tf32 "${P}bn:64,box:4x8x4,cl:1"
  python tools/conv_times.py $C2 3xtf32 "${P}bn:64,box:4x8x4,cl:1,ch:16"
  python tools/conv_times.py $C3 tf32 "${P}bn:128,box:4x4x8,cl:2"
  python tools/conv_times.py $C3 3xtf32 "${P}bn:128,box:4x4x8,cl:1,ks:3,eg:2,ch:16"
done > gpurun_out/skipb.txt 2>&1
echo done
