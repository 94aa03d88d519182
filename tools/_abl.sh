# Ablations of the small BASELINE layers (profiling switches, results wrong when set):
#   PSCONV_DEBUG 1 skip A loads, 2 skip MMAs, 4 skip stores; 8 = CTA-0 clock trace (trace build)
cd $GRAFT_REPO_ROOT
R1T="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu=bn:64,box:56x2x1,cl:2,halo:1"
R1X="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu=bn:64,box:8x4x4,cl:1,ch:12"
R3T="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu=bn:128,box:4x4x8,cl:2,eg:2"
R3X="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu=bn:128,box:4x4x8,cl:1,ks:3,ch:16"
R2X="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu=bn:64,box:4x8x4,cl:1,ch:16"
C1="conv:28,64,64,56,56,3,3,1,1,16,1,1,56,56"
C2="conv:28,64,256,56,56,1,1,1,1,16,0,0,56,56"
C3="conv:56,128,128,28,28,3,3,2,2,16,1,1,56,56"
for dbg in 0 1 2 4 3 5 6 7; do
  echo "== PSCONV_DEBUG=$dbg"
  PSCONV_DEBUG=$dbg python tools/conv_times.py $C1 tf32 "$R1T"
  PSCONV_DEBUG=$dbg python tools/conv_times.py $C1 3xtf32 "$R1X"
  PSCONV_DEBUG=$dbg python tools/conv_times.py $C3 tf32 "$R3T"
  PSCONV_DEBUG=$dbg python tools/conv_times.py $C3 3xtf32 "$R3X"
  PSCONV_DEBUG=$dbg python tools/conv_times.py $C2 3xtf32 "$R2X"
done > gpurun_out/abl.txt 2>&1
# (libpsconv_trace.so is built in the container: tools/build_variant.sh trace -DPSCONV_TRACE)
for c in "$C1 tf32 $R1T" "$C1 3xtf32 $R1X" "$C3 tf32 $R3T"; do
  set -- $c
  echo "== trace $1 $2"
  PSCONV_LIB_NAME=libpsconv_trace.so PSCONV_DEBUG=8 python tools/conv_times.py $1 $2 "$3" 2>&1 | tail -140
done > gpurun_out/trace.txt 2>&1
echo done
