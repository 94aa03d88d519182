# CTA-0 clock traces (PSCONV_TRACE build, PSCONV_DEBUG=8 [+1/2/4 skips]) of the small layers
cd $GRAFT_REPO_ROOT
R1T="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu=bn:64,box:56x2x1,cl:2,halo:1"
R1X="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu=bn:64,box:8x4x4,cl:1,ch:12"
R2X="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu=bn:64,box:4x8x4,cl:1,ch:16"
C1="conv:28,64,64,56,56,3,3,1,1,16,1,1,56,56"
C2="conv:28,64,256,56,56,1,1,1,1,16,0,0,56,56"
for dbg in 8 15; do
for spec in "c1t|$C1|tf32|$R1T" "c1x|$C1|3xtf32|$R1X" "c2x|$C2|3xtf32|$R2X"; do
  IFS="|" read -r tag conv mode rec <<< "$spec"
  echo "== trace $tag dbg=$dbg"
  PSCONV_LIB_NAME=libpsconv_trace.so PSCONV_DEBUG=$dbg python tools/conv_times.py "$conv" $mode "$rec" 2>&1 | tail -200 | grep -v "^conv:"
done
done > gpurun_out/trace2.txt 2>&1
echo done
