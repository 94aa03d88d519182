# ncu --set full of the small BASELINE layers' conv kernel (one launch each, after warm-up)
cd $GRAFT_REPO_ROOT
R1T="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu=bn:64,box:56x2x1,cl:2,halo:1"
R1X="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu=bn:64,box:8x4x4,cl:1,ch:12"
R3T="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu=bn:128,box:4x4x8,cl:2,eg:2"
C1="conv:28,64,64,56,56,3,3,1,1,16,1,1,56,56"
C3="conv:56,128,128,28,28,3,3,2,2,16,1,1,56,56"
python tools/conv_times.py $C1 tf32 "$R1T" > gpurun_out/ncu_small_plain.log 2>&1 && \
python tools/conv_times.py $C1 3xtf32 "$R1X" >> gpurun_out/ncu_small_plain.log 2>&1 && \
python tools/conv_times.py $C3 tf32 "$R3T" >> gpurun_out/ncu_small_plain.log 2>&1 && \
for spec in "c1t|$C1|tf32|$R1T" "c1x|$C1|3xtf32|$R1X" "c3t|$C3|tf32|$R3T"; do
  IFS="|" read -r tag conv mode rec <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:conv_fwd_sm100 -s 5 -c 1 \
      -o gpurun_out/ncu_$tag -f python tools/conv_times.py "$conv" $mode "$rec" > gpurun_out/ncu_$tag.log 2>&1
done
ls -la gpurun_out/
for tag in c1t c1x c3t; do
  if [ -f gpurun_out/ncu_$tag.ncu-rep ]; then
    ncu -i gpurun_out/ncu_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_${tag}_raw.csv 2>/dev/null
    ncu -i gpurun_out/ncu_$tag.ncu-rep --page details --csv > gpurun_out/ncu_${tag}_details.csv 2>/dev/null
    ncu -i gpurun_out/ncu_$tag.ncu-rep --page source --csv > gpurun_out/ncu_${tag}_source.csv 2>/dev/null
    rm -f gpurun_out/ncu_$tag.ncu-rep
  fi
done
du -sh gpurun_out
