cd $GRAFT_REPO_ROOT
C1="conv:28,64,64,56,56,3,3,1,1,16,1,1,56,56"
C2="conv:28,64,256,56,56,1,1,1,1,16,0,0,56,56"
L1A="conv:256,64,64,56,56,1,1,1,1,16,0,0,56,56"
L1B="conv:256,64,256,56,56,1,1,1,1,16,0,0,56,56"
L1C="conv:256,64,64,56,56,3,3,1,1,16,1,1,56,56"
for lib in libpsconv_base.so libpsconv.so; do
  echo "== $lib"
  PSCONV_LIB_NAME=$lib python tools/conv_times.py $C1 3xtf32 "gpu=bn:64,box:8x4x4,cl:1,ch:12" "gpu=bn:64,box:8x4x4,cl:1,ch:36" "gpu=bn:64,box:4x8x4,cl:1,ch:36"
  PSCONV_LIB_NAME=$lib python tools/conv_times.py $C2 3xtf32 "gpu=bn:64,box:4x8x4,cl:1,ch:16" "gpu=bn:64,box:8x4x4,cl:1,ch:16"
  PSCONV_LIB_NAME=$lib python tools/conv_times.py $L1A 3xtf32 "gpu=bn:64,box:8x1x16,cl:1,eg:2,ch:4"
  PSCONV_LIB_NAME=$lib python tools/conv_times.py $L1B 3xtf32 "gpu=bn:64,box:8x1x16,cl:1,ch:16"
  PSCONV_LIB_NAME=$lib python tools/conv_times.py $L1C 3xtf32 "gpu=bn:64,box:8x4x4,cl:1,ch:36" "gpu=bn:64,box:56x2x1,cl:1,halo:1,eg:2,ch:36"
done
