cd $GRAFT_REPO_ROOT
P="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu="
L43="conv:256,512,2048,7,7,1,1,1,1,16,0,0,7,7"
L42="conv:256,2048,512,7,7,1,1,1,1,16,0,0,7,7"
L31="conv:256,1024,256,14,14,1,1,1,1,16,0,0,14,14"
for spec in "l43|$L43|tf32|${P}bn:256,box:1x1x128,cl:2,ks:3,eg:2" "l43w|$L43|tf32|${P}bn:256,box:1x1x128,cl:2,ks:1" "l42|$L42|tf32|perm=oj,ofm_tile,ifm_tile,kj,ki;gpu=bn:256,box:1x1x128,cl:2,os:8" "l31|$L31|tf32|${P}bn:256,box:1x1x128,cl:2,os:8"; do
  IFS="|" read -r tag conv mode rec <<< "$spec"
  echo "== trace $tag"
  PSCONV_LIB_NAME=libpsconv_trace.so PSCONV_DEBUG=8 python tools/conv_times.py "$conv" $mode "$rec" 2>&1 | tail -220 | grep -v "^conv:"
done > gpurun_out/trace4.txt 2>&1
echo done
