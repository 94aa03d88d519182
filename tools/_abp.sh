cd $GRAFT_REPO_ROOT
P="perm=ifm_tile,ofm_tile,oj,kj,ki;gpu="
{
python tools/ab_bench_protocol.py r50_l1_1x1_64_64 3xtf32 "${P}bn:64,box:8x1x16,cl:1,ch:4" "${P}bn:64,box:8x1x16,cl:1,os:8,ch:4" "${P}bn:64,box:8x1x16,cl:1,os:12,ch:4"
python tools/ab_bench_protocol.py r50_l1_1x1_64_256 3xtf32 "${P}bn:256,box:8x1x16,cl:1,ch:4" "${P}bn:256,box:8x1x16,cl:1,os:8,ch:4"
python tools/ab_bench_protocol.py r50_l2_1x1_128_512 3xtf32 "${P}bn:256,box:4x4x8,cl:1,ch:8" "${P}bn:256,box:4x4x8,cl:1,os:8,ch:8"
python tools/ab_bench_protocol.py r50_l1_1x1_64_64 tf32 "${P}bn:32,box:8x1x16,cl:1" "${P}bn:32,box:8x1x16,cl:1,os:8" "${P}bn:64,box:8x1x16,cl:1,os:8"
python tools/ab_bench_protocol.py r50_l4_1x1_512_2048 tf32 "perm=oj,ofm_tile,ifm_tile,kj,ki;gpu=bn:256,box:1x1x128,cl:2" "perm=oj,ofm_tile,ifm_tile,kj,ki;gpu=bn:256,box:1x1x128,cl:2,os:8"
python tools/ab_bench_protocol.py r50_l3_1x1_1024_256 tf32 "${P}bn:256,box:2x1x64,cl:2" "${P}bn:256,box:2x1x64,cl:2,os:8"
python tools/ab_bench_protocol.py cfg2 tf32 "${P}bn:64,box:4x8x4,cl:1" "${P}bn:64,box:4x8x4,cl:1,os:8"
PSCONV_PP_OUT_BLOCKS=4 python tools/ab_bench_protocol.py r50_stem tf32 "${P}bn:64,box:8x16x1,pp:3"
PSCONV_PP_OUT_BLOCKS=8 python tools/ab_bench_protocol.py r50_stem tf32 "${P}bn:64,box:8x16x1,pp:3"
PSCONV_PP_OUT_BLOCKS=4 python tools/ab_bench_protocol.py r50_stem 3xtf32 "${P}bn:64,box:8x16x1,pp:3"
PSCONV_PP_OUT_BLOCKS=8 python tools/ab_bench_protocol.py r50_stem 3xtf32 "${P}bn:64,box:8x16x1,pp:3"
} > gpurun_out/abp.txt 2>&1
timeout 300 python -m pytest tests -q -x -m gpu -k "pp or stem or parity_plane or few" -p no:cacheprovider 2>&1 | tail -2
