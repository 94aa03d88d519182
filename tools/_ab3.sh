cd $GRAFT_REPO_ROOT
for pr in 256 64 0 128; do
  echo "== promo$pr"
  PSCONV_A_PROMO=$pr python tools/ab_sweep.py profiles/r02_sweep_first.jsonl --only cfg3,r50_l2_3x3s2_128_128,r50_l2_ds_1x1s2_256_512,r50_l3_3x3s2_256_256,r50_l3_ds_1x1s2_512_1024,r50_l4_3x3s2_512_512,r50_l4_ds_1x1s2_1024_2048 --steps 10
done > gpurun_out/ab3.log 2>&1
python tools/ab_cmp.py gpurun_out/ab3.log
