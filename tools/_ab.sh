timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for M in 3xtf32 tf32; do
for L in cfg1 cfg2; do
timeout 120 python tools/recipe_times.py $L $M --topk 3
timeout 120 python tools/recipe_times.py $L $M "gpu=bn:64,box:3x3x14"
done; done
