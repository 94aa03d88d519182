cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "tap_concat or halo" -p no:cacheprovider -s 2>&1 | tail -25
C1="conv:28,64,64,56,56,3,3,1,1,16,1,1,56,56"
L1="conv:256,64,64,56,56,3,3,1,1,16,1,1,56,56"
python tools/conv_times.py $C1 tf32 "gpu=bn:64,box:56x2x1,cl:2,halo:1" "gpu=bn:64,tc:1,cl:1" "gpu=bn:64,tc:1,cl:2" "gpu=bn:64,tc:1,cl:2,eg:2" "gpu=bn:64,tc:1,cl:1,eg:2" "gpu=bn:64,tc:1,cl:2,kg:1" "gpu=bn:64,tc:1,cl:1,br:0"
python tools/conv_times.py $L1 tf32 "gpu=bn:64,box:56x2x1,cl:2,halo:1,eg:2" "gpu=bn:64,tc:1,cl:1" "gpu=bn:64,tc:1,cl:2" "gpu=bn:64,tc:1,cl:2,eg:2" "gpu=bn:64,tc:1,cl:1,eg:2"
