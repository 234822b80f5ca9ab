# BW kernels after the pool / GAP rework: their tests, then the whole-GPU bandwidth table.
O=gpurun_out
T=${TAG:-v3}
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "pool or gap" > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 600 python scripts/membound_bw.py --out $O/${T}_membound.csv > $O/${T}_membound.log 2>&1
timeout 600 python scripts/kernel_roofline.py --model inception_v3 --points 0:19:8:5 --out $O/${T}_roof_incep.csv > $O/${T}_roof_incep.log 2>&1
timeout 600 python scripts/kernel_roofline.py --model resnet50 --points 0:18:16:2 --out $O/${T}_roof_r50.csv > $O/${T}_roof_r50.log 2>&1
