# BN=128 for epilogue-residual convs with K >= 256.
O=gpurun_out
T=${TAG:-v15}
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 600 python scripts/kernel_roofline.py --model resnet50 --points 0:18:16:2,0:18:16:6,2:18:16:6 --out $O/${T}_roof_r50.csv > $O/${T}_roof_r50.log 2>&1
