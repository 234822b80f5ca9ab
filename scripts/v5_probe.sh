# 8-channel stems on the cp.async A path: conv tests + Inception / VGG span tables.
O=gpurun_out
T=${TAG:-v5}
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_models_gpu.py -x -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 600 python scripts/kernel_roofline.py --model inception_v3 --points 0:19:8:5 --out $O/${T}_roof_incep.csv > $O/${T}_roof_incep.log 2>&1
timeout 600 python scripts/kernel_roofline.py --model vgg16 --points 0:5:4:3 --out $O/${T}_roof_vgg.csv > $O/${T}_roof_vgg.log 2>&1
