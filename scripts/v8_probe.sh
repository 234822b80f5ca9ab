# Halo conv with the nine taps unrolled (precomputed descriptors, resident weights waited once).
O=gpurun_out
T=${TAG:-v8}
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
if grep -q "rc=0" $O/${T}_tests.log; then
timeout 600 python scripts/kernel_roofline.py --model resnet50 --points 0:18:16:2,2:18:16:6 --out $O/${T}_roof_r50.csv > $O/${T}_roof_r50.log 2>&1
timeout 600 python scripts/kernel_roofline.py --model vgg16 --points 0:5:4:3 --out $O/${T}_roof_vgg.csv > $O/${T}_roof_vgg.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_gputest.log 2>&1; echo "rc=$?" >> $O/${T}_gputest.log
fi
