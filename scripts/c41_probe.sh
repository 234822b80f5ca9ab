O=gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "conv" > $O/c41_tests.log 2>&1; echo "rc=$?" >> $O/c41_tests.log
if grep -q "rc=0" $O/c41_tests.log; then
  timeout 900 python -m pytest tests -m gpu -x -q > $O/c41_gputest.log 2>&1; echo "rc=$?" >> $O/c41_gputest.log
  timeout 600 python scripts/kernel_roofline.py --model inception_v3 --points 0:19:8:5 --out $O/c41_roof_incep.csv > $O/c41_roof_incep.log 2>&1
  timeout 600 python scripts/kernel_roofline.py --model vgg16 --points 0:5:4:3 --out $O/c41_roof_vgg.csv > $O/c41_roof_vgg.log 2>&1
fi
