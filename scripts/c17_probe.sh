O=gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_models_gpu.py -x -q > $O/c17_tests.log 2>&1; echo "rc=$?" >> $O/c17_tests.log
GRAPH=1 timeout 300 python scripts/bench_conv.py l1_1x1_256_64_k16,l1_1x1_64_256_k16_res,l1_1x1_64_256_k16,l2_1x1_128_512_k16_res,l1_3x3_64_k16,l3_1x1_1024_256_k8,l3_3x3_256_k8,l4_3x3_512_k1,l4_1x1_512_2048_k1_res 2 > $O/c17_conv.log 2>&1
timeout 600 python scripts/kernel_roofline.py --model resnet50 --points 2:18:16:2,1:18:16:4 --out $O/c17_roof.csv > $O/c17_roof.log 2>&1
