for kps in 1 2; do GX_KPS=$kps python scripts/bench_conv.py l1_1x1_64_256_k8,l1_3x3_64_k8,l3_3x3_256_k8,l3_1x1_1024_256_k8,l4_3x3_512_k8 3 | sed "s/^/kps=$kps /"; done
python scripts/bench_conv.py l1_1x1_64_256_k8,l1_3x3_64_k8,l3_3x3_256_k8,l3_1x1_1024_256_k8,l4_3x3_512_k8,stem 3
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/kernel_roofline.py --points 0:18:16:148,0:18:8:3,0:18:1:2,9:18:4:2,15:18:1:1 --out gpurun_out/kr7.csv > gpurun_out/kr7.log 2>&1
