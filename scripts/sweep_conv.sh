GX_CONV_DBG=16 python scripts/probe_trace_tiles.py l1_1x1_64_256_k8 3 | head -4
python scripts/bench_conv.py l1_1x1_64_256_k8,l1_3x3_64_k8,l3_3x3_256_k8,l3_1x1_1024_256_k8,l4_3x3_512_k8 3
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 python scripts/kernel_roofline.py --points 0:18:8:3,0:18:16:148,0:18:1:2 --out gpurun_out/kr9.csv > gpurun_out/kr9.log 2>&1; grep "span" gpurun_out/kr9.log
