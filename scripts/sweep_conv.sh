for kps in 2 3; do GX_KPS=$kps python scripts/bench_conv.py l1_3x3_64_k8 3 | sed "s/^/kps=$kps /"; done
for kps in 2 3; do
GX_KPS=$kps timeout 300 python scripts/kernel_roofline.py --points 1:18:16:4,0:18:8:3,0:18:1:2 --out gpurun_out/kr_k$kps.csv 2>&1 | grep span | sed "s/^/kps=$kps /" | cut -c1-110
done
GX_KPS=3 timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
