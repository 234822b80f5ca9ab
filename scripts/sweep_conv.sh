timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python scripts/bench_conv.py l1_3x3_64_k8,l1_3x3_k1 3
GX_NO_HALO=1 python scripts/bench_conv.py l1_3x3_64_k8,l1_3x3_k1 3 | sed 's/^/nohalo /'
for v in 0 1; do
if [ $v = 1 ]; then export GX_NO_HALO=1; else unset GX_NO_HALO; fi
timeout 300 python scripts/kernel_roofline.py --points 1:18:16:4,0:18:8:3,0:18:1:2,2:18:4:2 --out gpurun_out/kr_halo$v.csv 2>&1 | grep span | sed "s/^/nohalo=$v /" | cut -c1-110
done
