timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in 2 0; do
GX_RES2_KB=$v timeout 300 python scripts/kernel_roofline.py --points 1:18:16:4,0:18:8:3,0:18:1:2 --out gpurun_out/kr_r2$v.csv 2>&1 | grep span | sed "s/^/kb=$v /" | cut -c1-110
done
