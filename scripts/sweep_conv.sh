for lib in _gx_old.so _gx.so _gx_old.so _gx.so; do
GX_LIB=paper_2312_10636_b200/$lib timeout 300 python scripts/kernel_roofline.py --points 0:18:8:3,5:18:16:2,0:18:1:2 --out gpurun_out/kr_$lib.csv 2>&1 | grep span | sed "s/^/$lib /" | cut -c1-110
done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
