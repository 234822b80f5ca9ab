O=gpurun_out
timeout 600 python scripts/kernel_roofline.py --model inception_v3 --points 0:19:8:5 --out $O/c34_roof_incep.csv > $O/c34_roof_incep.log 2>&1
timeout 1200 python bench.py --config inception_v3 --no-variants > $O/c34_bench_inception_v3.log 2>&1
