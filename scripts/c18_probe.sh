O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/c18_gputest.log 2>&1; echo "rc=$?" >> $O/c18_gputest.log
timeout 600 python scripts/membound_bw.py --out $O/c18_membound.csv > $O/c18_membound.log 2>&1
timeout 600 python scripts/kernel_roofline.py --model resnet50 --points 17:18:1:6,15:18:1:6,1:18:16:4 --out $O/c18_roof.csv > $O/c18_roof.log 2>&1
timeout 1200 python bench.py --no-cpu-baseline > $O/c18_bench.log 2>&1
