O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/c36_gputest.log 2>&1; echo "rc=$?" >> $O/c36_gputest.log
if grep -q "rc=0" $O/c36_gputest.log; then
  timeout 600 python scripts/kernel_roofline.py --model resnet50 --points 0:18:16:2,1:18:16:6 --out $O/c36_roof.csv > $O/c36_roof.log 2>&1
  timeout 1200 python bench.py --no-cpu-baseline --no-variants > $O/c36_bench.log 2>&1
fi
