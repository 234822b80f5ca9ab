O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/c30_gputest.log 2>&1; echo "rc=$?" >> $O/c30_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/c30_smoke.log 2>&1
timeout 1200 python bench.py > $O/c30_bench.log 2>&1
for F in 4; do
  timeout 400 python bench.py --plans resnet50_s2_m0 --clients 3072 --no-cpu-baseline --no-variants --sm-oversubscribe $F > $O/c30_F${F}_3072.log 2>&1
done
