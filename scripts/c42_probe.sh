O=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/c42_smoke.log 2>&1
timeout 1500 python bench.py > $O/c42_bench.log 2>&1
for c in inception_v3 vgg16_churn bert_base; do
  timeout 1200 python bench.py --config $c --no-variants > $O/c42_bench_$c.log 2>&1; echo "rc=$?" >> $O/c42_bench_$c.log
done
