O=gpurun_out
for c in bert_base inception_v3 vgg16_churn; do
  timeout 1200 python bench.py --config $c --no-variants > $O/c15_bench_$c.log 2>&1; echo "rc=$?" >> $O/c15_bench_$c.log
done
timeout 600 python scripts/membound_bw.py > $O/c15_membound.log 2>&1
