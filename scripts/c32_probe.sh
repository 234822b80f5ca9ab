O=gpurun_out
timeout 1200 python bench.py > $O/c32_bench.log 2>&1
for c in bert_base inception_v3 vgg16_churn; do
  timeout 1200 python bench.py --config $c --no-variants > $O/c32_bench_$c.log 2>&1; echo "rc=$?" >> $O/c32_bench_$c.log
done
