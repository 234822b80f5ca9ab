# SM-budget oversubscription: with <= 32 hardware queues only ~32 batches execute at once, so
# budgets summing to ~1x the SMs leave SMs idle; budgets may sum to F x the SMs
O=gpurun_out
for F in 1 2 3; do for n in 2304 2560; do
  GX_SERVE_DEBUG=1 timeout 300 python bench.py --plans resnet50_s2_m0 --clients $n --no-cpu-baseline --no-variants --sm-oversubscribe $F > $O/c10_F${F}_$n.log 2>&1
  echo "F=$F clients=$n $(grep '^{' $O/c10_F${F}_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['p99_ms'], 'e2e', d['e2e']['value'], d['e2e']['p99_ms'])")" >> $O/c10_over.log
done; done
