O=gpurun_out
for lp in time uniform; do for n in 2048 2304 2560; do
  echo "### lane=$lp clients=$n" >> $O/c6_lanes.log
  GX_SERVE_DEBUG=1 timeout 300 python bench.py --plans resnet50_s2_m0 --clients $n --no-cpu-baseline --no-variants --lane-priority $lp > $O/c6_${lp}_$n.log 2>&1
  grep "^{" $O/c6_${lp}_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['p99_ms'], d['e2e']['value'], d['e2e']['p99_ms'])" >> $O/c6_lanes.log 2>&1
done; done
