O=gpurun_out
for n in 2816 3072 3328; do
  GX_SERVE_DEBUG=1 timeout 300 python bench.py --plans $( [ $n = 3328 ] && echo resnet50_s1.5_m0 || echo resnet50_s2_m0 ) --clients $n --no-cpu-baseline --no-variants > $O/c29_$n.log 2>&1
  echo "$n $(grep '^{' $O/c29_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['p99_ms'], d['dropped'], d['unfinished_after_drain'])")" >> $O/c29.log
  grep "serve\] wall" $O/c29_$n.log >> $O/c29.log
done
