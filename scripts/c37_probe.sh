O=gpurun_out
run() { local tag=$1; shift
  timeout 400 python bench.py --no-cpu-baseline --no-variants "$@" > $O/c37_$tag.log 2>&1
  echo "$tag $(grep '^{' $O/c37_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['p99_ms'], d['dropped'], d['unfinished_after_drain'], d['clocks']['sm_mhz'])")" >> $O/c37.log
}
run s1.75_3200 --plans resnet50_s1.75_m0 --clients 3200
run s1.5_3200 --plans resnet50_s1.5_m0 --clients 3200
run s1.75_3328 --plans resnet50_s1.75_m0 --clients 3328
run s1.5_3328 --plans resnet50_s1.5_m0 --clients 3328
