O=gpurun_out
run() { local tag=$1; shift
  timeout 400 python bench.py --no-cpu-baseline --no-variants "$@" > $O/c38_$tag.log 2>&1
  echo "$tag $(grep '^{' $O/c38_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['p99_ms'], d['dropped'], d['unfinished_after_drain'], d['clocks']['sm_mhz'])")" >> $O/c38.log
}
run s1.75_3456 --plans resnet50_s1.75_m0 --clients 3456
run s1.75_3584 --plans resnet50_s1.75_m0 --clients 3584
run s1.75_3328b --plans resnet50_s1.75_m0 --clients 3328
