O=gpurun_out
run() { local tag=$1; shift
  timeout 400 python bench.py --no-cpu-baseline --no-variants "$@" > $O/c31_$tag.log 2>&1
  echo "$tag $(grep '^{' $O/c31_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['p99_ms'], d['dropped'], d['unfinished_after_drain'], d['clocks']['sm_mhz'])")" >> $O/c31.log
}
run F4_3072 --plans resnet50_s2_m0 --clients 3072 --sm-oversubscribe 4
run F4_3328 --plans resnet50_s1.5_m0 --clients 3328 --sm-oversubscribe 4
run F5_3072 --plans resnet50_s2_m0 --clients 3072 --sm-oversubscribe 5
run F5_3328 --plans resnet50_s1.5_m0 --clients 3328 --sm-oversubscribe 5
run F4_3584 --plans resnet50_s1.5_m0 --clients 3584 --sm-oversubscribe 4
