# oversubscribed SM budgets at larger fleets, and the earliest-free lane policy
O=gpurun_out
run() { # tag args...
  local tag=$1; shift
  GX_SERVE_DEBUG=1 timeout 300 python bench.py --no-cpu-baseline --no-variants "$@" > $O/c11_$tag.log 2>&1
  echo "$tag $(grep '^{' $O/c11_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['p99_ms'], 'e2e', d['e2e']['value'], d['e2e']['p99_ms'])")" >> $O/c11.log
}
run F3_s2_3072 --plans resnet50_s2_m0 --clients 3072 --sm-oversubscribe 3
run F4_s2_3072 --plans resnet50_s2_m0 --clients 3072 --sm-oversubscribe 4
run F3_s1.5_3584 --plans resnet50_s1.5_m0 --clients 3584 --sm-oversubscribe 3
run F3_s1.5_4096 --plans resnet50_s1.5_m0 --clients 4096 --sm-oversubscribe 3
run F4_s1.5_4096 --plans resnet50_s1.5_m0 --clients 4096 --sm-oversubscribe 4
run F3_s1_4608 --plans resnet50_s1_m0 --clients 4608 --sm-oversubscribe 3
run F3e_s2_3072 --plans resnet50_s2_m0 --clients 3072 --sm-oversubscribe 3 --lanes earliest
run F3e_s1.5_4096 --plans resnet50_s1.5_m0 --clients 4096 --sm-oversubscribe 3 --lanes earliest
