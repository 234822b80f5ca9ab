O=gpurun_out
run() { local tag=$1; shift
  GX_SERVE_DEBUG=1 timeout 300 python bench.py --no-cpu-baseline --no-variants "$@" > $O/c12_$tag.log 2>&1
  echo "$tag $(grep '^{' $O/c12_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['p99_ms'], 'e2e', d['e2e']['value'], d['e2e']['p99_ms'])")" >> $O/c12.log
}
for n in 2816 3072; do for l in least split; do
  run ${l}_$n --plans resnet50_s2_m0 --clients $n --sm-oversubscribe 3 --lanes $l
done; done
run split_2560 --plans resnet50_s2_m0 --clients 2560 --sm-oversubscribe 3 --lanes split
run split6_3072 --plans resnet50_s2_m0 --clients 3072 --sm-oversubscribe 6 --lanes split
