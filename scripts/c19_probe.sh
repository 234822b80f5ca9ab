O=gpurun_out
run() { local tag=$1; shift
  GX_SERVE_DEBUG=1 timeout 300 python bench.py --no-cpu-baseline --no-variants "$@" > $O/c19_$tag.log 2>&1
  echo "$tag $(grep '^{' $O/c19_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['p99_ms'], 'e2e', d['e2e']['value'], d['e2e']['p99_ms'], d['clocks']['sm_mhz'])")" >> $O/c19.log
}
for n in 3072 2816; do for l in split edf; do run ${l}_$n --plans resnet50_s2_m0 --clients $n --lanes $l; done; done
run edf_s1.5_3328 --plans resnet50_s1.5_m0 --clients 3328 --lanes edf
run edf4_3072 --plans resnet50_s2_m0 --clients 3072 --lanes edf --sm-oversubscribe 4
