for tc in resnet50_s1.5:1408 resnet50_s1.5:1024 resnet50_s1.25:1280 resnet50_s1.25:1408 resnet50:1152; do
tag=${tc%%:*}; c=${tc##*:}
timeout 300 python bench.py --plans $tag --clients $c --no-cpu-baseline --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$tag $c', d['value'], d['p99_ms'], 'e2e', d['e2e']['value'], d['e2e']['p99_ms'])"
done
GX_SERVE_DEBUG=1 timeout 300 python bench.py --plans resnet50_s1.5 --clients 1152 --no-cpu-baseline --steps 2 > /dev/null 2> gpurun_out/dbg_e2e.err
