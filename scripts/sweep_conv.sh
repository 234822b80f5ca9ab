for ns in 30 64 128; do for tc in resnet50_s1.5:1472 resnet50_s1.5:1536 resnet50_s1.5:1600; do
tag=${tc%%:*}; c=${tc##*:}
GX_SERVE_STREAMS=$ns timeout 300 python bench.py --plans $tag --clients $c --no-cpu-baseline --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('streams=$ns $tag $c', d['value'], d['p99_ms'], 'e2e', d['e2e']['value'], d['e2e']['p99_ms'])"
done; done
