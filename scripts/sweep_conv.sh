for tc in resnet50_s1.25_m0:1920 resnet50_s1.75_m0:1920 resnet50_s1.75_m0:1984 resnet50_s2_m0:1984 resnet50_s2_m0:2048; do
tag=${tc%%:*}; c=${tc##*:}
timeout 300 python bench.py --plans $tag --clients $c --no-cpu-baseline --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$tag $c', d['value'], d['p99_ms'])"
done
