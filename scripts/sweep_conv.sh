for c in 1024 1152; do for m in zero_copy dma; do
timeout 300 python bench.py --clients $c --e2e-ingress $m --no-cpu-baseline --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c $m', d['value'], d['p99_ms'], 'e2e', d['e2e']['value'], d['e2e']['p99_ms'])"
done; done
