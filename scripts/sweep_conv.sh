for ncs in 4 1 16; do for c in 1152 1280; do
GX_COPY_STREAMS=$ncs timeout 300 python bench.py --plans resnet50 --clients $c --no-cpu-baseline --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('copy=$ncs $c', d['value'], d['p99_ms'], 'e2e', d['e2e']['value'], d['e2e']['p99_ms'])"
done; done
