# serving lanes vs hardware queues (development build: GX_SERVE_STREAMS), then the conv A/B (c7)
O=gpurun_out
rm -f paper_2312_10636_b200/_gx.so; rm -rf paper_2312_10636_b200/_build
GX_BUILD_DEV=1 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for ns in 32 64 128; do
  GX_SERVE_STREAMS=$ns GX_SERVE_DEBUG=1 timeout 300 python bench.py --plans resnet50_s2_m0 --clients 2048 --no-cpu-baseline --no-variants --lane-priority uniform > $O/c8_streams_$ns.log 2>&1
  echo "streams=$ns $(grep '^{' $O/c8_streams_$ns.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['p99_ms'])")" >> $O/c8_streams.log
done
bash scripts/c7_probe.sh
