# GPU suite, bandwidth-bound kernel table (timed + ncu DRAM counts), then 3-step probes of the
# fleets named in $FLEETS (tag:clients ...)
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu2.log 2>&1; tail -3 gpurun_out/t_gpu2.log
timeout 300 python scripts/membound_bw.py --out gpurun_out/membound_bw.csv > gpurun_out/membound_bw.log 2>&1; cat gpurun_out/membound_bw.log
timeout 400 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:'gx::' --csv --log-file gpurun_out/membound_ncu.csv python scripts/membound_bw.py --iters 1 > /dev/null 2>&1
for spec in ${FLEETS:-}; do
  P=${spec%%:*}; Cn=${spec##*:}
  timeout 300 python bench.py --plans $P --clients $Cn --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p_${P}_${Cn}.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/p_${P}_${Cn}.log').read().strip().splitlines()[-1]);print('$P', $Cn, d['value'], d.get('p99_ms'))" 2>&1 | tail -1
done
