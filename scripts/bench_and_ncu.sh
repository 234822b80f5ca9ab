# bench once, then an ncu --set full capture of the conv launches of the busiest stage it reports
set -x
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench3.log 2> gpurun_out/bench3.err
KEY=$(python - <<'PY'
import json,re
d=json.loads(open("gpurun_out/bench3.log").read().strip().splitlines()[-1])
m=re.search(r"span \[(\d+),(\d+)\) k=(\d+) on (\d+) SMs", d["roofline"]["kernel"])
print(":".join(m.groups()))
PY
)
IFS=: read A B K BUD <<< "$KEY"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'conv_(tc|halo)_kernel' -c 60 -o /tmp/stage_conv python scripts/ncu_stage.py resnet50 $A $B $K $BUD > gpurun_out/ncu_stage.log 2>&1
python scripts/ncu_conv_summary.py /tmp/stage_conv.ncu-rep resnet50:$A:$B:$K:$BUD
cp profiles/ncu_conv_summary.json gpurun_out/
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_serving.csv python bench.py --clients 256 --steps 1 --warmup 3 --window 0.25 --no-cpu-baseline > /dev/null 2>&1
ncu --import /tmp/stage_conv.ncu-rep --page details --csv -k regex:conv_tc 2>/dev/null | head -400 > gpurun_out/stage_conv_details.csv
echo done
