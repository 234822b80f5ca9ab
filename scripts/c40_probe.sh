# ncu evidence for the bench line's dominant kernel (busiest stage [1,18) k=16 on 6 SMs) and a
# serving launch list (gpu__time_duration per launch of a short serving run)
O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'conv_(tc|halo)_kernel' -c 60 \
  -o /tmp/c40_stage python scripts/ncu_stage.py resnet50 2 18 16 6 > $O/c40_ncu_stage.log 2>&1
python scripts/ncu_conv_summary.py /tmp/c40_stage.ncu-rep resnet50:2:18:16:6 >> $O/c40_ncu_stage.log 2>&1
cp profiles/ncu_conv_summary.json $O/c40_ncu_conv_summary.json
ncu -i /tmp/c40_stage.ncu-rep --page details --csv > $O/c40_stage_conv_details.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/c40_launches.csv \
  python bench.py --clients 256 --steps 1 --warmup 3 --window 0.25 --no-cpu-baseline --no-variants > /dev/null 2>&1
gzip -f $O/c40_launches.csv
