timeout 300 ncu --set full --clock-control none --import-source on -k regex:fc_kernel -c 1 -o /tmp/fc python scripts/ncu_stage.py resnet50 15 18 1 1 > /dev/null 2>&1
ncu -i /tmp/fc.ncu-rep --page source --csv --print-source sass > gpurun_out/fc_source.csv 2>/dev/null
ncu -i /tmp/fc.ncu-rep --page raw --csv > gpurun_out/fc_raw.csv 2>/dev/null
ls -la gpurun_out
