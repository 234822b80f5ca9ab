# ncu --set full of the busiest stage of the 3392-client fleet ([0,18) k=16 on 6 SMs).
O=gpurun_out
T=${TAG:-v14}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'conv_(tc|halo)_kernel' -c 60 \
  -o /tmp/${T}_stage python scripts/ncu_stage.py resnet50 0 18 16 6 > $O/${T}_ncu_stage.log 2>&1
python scripts/ncu_conv_summary.py /tmp/${T}_stage.ncu-rep resnet50:0:18:16:6 >> $O/${T}_ncu_stage.log 2>&1
cp profiles/ncu_conv_summary.json $O/${T}_ncu_conv_summary.json
ncu -i /tmp/${T}_stage.ncu-rep --page details --csv > $O/${T}_stage_conv_details.csv 2>/dev/null
