# Final evidence pass at the round's last kernel commit: GPU suite, smoke, bench lines for every
# BASELINE config, bandwidth table (+ ncu DRAM bytes), per-op roofline tables, ncu capture of the
# headline's busiest-stage convs, serving launch list.
O=gpurun_out
T=${TAG:-f1}
timeout 1200 python -m pytest tests -m gpu -x -q > $O/${T}_gputest.log 2>&1; echo "rc=$?" >> $O/${T}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "rc=$?" >> $O/${T}_smoke.log
timeout 1500 python bench.py > $O/${T}_bench_resnet50.json 2> $O/${T}_bench_resnet50.log; echo "rc=$?" >> $O/${T}_bench_resnet50.log
for c in inception_v3 vgg16_churn bert_base; do
  timeout 900 python bench.py --config $c --no-variants > $O/${T}_bench_$c.json 2> $O/${T}_bench_$c.log; echo "rc=$?" >> $O/${T}_bench_$c.log
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > $O/${T}_bench_reference.json 2> $O/${T}_bench_reference.log
timeout 600 python scripts/membound_bw.py --out $O/${T}_membound.csv > $O/${T}_membound.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size \
  --clock-control none -k regex:'pool|gap|copy_channels|fc_kernel|gather_kernel|scatter_kernel|layernorm|conv_tc' --csv \
  --log-file $O/${T}_membound_ncu.csv python scripts/membound_bw.py --iters 1 --no-torch > $O/${T}_membound_ncu.log 2>&1
timeout 900 python scripts/kernel_roofline.py --model resnet50 --points 0:18:16:2,2:18:16:6,15:18:1:6 --out $O/${T}_roof_r50.csv > $O/${T}_roof_r50.log 2>&1
timeout 600 python scripts/kernel_roofline.py --model inception_v3 --points 0:19:8:5 --out $O/${T}_roof_incep.csv > $O/${T}_roof_incep.log 2>&1
timeout 600 python scripts/kernel_roofline.py --model vgg16 --points 0:5:4:3,5:8:1:6 --out $O/${T}_roof_vgg.csv > $O/${T}_roof_vgg.log 2>&1
timeout 600 python scripts/kernel_roofline.py --model bert_base --points 0:12:8:8 --out $O/${T}_roof_bert.csv > $O/${T}_roof_bert.log 2>&1
NCU=${NCU:-2:18:16:6}
IFS=: read A B K BUD <<< "$NCU"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'conv_(tc|halo)_kernel' -c 60 \
  -o /tmp/${T}_stage python scripts/ncu_stage.py resnet50 $A $B $K $BUD > $O/${T}_ncu_stage.log 2>&1
python scripts/ncu_conv_summary.py /tmp/${T}_stage.ncu-rep resnet50:$A:$B:$K:$BUD >> $O/${T}_ncu_stage.log 2>&1
cp profiles/ncu_conv_summary.json $O/${T}_ncu_conv_summary.json
ncu -i /tmp/${T}_stage.ncu-rep --page details --csv > $O/${T}_stage_conv_details.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/${T}_launches.csv \
  python bench.py --clients 256 --steps 1 --warmup 3 --window 0.25 --no-cpu-baseline --no-variants > /dev/null 2>&1
gzip -f $O/${T}_launches.csv
