# One GPU pass: the -m gpu suite, smoke, the bench line of each BASELINE config, and an ncu --set full
# capture of the headline's busiest-stage conv launches (profiles/ncu_conv_summary.json).
# Usage (GPU box): TAG=c4 bash scripts/gpu_check.sh
TAG=${TAG:-run}
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_gputest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1
for c in ${CONFIGS:-bert_base inception_v3 vgg16_churn}; do
  timeout 900 python bench.py --config $c --no-variants > $O/${TAG}_bench_$c.log 2>&1; echo "rc=$?" >> $O/${TAG}_bench_$c.log
done
if [ -n "$NCU" ]; then
  IFS=: read A B K BUD <<< "$NCU"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'conv_(tc|halo)_kernel' -c 60 \
    -o /tmp/${TAG}_stage_conv python scripts/ncu_stage.py resnet50 $A $B $K $BUD > $O/${TAG}_ncu_stage.log 2>&1
  python scripts/ncu_conv_summary.py /tmp/${TAG}_stage_conv.ncu-rep resnet50:$A:$B:$K:$BUD >> $O/${TAG}_ncu_stage.log 2>&1
  # the report itself stays on the box (too large to merge back): details pages only
  ncu -i /tmp/${TAG}_stage_conv.ncu-rep --page details --csv > $O/${TAG}_stage_conv_details.csv 2>/dev/null
  ncu -i /tmp/${TAG}_stage_conv.ncu-rep --page raw --csv > /tmp/raw.csv 2>/dev/null && gzip -c /tmp/raw.csv > $O/${TAG}_stage_conv_raw.csv.gz
  cp profiles/ncu_conv_summary.json $O/${TAG}_ncu_conv_summary.json
fi
