# ncu source-level stall sampling of one layer1 1x1 conv launch (2 SMs): where do the pipeline warps wait?
O=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:conv_tc_kernel -c 1 -o /tmp/c35 \
  python scripts/bench_conv.py l1_1x1_256_64_k16 2 > $O/c35_ncu.log 2>&1
ncu -i /tmp/c35.ncu-rep --page source --csv --print-source sass > $O/c35_source_sass.csv 2>/dev/null
ncu -i /tmp/c35.ncu-rep --page details --csv > $O/c35_details.csv 2>/dev/null
gzip -f $O/c35_source_sass.csv
