# Bandwidth-kernel evidence + Inception per-op table.
O=gpurun_out
T=${TAG:-v2}
timeout 600 python scripts/membound_bw.py --out $O/${T}_membound.csv > $O/${T}_membound.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__block_size,launch__occupancy_limit_registers,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum \
  --clock-control none -k regex:'pool|gap|copy_channels|fc_kernel|gather_kernel|scatter_kernel|layernorm' --csv \
  --log-file $O/${T}_membound_ncu.csv python scripts/membound_bw.py --iters 1 --no-torch > $O/${T}_membound_ncu.log 2>&1
timeout 600 python scripts/kernel_roofline.py --model inception_v3 --points 0:19:8:5 --out $O/${T}_roof_incep.csv > $O/${T}_roof_incep.log 2>&1
