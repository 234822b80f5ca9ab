# conv pipeline waits A/B (development builds): epilogue wait flavour and single-lane producer waits,
# plus the serving tail-stage breakdown (GPU time vs dispatch->completion) at 2048 / 2304 clients
O=gpurun_out
S=l1_1x1_256_64_k16,l1_1x1_64_256_k16_res,l2_1x1_128_512_k16_res,l1_3x3_64_k16,l3_1x1_1024_256_k8
for v in "" "-DGX_EPI_WAIT=0" "-DGX_EPI_WAIT=2" "-DGX_WAIT1" "-DGX_EPI_WAIT=0 -DGX_WAIT1"; do
  rm -f paper_2312_10636_b200/_gx.so; rm -rf paper_2312_10636_b200/_build
  GX_BUILD_DEV=1 GX_EXTRA_NVCC="$v" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "### ${v:-default}" >> $O/c9_ab.log
  GRAPH=1 timeout 120 python scripts/bench_conv.py $S 2 >> $O/c9_ab.log 2>&1
done
rm -f paper_2312_10636_b200/_gx.so; rm -rf paper_2312_10636_b200/_build
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python scripts/probe_exec_modes.py > $O/c9_exec_modes.log 2>&1
for n in 2048 2304; do
  GX_SERVE_DEBUG=1 timeout 300 python bench.py --plans resnet50_s2_m0 --clients $n --no-cpu-baseline --no-variants --lane-priority uniform > $O/c9_dbg_$n.log 2>&1
done
