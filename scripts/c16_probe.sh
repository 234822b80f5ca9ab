# conv k-block / tile timeline under skip variants (development build): which handoff paces a tile
O=gpurun_out
rm -f paper_2312_10636_b200/_gx.so; rm -rf paper_2312_10636_b200/_build
GX_BUILD_DEV=1 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for d in 16 17 20 21 24 25 28 29; do
  echo "### GX_CONV_DBG=$d" >> $O/c16_timeline.log
  GX_CONV_DBG=$d timeout 120 python scripts/probe_conv_timeline.py l1_1x1_256_64_k16 2 >> $O/c16_timeline.log 2>&1
done
