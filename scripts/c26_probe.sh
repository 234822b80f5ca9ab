O=gpurun_out
rm -f paper_2312_10636_b200/_gx.so; rm -rf paper_2312_10636_b200/_build
GX_BUILD_DEV=1 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in "" GX_KPS=2 GX_KPS=3 GX_BN=128 GX_BN=256 "GX_BN=128 GX_KPS=2" GX_STAGES=2 GX_FC_SIMT=1; do
  echo "### ${v:-default}" >> $O/c26_fc.log
  env $v timeout 120 python scripts/probe_fc.py >> $O/c26_fc.log 2>&1
done
