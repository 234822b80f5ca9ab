# conv A/B on a development build: which part of the layer1 1x1 convs at 2 SMs paces the kernel
O=gpurun_out
rm -f paper_2312_10636_b200/_gx.so; rm -rf paper_2312_10636_b200/_build
GX_BUILD_DEV=1 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
S=l1_1x1_256_64_k16,l1_1x1_64_256_k16_res,l1_1x1_64_256_k16,l2_1x1_128_512_k16_res
for v in "" GX_CONV_DBG=4 GX_CONV_DBG=8 GX_CONV_DBG=12 GX_CONV_DBG=1 GX_CONV_DBG=2 GX_STAGES=2 GX_STAGES=3 GX_KPS=1 GX_NO_BRES=1 GX_NO_WSTORE=1 GX_NO_YSTORE=1 GX_NO_RES_MMA=1 GX_BN=128; do
  echo "### ${v:-default}" >> $O/c7_ab.log
  env $v GRAPH=1 timeout 120 python scripts/bench_conv.py $S 2 >> $O/c7_ab.log 2>&1
done
