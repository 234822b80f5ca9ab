# A/B of conv kernel-selection switches on a development build (GX_BUILD_DEV=1), 2-SM budget, k=16.
# Usage (GPU box, scratch copy): bash scripts/conv_ab.sh > gpurun_out/conv_ab.log
set -e
rm -rf paper_2312_10636_b200/_build paper_2312_10636_b200/_gx.so
GX_BUILD_DEV=1 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
S=${SHAPES:-l1_1x1_64_256_k16_res,l1_1x1_64_256_k16,l1_1x1_256_64_k16,l1_1x1_64_64_k16,l1_3x3_64_k16,l2_1x1_128_512_k16_res,l2_3x3_128_k16,l3_1x1_256_1024_k16_res}
for v in "" GX_NO_BRES=1 GX_NO_YSTORE=1 GX_NO_RES_MMA=1 "GX_NO_YSTORE=1 GX_NO_RES_MMA=1" GX_NO_WSTORE=1 GX_CONV_DBG=8 GX_CONV_DBG=1 GX_CONV_DBG=4; do
  echo "### ${v:-default}"
  env $v python scripts/bench_conv.py $S 2
done
