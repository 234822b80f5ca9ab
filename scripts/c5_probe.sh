set -x
O=gpurun_out
timeout 600 python scripts/kernel_roofline.py --model resnet50 --points 17:18:1:2,15:18:1:2,14:18:2:2,9:18:4:2,17:18:4:2 --out $O/c5_roof_tail.csv > $O/c5_roof_tail.log 2>&1
rm -f paper_2312_10636_b200/_gx.so; rm -rf paper_2312_10636_b200/_build
GX_BUILD_DEV=1 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for s in l1_1x1_256_64_k16 l1_1x1_64_256_k16_res l1_3x3_64_k16 l4_3x3_512_k1 l4_1x1_512_2048_k1_res; do
  GX_CONV_DBG=16 timeout 120 python scripts/probe_conv_timeline.py $s 2 >> $O/c5_timeline.log 2>&1
done
GRAPH=1 timeout 300 python scripts/bench_conv.py l4_1x1_2048_512_k1,l4_3x3_512_k1,l4_1x1_512_2048_k1_res,l4_1x1_512_2048_k4_res,l1_1x1_256_64_k16,l1_1x1_64_256_k16_res,l1_3x3_64_k16 2 > $O/c5_bench_conv.log 2>&1
