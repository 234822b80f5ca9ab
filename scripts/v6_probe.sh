# Short A boxes for single-tile small-M GEMMs (batch-1 FC, layer4 1x1 at k=1-2): kernel tests,
# bandwidth table (FC rows), tail-span tables.
O=gpurun_out
T=${TAG:-v6}
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
if grep -q "rc=0" $O/${T}_tests.log; then
timeout 600 python scripts/membound_bw.py --no-torch --out $O/${T}_membound.csv > $O/${T}_membound.log 2>&1
timeout 600 python scripts/kernel_roofline.py --model resnet50 --points 15:18:1:6,14:18:2:6,17:18:1:2 --out $O/${T}_roof_tail.csv > $O/${T}_roof_tail.log 2>&1
timeout 600 python scripts/kernel_roofline.py --model vgg16 --points 5:8:1:6,5:8:4:6 --out $O/${T}_roof_vggtail.csv > $O/${T}_roof_vggtail.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_gputest.log 2>&1; echo "rc=$?" >> $O/${T}_gputest.log
fi
