# conv_tc: descriptor bases + offsets in the common MMA branch.
O=gpurun_out
T=${TAG:-v10}
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_models_gpu.py -x -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
if grep -q "rc=0" $O/${T}_tests.log; then
timeout 600 python scripts/kernel_roofline.py --model resnet50 --points 0:18:16:2,2:18:16:6 --out $O/${T}_roof_r50.csv > $O/${T}_roof_r50.log 2>&1
timeout 600 python scripts/kernel_roofline.py --model inception_v3 --points 0:19:8:5 --out $O/${T}_roof_incep.csv > $O/${T}_roof_incep.log 2>&1
timeout 600 python scripts/kernel_roofline.py --model vgg16 --points 0:5:4:3,5:8:1:6 --out $O/${T}_roof_vgg.csv > $O/${T}_roof_vgg.log 2>&1
timeout 600 python scripts/kernel_roofline.py --model bert_base --points 0:12:8:8 --out $O/${T}_roof_bert.csv > $O/${T}_roof_bert.log 2>&1
fi
