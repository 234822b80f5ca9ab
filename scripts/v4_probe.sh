# Inception with 64-multiple intermediates: full GPU suite + the per-op table.
O=gpurun_out
T=${TAG:-v4}
timeout 600 python scripts/kernel_roofline.py --model inception_v3 --points 0:19:8:5 --out $O/${T}_roof_incep.csv > $O/${T}_roof_incep.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${T}_gputest.log 2>&1; echo "rc=$?" >> $O/${T}_gputest.log
