# 3x3/1 pool with 4 channels per thread (8-byte vectors).
O=gpurun_out
T=${TAG:-v12}
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "pool" > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 600 python scripts/membound_bw.py --no-torch > $O/${T}_membound.log 2>&1
