O=gpurun_out
which nvidia-cuda-mps-control nvidia-cuda-mps-server > $O/c13_mps.txt 2>&1; ls /usr/bin | grep -i nvidia >> $O/c13_mps.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/c13_gputest.log 2>&1; echo "rc=$?" >> $O/c13_gputest.log
CUDA_DEVICE_MAX_CONNECTIONS=16 timeout 300 python bench.py --plans resnet50_s2_m0 --clients 2560 --no-cpu-baseline --no-variants > $O/c13_conn16.log 2>&1
timeout 1200 python bench.py > $O/c13_bench.log 2>&1
