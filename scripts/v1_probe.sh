# Re-entry verification at HEAD: GPU suite, smoke, default bench line.
O=gpurun_out
TAG=${TAG:-v1} CONFIGS=" " bash scripts/gpu_check.sh
timeout 1200 python bench.py > $O/${TAG:-v1}_bench.json 2> $O/${TAG:-v1}_bench.log; echo "rc=$?" >> $O/${TAG:-v1}_bench.log
