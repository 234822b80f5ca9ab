# MPS feasibility: two serving processes, each its own CUDA context (own hardware queues)
O=gpurun_out
export CUDA_MPS_PIPE_DIRECTORY=/tmp/gx-mps-pipe CUDA_MPS_LOG_DIRECTORY=/tmp/gx-mps-log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d; echo "mps start rc=$?" > $O/c14.log
for n in 1536 1792; do
  (timeout 400 python bench.py --plans resnet50_s2_m0 --clients $n --no-cpu-baseline --no-variants --sm-oversubscribe 1.5 > $O/c14_a_$n.log 2>&1) &
  (timeout 400 python bench.py --plans resnet50_s2_m0 --clients $n --no-cpu-baseline --no-variants --sm-oversubscribe 1.5 > $O/c14_b_$n.log 2>&1) &
  wait
  for x in a b; do echo "mps 2x$n $x: $(grep '^{' $O/c14_${x}_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['p99_ms'], d['clocks'])")" >> $O/c14.log; done
done
echo quit | nvidia-cuda-mps-control; echo "mps stop rc=$?" >> $O/c14.log
