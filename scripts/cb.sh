timeout 300 python -m pytest tests/test_models_gpu.py -x -q 2>&1 | tail -2
timeout 300 python scripts/probe_perf.py resnet50 148,30,8,4 1,4,16 2>&1
timeout 300 python scripts/probe_serve.py 448,640,1024 2.0 2>&1 | sed 's/^/span  /'
