timeout 300 python -m pytest tests/test_models_gpu.py tests/test_kernels_gpu.py -x -q 2>&1 | tail -3
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 120 python scripts/probe_trace.py 4 1 2>&1 | grep -v Warn | grep -v nanm | head -5
timeout 300 python scripts/probe_perf.py resnet50 148,30,8,4,2 1,4,16 2>&1
GX_EXEC=graph timeout 300 python scripts/probe_perf.py resnet50 148,8,4 1,16 2>&1 | sed 's/^/graph /'
