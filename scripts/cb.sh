python scripts/probe_perf.py resnet50 148 1,16
GX_NO_PDL=1 python scripts/probe_perf.py resnet50 148 1,16
