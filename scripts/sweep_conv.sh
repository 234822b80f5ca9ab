GX_CONV_DBG=16 python scripts/probe_trace_tiles.py l1_1x1_64_256_k8 3 2>&1 | head -5
GX_CONV_DBG=16 GX_BN=128 python scripts/probe_trace_tiles.py l1_1x1_64_256_k8 3 2>&1 | head -5
