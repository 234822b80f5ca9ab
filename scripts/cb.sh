for st in 2 4 6 8; do GX_STAGES=$st GRAPH=1 python scripts/bench_conv.py l1_3x3_k1,l3_3x3_k1,l1_1x1_576_k1 4 | sed "s/^/st=$st /"; done
