EKS_GRID_DEBUG=1 OP=cfg5 python tools/debug_t64.py 16 1 2>&1 | tail -12
