#!/bin/bash
# compact chol_diag_warp: phase trace, per-kernel times, GPU tests
VARIANT_ROOT=scripts/debug/variants/k2wi timeout 300 python scripts/debug/k2wi_trace.py
VARIANT=new timeout 300 python scripts/debug/stress_time.py 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
