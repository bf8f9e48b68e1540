#!/bin/bash
# int8 SYRK diagonal pairs with 7 MMAs: ncu time, then the -m gpu suite
bash scripts/gpu_exp16.sh
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
