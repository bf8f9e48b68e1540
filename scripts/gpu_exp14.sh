#!/bin/bash
# k1w_quant addressing diet: bitwise A/B of the outputs, ncu time of the kernel, GPU tests
VARIANT_ROOT=scripts/debug/variants/head OUT=/tmp/head.npz timeout 600 python scripts/debug/bitwise_ab.py
OUT=/tmp/new.npz timeout 600 python scripts/debug/bitwise_ab.py
python -c "
import numpy as np
a=np.load('/tmp/head.npz'); b=np.load('/tmp/new.npz')
for k in a.files: print(k, 'bitwise equal' if np.array_equal(a[k].view(np.uint32) if a[k].dtype==np.float32 else a[k], b[k].view(np.uint32) if b[k].dtype==np.float32 else b[k]) else 'DIFFERENT')"
bash scripts/gpu_exp15.sh
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
