#!/bin/bash
# k1w_quant write-out strength reduction: bitwise A/B of the outputs, per-kernel times, GPU tests
mkdir -p gpurun_out/e9
VARIANT_ROOT=scripts/debug/variants/head OUT=/tmp/head.npz timeout 600 python scripts/debug/bitwise_ab.py
OUT=/tmp/new.npz timeout 600 python scripts/debug/bitwise_ab.py
python -c "
import numpy as np
a=np.load('/tmp/head.npz'); b=np.load('/tmp/new.npz')
for k in a.files: print(k, 'bitwise equal' if np.array_equal(a[k].view(np.uint32) if a[k].dtype==np.float32 else a[k], b[k].view(np.uint32) if b[k].dtype==np.float32 else b[k]) else 'DIFFERENT')"
for rep in 1 2; do
VARIANT=head VARIANT_ROOT=scripts/debug/variants/head timeout 300 python scripts/debug/stress_time.py 2>&1 | tail -1
VARIANT=new timeout 300 python scripts/debug/stress_time.py 2>&1 | tail -1
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/e9/gpu_tests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/e9/gpu_tests.log
