#!/bin/bash
# K1 change check on the GPU box: parity tests touching K1 + per-kernel times of one C2 turn-3 prefill
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_c2_parity.py tests/test_gpu_parity.py -q -x 2>&1 | tail -4 > gpurun_out/k1_check_tests.log
timeout 300 python tools/kprof.py > gpurun_out/k1_check_kprof.txt 2>&1
