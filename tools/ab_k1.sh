# K1 A/B on the GPU box: build/ab/libA.so vs the in-tree library (plan digests + per-kernel times), phase clocks
mkdir -p gpurun_out
for i in 1 2; do for lib in build/ab/libA.so paper_2507_13681_b200/libloopserve_b200.so; do
 LS_LIB_PATH=$lib timeout 300 python tools/select_timing.py 2>&1 | grep -v -i warn | head -6
done; done > gpurun_out/ab_k1.txt
for lib in build/ab/libA.so paper_2507_13681_b200/libloopserve_b200.so; do
 echo "== $lib"; LS_LIB_PATH=$lib timeout 300 python tools/k1_timeline.py 2>&1 | grep -v -i warn | head -40
done > gpurun_out/ab_k1_tl.txt
[ -n "${TESTS:-}" ] && timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_c2_parity.py tests/test_gpu_parity.py tests/test_gpu_c5_parity.py tests/test_gpu_c3_parity.py -q -x 2>&1 | tail -4 > gpurun_out/ab_k1_tests.txt
exit 0
