# per-kernel times of one C2 turn-3 prefill for each library in $LIBS (A/B diagnostics)
mkdir -p gpurun_out
for i in 1 2; do for lib in $LIBS; do
 LS_LIB_PATH=$lib timeout 300 python tools/select_timing.py 2>&1 | grep -v -i warn | head -${TOP:-6}
done; done > gpurun_out/ab_multi.txt
exit 0
