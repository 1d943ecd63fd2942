#!/bin/bash
# compute-sanitizer runs on a small workload of every kernel family (tools/san_small.py)
#  memcheck / racecheck: every kernel
#  synccheck: every kernel except the mbarrier-pipelined tcgen05 kernels, whose
#  protocols observe some mbarrier phases lazily (synccheck's "missing wait";
#  see profiles/r2_sanitizers.md)
OUT=gpurun_out; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
rm -f $OUT/san_summary.txt
for tool in memcheck racecheck; do
  timeout 1500 $CS --tool $tool --print-limit 20 python tools/san_small.py > $OUT/san_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/san_summary.txt
  tail -3 $OUT/san_$tool.log >> $OUT/san_summary.txt
done
timeout 1500 $CS --tool synccheck --print-limit 20 \
  --kernel-name-exclude kns=vs_attention_ws_kernel --kernel-name-exclude kns=k1_stats_kernel \
  --kernel-name-exclude kns=k1_lines_kernel --kernel-name-exclude kns=greedy_kernel \
  --kernel-name-exclude kns=decode_mma_kernel \
  python tools/san_small.py > $OUT/san_synccheck.log 2>&1
echo "synccheck (excl. mbarrier pipelines) rc=$?" >> $OUT/san_summary.txt
tail -3 $OUT/san_synccheck.log >> $OUT/san_summary.txt
