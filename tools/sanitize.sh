#!/bin/bash
# compute-sanitizer runs (memcheck, racecheck, synccheck) on a small workload of every kernel family
OUT=gpurun_out; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --print-limit 20 python tools/san_small.py > $OUT/san_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/san_summary.txt
  tail -3 $OUT/san_$tool.log >> $OUT/san_summary.txt
done
