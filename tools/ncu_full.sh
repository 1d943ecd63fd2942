#!/bin/bash
# ncu --set full captures: args are "kernel_regex:skip" pairs (1 GPU, bench C2 warm-up dialogue)
OUT=gpurun_out; mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for ks in "$@"; do
  k=${ks%%:*}; s=${ks##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c 1 \
    -o $OUT/full_${k}_$s -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $OUT/full_${k}_$s.log 2>&1
  echo "full $k skip $s rc=$?"
done
