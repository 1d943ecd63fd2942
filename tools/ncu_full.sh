#!/bin/bash
# ncu --set full captures: args are "kernel_regex:skip" pairs (1 GPU; workload: tools/one_turn.py, C2 turn 3)
OUT=gpurun_out; mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for ks in "$@"; do
  k=${ks%%:*}; s=${ks##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c 1 \
    -o $OUT/full_${k}_$s -f python ${WORKLOAD:-tools/one_turn.py} > $OUT/full_${k}_$s.log 2>&1
  echo "full $k skip $s rc=$?"
done
