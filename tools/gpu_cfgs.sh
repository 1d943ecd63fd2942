#!/bin/bash
# extra-config benches + ncu captures of the prefill kernels (one gpurun call)
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for c in ${CFGS:-c4 c3 c5}; do
  timeout 900 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "$c rc=$?"; tail -c 600 $OUT/bench_$c.json; tail -2 $OUT/bench_$c.err
done
