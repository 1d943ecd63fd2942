#!/bin/bash
# K5 A/B: per-kernel times (C2 turn 3, sparse and dense mode) for each library
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
for r in 1 2; do
for lib in ${LIBS:-build/ab/libA.so paper_2507_13681_b200/libloopserve_b200.so}; do
  LS_LIB_PATH=$lib python tools/select_timing.py 2>&1 | grep -E "sha1|vs_attention_ws"
  DENSE=1 LS_LIB_PATH=$lib python tools/select_timing.py 2>&1 | grep -E "sha1|vs_attention_ws"
done; done
