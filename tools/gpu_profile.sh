#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (both arms), the ncu launch list of one
# C2 turn-3 prefill + decode (tools/one_turn.py) and ncu --set full captures of
# the top kernels on the same workload. Each stage has its own timeout.
set -u
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
OURS='^(sample_rows|k1_|sort_prefix|sort_block|greedy|plan_bits|compact_bits|gather_vert|vert_bits|reverse_bits|vs_attention|plan_scores|plan_norm|decode_mma|advance_kernel|select_kernel|select_ws_kernel|compact_kernel|set_bits)'
# the ncu stages profile the kernels as bench.py's per-entry breakdown runs them:
# one launch per layer, without the head-group K3/K5 overlap
NCU_ENV="LS_K5_OVERLAP_MIN=100000000"
for s in ${STAGES:-tests smoke bench ref launches full}; do
  case $s in
    tests) timeout 1500 python -m pytest tests -m gpu -q > $OUT/tests_gpu.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests_gpu.log;;
    smoke) timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log;;
    bench) timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 400 $OUT/bench.json;;
    ref) timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"; tail -c 300 $OUT/bench_ref.json;;
    launches) env $NCU_ENV timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:$OURS" --csv \
                --log-file $OUT/launches.csv python tools/one_turn.py > $OUT/launches.log 2>&1; echo "launches rc=$?";;
    full)
      for ks in "vs_attention_ws_kernel 8" "k1_lines_kernel 8" "k1_stats_kernel 8" "greedy_kernel 16" "sort_prefix_kernel 8" \
                "decode_mma_kernel 200" "decode_mma_kernel 1500" "select_ws_kernel 2" "select_kernel 2" "compact_kernel 2"; do
        set -- $ks
        env $NCU_ENV timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 \
          -o $OUT/full_${1}_$2 -f python tools/one_turn.py > $OUT/full_${1}_$2.log 2>&1; echo "full $1 $2 rc=$?"
      done;;
  esac
done
