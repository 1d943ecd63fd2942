#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (both arms), ncu launch list and
# full captures of the top kernels. Each stage is bounded by its own timeout.
# usage: tools/gpu_round.sh [stages...]   stages: tests smoke bench ref launches full
set -u
OUT=gpurun_out
mkdir -p $OUT
STAGES="${@:-tests smoke bench launches full}"
OURS='^(sample_rows|k1_|score_lines|sort_lines|sort_keys|sort_scatter|greedy|chain_kernel|cross_kernel|finalize_kernel|load_lists|row_of|set_bits|compact_bits|plan_bits|vert_bits|reverse_bits|gather_vert|vs_attention|plan_rows|plan_scores|plan_norm|decode_kernel|decode_mma_kernel|DeviceRadixSort|advance_kernel|select_kernel|compact_kernel|total_kernel|reduce_kernel)'

nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
python -c 'import __graft_entry__ as g; g.build()' > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for s in $STAGES; do
  case $s in
    tests)  timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/tests_gpu.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests_gpu.log;;
    smoke)  timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log;;
    bench)  timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 3000 $OUT/bench.json; tail -5 $OUT/bench.err;;
    benchq) timeout 600 python bench.py --no-cpu-baseline --no-dense > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 3000 $OUT/bench.json; tail -5 $OUT/bench.err;;
    ref)    timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"; cat $OUT/bench_ref.json; tail -3 $OUT/bench_ref.err;;
    launches) timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:$OURS" --csv \
                --log-file $OUT/launches.csv python tools/one_turn.py > $OUT/launches.log 2>&1; echo "launches rc=$?"; tail -2 $OUT/launches.log;;
    kprof)  timeout 600 python tools/kprof.py > $OUT/kprof.log 2>&1; echo "kprof rc=$?"; cat $OUT/kprof.log | grep -v Warning | head -70;;
    prof)   timeout 600 python tools/prof_prefill.py > $OUT/prof_prefill.log 2>&1; echo "prof rc=$?"; head -40 $OUT/prof_prefill.log;;
    full)   for k in ${FULL_KERNELS:-vs_attention_ws_kernel k1_lines_kernel k1_stats_kernel decode_kernel select_kernel greedy_kernel}; do
              timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 2 \
                -o $OUT/prof_$k -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
                > $OUT/prof_$k.log 2>&1; echo "full $k rc=$?"; done;;
  esac
done
