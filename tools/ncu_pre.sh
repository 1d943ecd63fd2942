# ncu --set full of one turn-3 launch of each prefill kernel (C2; tools/kprof.py ONLY=prefill)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
for k in ${KERNELS:-k1_lines_kernel k1_stats_kernel greedy_kernel vs_attention_ws_kernel}; do
  env $CFG ONLY=prefill timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 1 \
    -o gpurun_out/pre_$k -f python tools/kprof.py > gpurun_out/pre_$k.log 2>&1; echo "$k rc=$?"
done
