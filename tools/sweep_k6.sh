# K6 decode launch-shape sweep (diagnostics): per-kernel means of a C2 turn-3 decode
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
CFGS=${CFGS:-"X=0|LS_K6_CTAS_PER_SM=4|LS_K6_CTAS_PER_SM=1|LS_K6_CLUSTER=1|LS_K6_SPLIT_COMP=17|LS_K6_SPLIT_COMP=8 LS_K6_CLUSTER=1"}
IFS='|'
for cfg in $CFGS; do
  echo "== $cfg"
  IFS=' ' env $cfg ONLY=decode timeout 300 python tools/kprof.py 2>&1 | grep -E "decode turn|decode_|Error|error"
done
