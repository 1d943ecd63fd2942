# decode step time by kind for several launch shapes (tools/dec_bench.py)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
CFGS=${CFGS:-"X=0|LS_K6_SIMT=1"}
IFS='|'
for cfg in $CFGS; do
  echo "== $cfg"
  IFS=' ' env $cfg timeout 300 python tools/dec_bench.py 2>&1 | grep -vi warn | tail -2
done
