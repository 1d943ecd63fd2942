# ncu --set full of one dense and one compressed K6 launch (C2 turn-3 decode)
# env: CFGS="cfgA|cfgB" (env assignments per capture), SKIPS (launch skips)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
CFGS=${CFGS:-"X=0"}
IFS='|'
n=0
for cfg in $CFGS; do
  n=$((n+1))
  for sk in ${SKIPS:-200 1500}; do
    IFS=' ' env $cfg ONLY=decode timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_ -s $sk -c 1 \
      -o gpurun_out/dec_c${n}_$sk -f python tools/kprof.py > gpurun_out/dec_c${n}_$sk.log 2>&1; echo "c$n ($cfg) $sk rc=$?"
  done
done
