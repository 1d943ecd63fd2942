python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
for hg in 1 2 4 8; do echo "== groups $hg"; LS_HEAD_GROUPS=$hg LAYERS=32 timeout 300 python tools/prof_prefill.py 2>&1 | grep -E "host enqueue"; done
