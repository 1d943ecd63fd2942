python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
for i in 1 2; do
for lib in build/ab/libA.so paper_2507_13681_b200/libloopserve_b200.so; do
  echo "== $lib $CFG"
  env LS_LIB_PATH=$lib $CFG ONLY=decode timeout 300 python tools/kprof.py 2>&1 | grep -E "decode turn|decode_kernel|rror"
done; done
