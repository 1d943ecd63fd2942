# decode launch-shape A/B over compile-time variants (build/ab/lib*.so, see tools/ab_lib.sh)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
for v in ${VARIANTS:-"paper_2507_13681_b200/libloopserve_b200.so X=0"}; do
  set -- $(echo $v | tr ',' ' '); echo "== $v"; env LS_LIB_PATH=$1 $2 timeout 300 python tools/dec_bench.py 2>&1 | grep -v -i warn | tail -1
done
