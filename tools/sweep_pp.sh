python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
for v in "paper_2507_13681_b200/libloopserve_b200.so X=0" "build/ab/libpp_4_2.so LS_K6_SPLIT_COMP=4" "build/ab/libpp_4_2.so LS_K6_SPLIT_COMP=5" "build/ab/libpp_2_2.so X=0" "build/ab/libpp_2_2.so LS_K6_SPLIT_COMP=8"; do
  set -- $v; echo "== $v"; env LS_LIB_PATH=$1 $2 timeout 300 python tools/dec_bench.py 2>&1 | grep -v -i warn | tail -1
done
