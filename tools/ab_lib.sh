#!/bin/bash
# Build an A/B variant of the C-ABI library with one source file taken from a
# git revision: tools/ab_lib.sh <rev> <file.cu> <out.so>  (diagnostics only)
set -e
REV=$1; F=$2; OUT=$3
C=paper_2507_13681_b200/csrc
mkdir -p build/ab
git show $REV:$C/$F > build/ab/$F
cp $C/*.cuh build/ab/
OBJS=""
for s in capi sampler score_lines score_lines_tc select_lines vs_attention vs_attention_ws decode; do
  if [ "$s.cu" = "$F" ]; then
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      --expt-relaxed-constexpr -Iinclude -I$C -c build/ab/$F -o build/ab/${s}.o
    OBJS="$OBJS build/ab/${s}.o"
  else
    OBJS="$OBJS build/obj/${s}.o"
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT $OBJS -lcudart
echo built $OUT
