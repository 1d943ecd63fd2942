#!/bin/bash
# Build an A/B variant of the C-ABI library (diagnostics only):
#   tools/ab_lib.sh <rev|WORK> <file.cu> <out.so> [extra nvcc flags...]
# one source file is taken from git revision <rev> (or the working tree for
# WORK) and compiled with the extra flags; every other object is the current build.
set -e
REV=$1; F=$2; OUT=$3; shift 3
C=paper_2507_13681_b200/csrc
mkdir -p build/ab
if [ "$REV" = "WORK" ]; then cp $C/$F build/ab/$F; else git show $REV:$C/$F > build/ab/$F; fi
cp $C/*.cuh build/ab/
OBJS=""
for s in capi sampler score_lines score_lines_tc select_lines vs_attention vs_attention_ws decode dropin_ops; do
  if [ "$s.cu" = "$F" ]; then
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      --expt-relaxed-constexpr -Iinclude -I$C "$@" -c build/ab/$F -o build/ab/${s}_$(basename $OUT .so).o
    OBJS="$OBJS build/ab/${s}_$(basename $OUT .so).o"
  else
    OBJS="$OBJS build/obj/${s}.o"
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT $OBJS -lcudart
echo built $OUT
