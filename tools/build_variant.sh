#!/bin/bash
# Build an A/B variant of the library: tools/build_variant.sh NAME "-DFLAG=.. -DFLAG2=.."
# -> paper_2512_14142_b200/lib/variants/NAME/libastraea_b200.so (select with ASTRAEA_LIB=...)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
OUT=$ROOT/paper_2512_14142_b200/lib/variants/$NAME
mkdir -p $OUT $ROOT/build/variants/$NAME
cd $ROOT/paper_2512_14142_b200/csrc
for f in ${SRCS:-decode_step.cu}; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I$ROOT/include -Xcompiler -fPIC,-fvisibility=hidden --expt-relaxed-constexpr $@ -c $f -o $ROOT/build/variants/$NAME/${f%.cu}.o
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $OUT/libastraea_b200.so $(for f in kvpool attention ops gemm decode_step prefill_tc; do if [ -f $ROOT/build/variants/$NAME/$f.o ]; then echo $ROOT/build/variants/$NAME/$f.o; else echo $ROOT/build/$f.o; fi; done)
echo $OUT/libastraea_b200.so
