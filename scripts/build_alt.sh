#!/bin/bash
# build_alt.sh NAME "NVCC FLAGS": an alternative libsfgpu.so for A/B runs
# (SFG_LIB=old_lib/NAME/libsfgpu.so), built from the current sources.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
OUT=$ROOT/old_lib/$NAME
mkdir -p $OUT/build
cp $ROOT/paper_2111_12238_b200/build/*.o $OUT/build/
make -s -C $ROOT/paper_2111_12238_b200 OBJ=$OUT/build NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr -Xptxas -v $*" $OUT/build/chain.o $OUT/build/fact.o $OUT/build/mline.o -B >/dev/null
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $OUT/libsfgpu.so $OUT/build/*.o
grep -A2 "k_chain_smILi8ELi4ELi12ELi8" $OUT/build/chain.ptxas.log | grep -i "spill\|registers" || true
rm -rf $OUT/build
echo built $OUT/libsfgpu.so
