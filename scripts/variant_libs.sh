#!/bin/bash
# build abl_libs/<name>.so: libfno with several translation units recompiled under extra -D flags
# usage: scripts/variant_libs.sh <name> "<src1.cu src2.cu ...>" -DFOO=1 ...
set -eu
NAME=$1; SRCS=$2; shift 2
B=paper_2204_01205_b200/build
NCCL_INC=$(python -c "import paper_2204_01205_b200.build as b; print(b._nccl_dirs()[0])")
NCCL_LIB=$(python -c "import paper_2204_01205_b200.build as b; print(b._nccl_dirs()[1])")
mkdir -p abl_libs /tmp/variant_$NAME
EXCL=""
pids=""
for SRC in $SRCS; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --expt-relaxed-constexpr \
    -Xcompiler -fPIC -diag-suppress 20013 -I include -I $NCCL_INC "$@" \
    -c paper_2204_01205_b200/csrc/$SRC -o /tmp/variant_$NAME/${SRC%.cu}.o &
  pids="$pids $!"
  EXCL="$EXCL|/${SRC%.cu}.o$"
done
for p in $pids; do wait $p; done
OBJS=$(ls $B/*.o | grep -vE "${EXCL#|}")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o abl_libs/$NAME.so $OBJS /tmp/variant_$NAME/*.o \
  -cudart static -L $NCCL_LIB -l:libnccl.so.2 -Xlinker -rpath=$NCCL_LIB
echo abl_libs/$NAME.so
