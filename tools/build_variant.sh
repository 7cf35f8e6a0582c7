#!/bin/bash
# Build liblbfs with extra -D flags into _native/variants/<name>.so (A/B
# experiments, selected at run time with LBFS_LIB=<path>).
#   tools/build_variant.sh w16c512 -DLBFS_EXPAND_WARPS=16 -DLBFS_WARP_CHUNK=512
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_1604_02844_b200/csrc
OUT=$ROOT/paper_1604_02844_b200/_native/variants
OBJ=$OUT/obj_$NAME
mkdir -p $OBJ
NCCL_INC=$(python3 -c "import nvidia.nccl, os; print(os.path.join(list(nvidia.nccl.__path__)[0], \"include\"))")
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$ROOT/include -I$NCCL_INC --expt-relaxed-constexpr $*"
for f in api bfs bottomup cluster construct layout multi partition stream sweep validate; do
  $NV -c $SRC/$f.cu -o $OBJ/$f.o -Xptxas -v 2> $OBJ/$f.ptxas.log &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/$NAME.so $OBJ/*.o --cudart static -ldl
echo "$OUT/$NAME.so"
