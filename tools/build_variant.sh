#!/bin/sh
# Build an instrumented / A-B variant of the native library into tools/ab/<name>.so
# reusing the in-tree objects for every file except qx_tc.cu and qx_ntt.cu when
# listed: tools/build_variant.sh <name> "<nvcc defines>" [sources...]
# Load it with QX_NATIVE_LIB=tools/ab/<name>.so.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; DEFS=$2; shift 2
SRCS=${*:-qx_tc.cu}
C=$ROOT/paper_2509_19974_b200/csrc
OUT=$ROOT/tools/ab/$NAME
mkdir -p $OUT
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DQX_NTT_THREADS=512 -DQX_NTT_MAXR=5 -Xcompiler -fPIC,-ffp-contract=off --expt-relaxed-constexpr -I$ROOT/include -I$(python3 -c "import nvidia.nccl as m; print(list(m.__path__)[0] + '/include')") $DEFS"
OBJS=""
for f in qx_abi.cu qx_ntt.cu qx_quant.cu qx_tc.cu qx_tc_i8.cu qx_popc.cu qx_dist.cu; do
  o=$C/build/${f%.cu}.o
  case " $SRCS " in *" $f "*) o=$OUT/${f%.cu}.o; $NV -c $C/$f -o $o;; esac
  OBJS="$OBJS $o"
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/tools/ab/$NAME.so $OBJS -cudart static -ldl -Xlinker --exclude-libs,ALL
echo built tools/ab/$NAME.so
