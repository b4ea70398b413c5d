#!/bin/bash
# A/B timing builds: tools/build_variant.sh NAME FILE.cu [-DFLAG ...]
# recompiles one source with extra flags and links lib/libpqrr_b200_NAME.so
# next to the product library; select it with PQRR_LIB_PATH.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_1102_3828_b200/csrc
NAME=$1; SRC=$2; shift 2
make -s -C "$CS" >/dev/null
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="-O3 $ARCH -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-O3 -ccbin /usr/bin/g++ --expt-relaxed-constexpr -I$ROOT/include"
mkdir -p /tmp/pqrr_var
/usr/local/cuda/bin/nvcc $FL "$@" -c -o /tmp/pqrr_var/$NAME.o "$CS/$SRC"
OBJS=$(ls "$CS"/build/*.o | grep -v "/${SRC%.cu}.o$")
/usr/local/cuda/bin/nvcc $ARCH -shared -o "$ROOT/paper_1102_3828_b200/lib/libpqrr_b200_$NAME.so" $OBJS /tmp/pqrr_var/$NAME.o -lcudart
echo "built lib/libpqrr_b200_$NAME.so"
