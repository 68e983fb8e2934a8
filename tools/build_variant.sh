#!/bin/bash
# Build _laud_<name>.so = the current objects with one source recompiled with extra flags.
# usage: tools/build_variant.sh <name> <source.cu> <nvcc flags...>   (then LAUD_SO_VARIANT=<name>)
set -e
name=$1; src=$2; shift 2
cd "$(dirname "$0")/.."
python -c "from paper_2308_15949_b200 import build as B; B.build()" > /dev/null
mkdir -p build/variants; objs=$(ls build/*.o | grep -v "/$(basename $src .cu).o")
srcpath=paper_2308_15949_b200/csrc/$src
[ -f "$src" ] && srcpath=$src  # a full path: an alternative copy of a csrc file (A/B of two versions)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -I include -I paper_2308_15949_b200/csrc "$@" -c $srcpath -o build/variants/$name.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $objs build/variants/$name.o \
  -o paper_2308_15949_b200/_laud_$name.so
echo paper_2308_15949_b200/_laud_$name.so
