#!/bin/bash
# A/B build: recompile ONE csrc file with extra -D flags and link it with the
# other in-tree objects into build/variants/<name>.so (load with FQ_LIB=...).
# Usage: bash scripts/build_variant.sh <name> <file.cu> [-DFOO=1 ...]
set -e
N=$1; F=$2; shift 2
cd "$(dirname "$0")/.."
python -m paper_2010_13887_b200.build > /dev/null
mkdir -p build/variants
B=$(basename $F .cu)
SRC=paper_2010_13887_b200/csrc/$F
[ -f "$F" ] && SRC=$F  # a path: e.g. an older revision of a csrc file (same basename)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I include -I paper_2010_13887_b200/csrc "$@" \
  -c $SRC -o build/variants/$N.$B.o
OBJS=$(ls build/obj/*.o | grep -v "/$B.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/$N.so $OBJS \
  build/variants/$N.$B.o -lcudart -ldl
echo build/variants/$N.so
