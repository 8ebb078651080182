#!/bin/bash
# Development aid: build libsparvar with extra -D flags into variants/lib_<name>.so
#   scripts/build_variant.sh <name> [-DFLAG ...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p variants /tmp/svobj/$name
for f in api attention predictor masks token; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include "$@" \
       -c paper_2602_04361_b200/csrc/$f.cu -o /tmp/svobj/$name/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/lib_$name.so /tmp/svobj/$name/*.o
echo variants/lib_$name.so
