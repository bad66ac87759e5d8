#!/bin/bash
# Build ab/libmoa_<name>.so = the product with extra nvcc flags on every CUDA/C++
# source (A/B experiments): tools/build_variant.sh <name> -DFOO ...
set -e
name=$1; shift
cd "$(dirname "$0")/.."
python tools/build.py moa > /dev/null
NCCL=$(python -c "import tools.build as b; print(b._nccl_root())")
mkdir -p ab build/variant/$name
objs=""
for src in paper_2306_11148_b200/csrc/*.cu paper_2306_11148_b200/csrc/*.cpp; do
  o=build/variant/$name/$(basename $src).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I include -I paper_2306_11148_b200/csrc -I $NCCL/include "$@" -c $src -o $o &
  objs="$objs $o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs -o ab/libmoa_$name.so -L $NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL/lib -lcudart
echo ab/libmoa_$name.so
