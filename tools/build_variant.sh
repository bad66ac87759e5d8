#!/bin/bash
# Build ab/libmoa_<name>.so = the product with extra nvcc flags on moa_dgemm.cu (A/B experiments).
set -e
name=$1; shift
cd "$(dirname "$0")/.."
python tools/build.py moa > /dev/null
NCCL=$(python -c "import tools.build as b; print(b._nccl_root())")
mkdir -p ab build/variant
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I include -I paper_2306_11148_b200/csrc -I $NCCL/include "$@" -c paper_2306_11148_b200/csrc/moa_dgemm.cu -o build/variant/moa_dgemm_$name.o
for extra in moa_host.cpp; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I include -I paper_2306_11148_b200/csrc -I $NCCL/include "$@" -c paper_2306_11148_b200/csrc/$extra -o build/variant/${extra}_$name.o; done
objs=$(ls build/moa/*.o | grep -v moa_dgemm.cu.o | grep -v moa_host.cpp.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs build/variant/moa_dgemm_$name.o build/variant/moa_host.cpp_$name.o -o ab/libmoa_$name.so -L $NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL/lib -lcudart
echo ab/libmoa_$name.so
