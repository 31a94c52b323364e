#!/bin/bash
# Build variant libraries for kernel A/B timing (tools/ab_kernels.py):
#   tools/ab_build.sh name "-DFLAG1 -DFLAG2" ...   -> ab_libs/<name>/libulysses_b200.so
set -e
cd "$(dirname "$0")/.."
ARCH="-gencode arch=compute_100a,code=sm_100a"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  mkdir -p ab_libs/$name
  nvcc -O3 -std=c++17 -lineinfo $ARCH -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -Iinclude $flags \
    -shared -o ab_libs/$name/libulysses_b200.so paper_2309_14509_b200/csrc/*.cu -lcudart_static -ldl -lrt -lpthread &
done
wait
