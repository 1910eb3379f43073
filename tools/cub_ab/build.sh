#!/bin/bash
# CUB SortPairs baseline for tools/k12_scale.py (library comparison only)
cd "$(dirname "$0")" && /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode=arch=compute_100a,code=sm_100a \
  -shared -Xcompiler -fPIC -o libcub_sort.so cub_sort.cu
