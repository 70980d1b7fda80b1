#!/bin/bash
# Developer helper: a variant that differs from tools/bin/dev only in ONE .cu file
# (tools/build_one_variant.sh <name> <file-stem> [nvcc flags...]); tools/bin/dev must exist.
set -e
name=$1; stem=$2; shift 2
d="tools/bin/${name:?name}"
mkdir -p "$d"
cp tools/bin/dev/*.o "$d"/
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \
  -I include -I paper_2401_03365_b200/csrc --expt-relaxed-constexpr -DPCSB_DEV_KNOBS -Xptxas -v "$@" \
  -c paper_2401_03365_b200/csrc/$stem.cu -o "$d/$stem.o" 2> "$d/$stem.ptxas.log"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$d/libpcs_lop_b200.so" \
  "$d"/{grid_sort,lop_fast,lop_exact,plan,comm,c_api,nn,io,mls}.o \
  paper_2401_03365_b200/build/{nccl_dl,generators,pcs_api,shard,host_io,mls_api}.o -ldl -lgomp
