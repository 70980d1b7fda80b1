#!/bin/bash
# Developer helper: builds an experimental variant of the library into
# tools/bin/<name>/ with extra nvcc flags (e.g. -DPCSB_HR=96).  Variants read
# the PCSB_* developer knobs (-DPCSB_DEV_KNOBS); the shipped library does not.
set -e
name=$1; shift
d="tools/bin/${name:?name}"
mkdir -p "$d"
for f in grid_sort lop_fast lop_exact plan comm c_api nn io mls; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \
    -I include -I paper_2401_03365_b200/csrc --expt-relaxed-constexpr -DPCSB_DEV_KNOBS "$@" \
    -c paper_2401_03365_b200/csrc/$f.cu -o "$d/$f.o" &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$d/libpcs_lop_b200.so" \
  "$d"/{grid_sort,lop_fast,lop_exact,plan,comm,c_api,nn,io,mls}.o \
  paper_2401_03365_b200/build/{nccl_dl,generators,pcs_api,shard,host_io,mls_api}.o -ldl -lgomp
