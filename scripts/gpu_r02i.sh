#!/bin/bash
set -u
mkdir -p gpurun_out
for v in base rw4; do GSE_LIB_PATH=$PWD/ab/$v.so timeout 900 python scripts/rw_ab_c5.py > gpurun_out/rwab_c5_$v.json 2> gpurun_out/rwab_c5_$v.err; done
PROF_MAT=powerlaw PROF_N=10000000 PROF_CG_ITERS=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_spmv_win -c 4 -o gpurun_out/prof_c3_r02i python scripts/prof_spmv.py > gpurun_out/prof_c3_r02i.log 2>&1
TAG=r02i bash scripts/gpu_sanitize.sh
echo done
