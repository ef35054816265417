#!/bin/bash
# window-kernel A/B: parity tests on the in-tree build, C3 sweep per variant, ncu of the in-tree kernel
set -u
TAG=${TAG:-w}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "spmv or powerlaw or window or win or decode" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for v in ${VARIANTS:-win_old win_st win_st3}; do
  GSE_LIB_PATH=$PWD/ab/$v.so MODES=win timeout 600 python scripts/win_ab.py > gpurun_out/winab_${TAG}_$v.json 2> gpurun_out/winab_${TAG}_$v.err
done
[ "${SKIP_PROF:-0}" = 1 ] || PROF_MAT=powerlaw PROF_N=10000000 PROF_CG_ITERS=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_spmv_win -c 4 -o gpurun_out/prof_c3_$TAG python scripts/prof_spmv.py > gpurun_out/prof_c3_$TAG.log 2>&1
echo done
