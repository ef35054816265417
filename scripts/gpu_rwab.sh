#!/bin/bash
# row-walk A/B: parity subset per variant, C5 SpMV + CG (rw_ab_c5.py) and C2 per variant
set -u
TAG=${TAG:-ra}
mkdir -p gpurun_out
for v in ${VARIANTS:-base rwh}; do
  GSE_LIB_PATH=$PWD/ab/$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "spmv or poisson or cg_parity or dot" > gpurun_out/pytest_${TAG}_$v.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}_$v.log
  GSE_LIB_PATH=$PWD/ab/$v.so timeout 900 python scripts/rw_ab_c5.py > gpurun_out/rwab_${TAG}_$v.json 2> gpurun_out/rwab_${TAG}_$v.err
  GSE_LIB_PATH=$PWD/ab/$v.so PROF_N=128 timeout 900 python scripts/rw_ab_c5.py > gpurun_out/rwab_c2_${TAG}_$v.json 2>> gpurun_out/rwab_${TAG}_$v.err
done
echo done
