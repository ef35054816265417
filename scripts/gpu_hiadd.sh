#!/bin/bash
set -u
TAG=${TAG:-h}
mkdir -p gpurun_out
GSE_LIB_PATH=$PWD/ab/hiadd.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "spmv or powerlaw or window or win" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for v in base hiadd; do
  GSE_LIB_PATH=$PWD/ab/$v.so MODES=win timeout 600 python scripts/win_ab.py > gpurun_out/winab_${TAG}_$v.json 2> gpurun_out/winab_${TAG}_$v.err
done
echo done
