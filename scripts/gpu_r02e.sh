#!/bin/bash
set -u
TAG=${TAG:-r02e}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
for v in ${VARIANTS:-pf0 pf1 pf2 pf2m2 pf1m2}; do
  GSE_LIB_PATH=$PWD/ab/$v.so MODES=win timeout 600 python scripts/win_ab.py > gpurun_out/winab_${TAG}_$v.json 2> gpurun_out/winab_${TAG}_$v.err
done
echo done
