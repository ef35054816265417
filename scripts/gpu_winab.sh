#!/bin/bash
# window-kernel A/B on configs[2]: parity subset per variant, then the C3 sweep per variant
set -u
TAG=${TAG:-wa}
mkdir -p gpurun_out
for v in ${VARIANTS:-base cp smallwin}; do
  GSE_LIB_PATH=$PWD/ab/$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "spmv or powerlaw or window or win or perturb" > gpurun_out/pytest_${TAG}_$v.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}_$v.log
  GSE_LIB_PATH=$PWD/ab/$v.so MODES=win timeout 600 python scripts/win_ab.py > gpurun_out/winab_${TAG}_$v.json 2> gpurun_out/winab_${TAG}_$v.err
done
echo done
