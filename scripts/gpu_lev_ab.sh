set -u
mkdir -p gpurun_out
for v in ${VARIANTS:-l3dec0 l3dec2 magic}; do
  for N in ${NS:-256 512}; do
    GSE_LIB_PATH=$PWD/ab/$v.so SPMV_N=$N SPMV_VARIANT=varcoef timeout 600 python scripts/spmv_levels.py 2>/dev/null | tail -1 > gpurun_out/lev_${v}_$N.json
  done
done
GSE_LIB_PATH=$PWD/ab/magic.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "spmv or decode or level" > gpurun_out/lev_pytest.log 2>&1; echo rc=$? >> gpurun_out/lev_pytest.log
echo done
