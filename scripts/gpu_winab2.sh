set -u
mkdir -p gpurun_out
for rep in 1 2; do for v in ${VARIANTS:-m0 m1}; do
  GSE_LIB_PATH=$PWD/ab/$v.so MODES=win timeout 600 python scripts/win_ab.py > gpurun_out/wab_${v}_$rep.json 2> gpurun_out/wab_${v}_$rep.err
done; done
GSE_LIB_PATH=$PWD/ab/${PYTEST_LIB:-m1}.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "spmv or powerlaw or window or win or perturb" > gpurun_out/wab_pytest.log 2>&1; echo rc=$? >> gpurun_out/wab_pytest.log
echo done
