#!/bin/bash
# Sanity session after a restore: GPU tests, smoke, bench, C3 sweep, ncu capture of the SP kernel on C3.
set -u
TAG=${TAG:-r01d}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 python scripts/sweep_c3.py > gpurun_out/c3_$TAG.json 2> gpurun_out/c3_$TAG.err
PROF_MAT=powerlaw PROF_N=${PROF_N:-10000000} PROF_CG_ITERS=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_spmv -c 4 -o gpurun_out/prof_c3_$TAG python scripts/prof_spmv.py > gpurun_out/prof_c3_$TAG.log 2>&1
echo done
