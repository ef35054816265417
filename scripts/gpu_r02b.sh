#!/bin/bash
# bench (C5 default) + new tests + ncu of the C5 dominant kernel
set -u
TAG=${TAG:-r02b}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_bench_contract.py -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 1500 python bench.py --steps 3 --warmup 2 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
[ "${SKIP_PROF:-0}" = 1 ] || PROF_N=512 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_rw -c 4 -o gpurun_out/prof_c5_$TAG python scripts/prof_c5.py > gpurun_out/prof_c5_$TAG.log 2>&1
echo done
