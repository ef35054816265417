#!/bin/bash
# Round-2 session: build, GPU tests, smoke, bench, C3 window sweep, ncu of the C3 window kernel.
set -u
TAG=${TAG:-r02a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
[ "${SKIP_TESTS:-0}" = 1 ] || { timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
MODES=win timeout 600 python scripts/win_ab.py > gpurun_out/winab_$TAG.json 2> gpurun_out/winab_$TAG.err
PROF_MAT=powerlaw PROF_N=10000000 PROF_CG_ITERS=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_spmv_win -c 4 -o gpurun_out/prof_c3_$TAG python scripts/prof_spmv.py > gpurun_out/prof_c3_$TAG.log 2>&1
echo done
