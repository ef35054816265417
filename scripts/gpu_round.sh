#!/bin/bash
# One GPU session: tests, smoke, bench, launch list, full ncu capture of the dominant kernel.
# Output under gpurun_out/ (scratch); summaries are copied into profiles/ afterwards.
set -u
TAG=${TAG:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
# launch list of the same workload (host-driven CG so ncu can see the kernels)
GSE_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-sweep > /dev/null 2>&1
# full capture of the dominant kernel (level-1 SpMV of the CG: DOT variant) + levels 2/3
PROF_CG_ITERS=4 GSE_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_spmv -c 5 -o gpurun_out/prof_$TAG python scripts/prof_spmv.py > gpurun_out/prof_$TAG.log 2>&1
echo done-c2
# the strided-products kernel on configs[2] (power-law, 10M rows)
PROF_MAT=powerlaw PROF_N=10000000 PROF_CG_ITERS=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_spmv_sp -c 4 -o gpurun_out/prof_c3_$TAG python scripts/prof_spmv.py > gpurun_out/prof_c3_$TAG.log 2>&1
echo done-c3
