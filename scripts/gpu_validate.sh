#!/bin/bash
# full GPU tests + smoke, the default bench line, the reference arm, the C5 launch list
set -u
TAG=${TAG:-v}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
T0=$(date +%s); timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench_s=$(( $(date +%s) - T0 ))" >> gpurun_out/bench_$TAG.err
T0=$(date +%s); timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref_s=$(( $(date +%s) - T0 ))" >> gpurun_out/bench_ref_$TAG.err
GSE_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 500 --csv --log-file gpurun_out/launches_c5_$TAG.csv \
  python bench.py --steps 1 --warmup 0 --quick --no-e2e --no-cpu-baseline --no-sweep > /dev/null 2>&1
echo done
