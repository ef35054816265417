#!/bin/bash
set -u
TAG=${TAG:-r02g}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/pytest_dist_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dist_$TAG.log
timeout 900 python bench.py --steps 3 --warmup 2 --dist1 --no-cpu-baseline > gpurun_out/bench_dist1_$TAG.json 2> gpurun_out/bench_dist1_$TAG.err
timeout 900 python bench.py --steps 3 --warmup 2 --quick --no-cpu-baseline > gpurun_out/bench_quick_$TAG.json 2> gpurun_out/bench_quick_$TAG.err
echo done
