#!/bin/bash
# One measurement session: build, GPU tests, smoke, bench, C3 sweeps, other configs.
set -u
TAG=${TAG:-r01e}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi_$TAG.txt 2>&1
if [ -z "${SKIP_TESTS:-}" ]; then
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
fi
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
for s in ${EXTRA_SCRIPTS:-}; do
  timeout 1500 python scripts/$s.py > gpurun_out/${s}_$TAG.json 2> gpurun_out/${s}_$TAG.err
done
echo done
