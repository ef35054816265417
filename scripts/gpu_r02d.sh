#!/bin/bash
# full GPU tests, smoke, the stepped-solver R29 sweep
set -u
TAG=${TAG:-r02d}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python scripts/stepped_time.py > gpurun_out/stepped_$TAG.json 2> gpurun_out/stepped_$TAG.err
echo done
