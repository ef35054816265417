#!/bin/bash
# final round validation: full GPU suite + smoke + bench + reference arm + C5 launch list,
# then compute-sanitizer memcheck over the R30 (kept direction) tests
set -u
TAG=${TAG:-f}
bash scripts/gpu_validate.sh
D=gpurun_out/sanitizer_$TAG
mkdir -p $D
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "kept_direction and not full_size" > $D/memcheck_r30.log 2>&1; echo "rc=$?" >> $D/memcheck_r30.log
echo done
