#!/bin/bash
# compute-sanitizer over the round-2 code paths (device plan, captured NCCL graphs, R29 xpay
# reduction, gse_spmv_dot, window kernel decode, allocator hook), racecheck on the window and
# row-walk kernels.  Output under gpurun_out/sanitizer_$TAG/
set -u
TAG=${TAG:-s}
D=gpurun_out/sanitizer_$TAG
mkdir -p $D
CS=/usr/local/cuda/bin/compute-sanitizer
K1="perturb or spmv_dot or allocator or max_level or window or win or k_sweep or sampled_bit"
timeout 2400 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "$K1" > $D/memcheck_parity.log 2>&1; echo "rc=$?" >> $D/memcheck_parity.log
timeout 1800 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_dist.py -q -x -k "not multi_rank and not graph_capture" > $D/memcheck_dist.log 2>&1; echo "rc=$?" >> $D/memcheck_dist.log
timeout 1800 $CS --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "spmv_levels_parity or window" > $D/racecheck_spmv.log 2>&1; echo "rc=$?" >> $D/racecheck_spmv.log
echo done
