#!/bin/bash
# Blocked-chain CD consumer on the B200: microbenchmarks, targeted parity
# tests, and path times per consumer mode.   usage: tools/gpu_blk.sh TAG
TAG=${1:-blk}; O=gpurun_out/$TAG; mkdir -p $O
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ubench_fp64 tools/ubench_fp64.cu && /tmp/ubench_fp64 > $O/ubench.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_path.py tests/test_gpu_kernels.py -m gpu -q -rf -x \
    -k "blocked or cd_modes or certify or cfg0_full or cd_pass or stress or cfg1_shape" > $O/pytest_blk.log 2>&1
echo "pytest rc=$?" >> $O/pytest_blk.log
for mode in 2 0; do
  GS_CD_GRAM=$mode timeout 600 python tools/time_path.py cfg1 --once > $O/cfg1_mode$mode.json 2> $O/cfg1_mode$mode.err
done
for mode in 2 1; do
  GS_CD_GRAM=$mode timeout 300 python tools/time_path.py cfg0 --once > $O/cfg0_mode$mode.json 2> $O/cfg0_mode$mode.err
done
