#!/bin/bash
# GPU-box check: the gpu test suite (no -x: every failure listed) and a short
# bench line with its parity block.   usage: tools/gpu_check.sh TAG [steps] [pytest-args]
TAG=${1:-r02}; STEPS=${2:-1}; shift 2; PYARGS=${@:-tests}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest $PYARGS -m gpu -q -rf --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
if [ "$STEPS" != "0" ]; then
timeout 900 python bench.py --steps $STEPS --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
fi
