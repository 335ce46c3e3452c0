#!/bin/bash
# One GPU-box session: gpu tests, bench, ncu launch list, ncu full captures.
# usage: tools/gpu_round.sh TAG [steps]
TAG=${1:-r01}; STEPS=${2:-2}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps $STEPS --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $O/ncu_launch.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_screen_full -s 2 -c 1 -o $O/screen_full -f \
   python tools/time_screen.py cfg1 3 > $O/ncu_screen.log 2>&1; echo "ncu screen rc=$?" >> $O/ncu_screen.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -s 40 -c 1 -o $O/solve_cfg1 -f \
   python tools/prof_path.py cfg1 45 > $O/ncu_solve.log 2>&1; echo "ncu solve rc=$?" >> $O/ncu_solve.log
