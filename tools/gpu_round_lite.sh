#!/bin/bash
# GPU tests, bench, launch list and the screening-pass capture, summarised ON
# THE BOX (the .ncu-rep files are deleted: gpurun copies back <= 64 MiB).
TAG=${1:-r01}; STEPS=${2:-2}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --steps $STEPS --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $O/ncu_launch.log
python tools/ncu_summary.py --launches $O/launches.csv > $O/launches.md 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_screen_full -s 2 -c 1 -o /tmp/screen_full -f \
   python tools/time_screen.py cfg1 3 > $O/ncu_screen.log 2>&1; echo "ncu screen rc=$?" >> $O/ncu_screen.log
python tools/ncu_summary.py /tmp/screen_full.ncu-rep > $O/ncu_screen_full.md 2>&1
