#!/bin/bash
O=gpurun_out/c2; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_batch.py -m gpu -q -rf > $O/pytest_batch.log 2>&1; echo "rc=$?" >> $O/pytest_batch.log
bash tools/gpu_prof_cd.sh c2
python tools/ncu_lines.py $O/solve_cfg1.ncu-rep gs_cd_blk 1 400 60 > $O/blk_lines.txt 2>&1
python tools/ncu_summary.py $O/solve_cfg1.ncu-rep > $O/blk_summary.md 2>&1
bash tools/gpu_sanitize.sh c2san
