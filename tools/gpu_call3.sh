#!/bin/bash
O=gpurun_out/c3; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_batch.py -m gpu -q -rf > $O/pytest_batch.log 2>&1; echo "rc=$?" >> $O/pytest_batch.log
for mf in 32 128; do
GS_BLK_MFAC=$mf GS_CD_PROF=1 timeout 600 python tools/time_path.py cfg1 --once > $O/cfg1_mf$mf.json 2> $O/cfg1_mf$mf.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -s 88 -c 1 -o $O/solve_cfg1_l88 -f \
   python tools/prof_path.py cfg1 92 > $O/ncu_solve.log 2>&1; echo "ncu solve rc=$?" >> $O/ncu_solve.log
python tools/ncu_lines.py $O/solve_cfg1_l88.ncu-rep gs_cd_blk 1 400 60 > $O/blk_lines_l88.txt 2>&1
python tools/ncu_summary.py $O/solve_cfg1_l88.ncu-rep > $O/blk_summary_l88.md 2>&1
