#!/bin/bash
O=gpurun_out/c8; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_path.py -m gpu -q -rf -k "fused_screen or cfg2_generator or sparse or screen_matches or rules_match or elastic or tail" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python tools/time_screen.py cfg3 20 > $O/screen_cfg3.json 2> $O/screen_cfg3.err
timeout 1200 python tools/time_path.py cfg3 --once --lambdas 40 > $O/cfg3_l40_chunk.json 2> $O/cfg3_l40_chunk.err
GS_CD_CHUNK=0 timeout 1200 python tools/time_path.py cfg3 --once --lambdas 40 > $O/cfg3_l40_nochunk.json 2> $O/cfg3_l40_nochunk.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -s 88 -c 1 -o $O/solve_cfg1_l88 -f \
   python tools/prof_path.py cfg1 92 > $O/ncu_solve.log 2>&1; echo "ncu solve rc=$?" >> $O/ncu_solve.log
python tools/ncu_lines.py $O/solve_cfg1_l88.ncu-rep gs_cd_blk 1 500 70 > $O/blk_lines_l88.txt 2>&1
python tools/ncu_summary.py $O/solve_cfg1_l88.ncu-rep > $O/blk_summary_l88.md 2>&1
