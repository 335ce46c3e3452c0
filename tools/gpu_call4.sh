#!/bin/bash
O=gpurun_out/c4; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_path.py -m gpu -q -rf -x -k "fused_screen or cfg2_generator or sparse or screen_matches" > $O/pytest_gemv.log 2>&1; echo "rc=$?" >> $O/pytest_gemv.log
timeout 600 python tools/time_screen.py cfg2 20 100000 > $O/screen_cfg2_p100k.json 2> $O/screen_cfg2.err
GS_GEMV_WIDE=0 timeout 600 python tools/time_screen.py cfg2 20 100000 > $O/screen_cfg2_p100k_old.json 2>> $O/screen_cfg2.err
timeout 900 python tools/time_screen.py cfg3 20 > $O/screen_cfg3.json 2> $O/screen_cfg3.err
GS_CSC_SHORT=0 timeout 900 python tools/time_screen.py cfg3 20 > $O/screen_cfg3_old.json 2>> $O/screen_cfg3.err
timeout 300 python tools/time_screen.py cfg1 20 > $O/screen_cfg1.json 2> $O/screen_cfg1.err
timeout 600 python tools/time_path.py cfg1 --once --per-lambda > $O/cfg1_perlam.json 2> $O/cfg1_perlam.err
