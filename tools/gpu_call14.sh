#!/bin/bash
O=gpurun_out/c14; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_path.py -m gpu -q -rf -x -k "fused_screen or cfg2_generator or sparse or screen_matches or blocked or cd_modes or certify or deterministic or cfg0_shape" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/time_path.py cfg1 --once --per-lambda > $O/cfg1.json 2> $O/cfg1.err
GS_CD_GRAM=0 timeout 600 python tools/time_path.py cfg1 --once > $O/cfg1_direct.json 2> $O/cfg1_direct.err
timeout 600 python tools/time_path.py cfg0 --once > $O/cfg0.json 2> $O/cfg0.err
timeout 900 python tools/time_screen.py cfg3 20 > $O/screen_cfg3.json 2> $O/screen_cfg3.err
GS_CSC_FLAT=0 timeout 900 python tools/time_screen.py cfg3 20 > $O/screen_cfg3_noflat.json 2> $O/screen_cfg3.err
timeout 300 python tools/time_screen.py cfg1 20 > $O/screen_cfg1.json 2> $O/screen_cfg1.err
timeout 600 python tools/time_screen.py cfg2 20 100000 > $O/screen_cfg2_p100k.json 2> $O/screen_cfg2.err
