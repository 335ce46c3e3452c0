#!/bin/bash
O=gpurun_out/c18; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_path.py -m gpu -q -rf -x -k "constructors or fused_screen or blocked or cd_modes or certify or deterministic or cfg0_shape or cfg1_shape" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/time_path.py cfg1 --once > $O/cfg1.json 2> $O/cfg1.err
timeout 600 python tools/time_path.py cfg0 --once > $O/cfg0.json 2> $O/cfg0.err
timeout 300 python tools/time_screen.py cfg1 20 > $O/screen_cfg1.json 2>> $O/err.txt
timeout 600 python tools/time_screen.py cfg2 20 100000 > $O/screen_cfg2_p100k.json 2>> $O/err.txt
timeout 900 python tools/time_screen.py cfg3 20 > $O/screen_cfg3.json 2>> $O/err.txt
for ch in 1024 4096; do
GS_CD_CHUNK=$ch timeout 900 python tools/time_path.py cfg3 --once --lambdas 70 > $O/cfg3_l70_chunk$ch.json 2> $O/cfg3_chunk$ch.err
done
timeout 900 python tools/time_path.py cfg3 --once --lambdas 70 > $O/cfg3_l70_chunk2048.json 2> $O/cfg3_chunk2048.err
