#!/bin/bash
O=gpurun_out/c12; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for h in 1 0; do
GS_L2_HINT=$h GS_CD_PROF=1 timeout 600 python tools/time_path.py cfg1 --once > $O/cfg1_h$h.txt 2> $O/cfg1_h$h.err
done
timeout 600 python tools/time_path.py cfg0 --once > $O/cfg0.json 2> $O/cfg0.err
timeout 900 python tools/time_screen.py cfg3 20 > $O/screen_cfg3.json 2> $O/screen_cfg3.err
timeout 300 python tools/time_screen.py cfg1 20 > $O/screen_cfg1.json 2> $O/screen_cfg1.err
GS_LDS_EXPLICIT=0 timeout 300 python tools/time_screen.py cfg1 20 > $O/screen_cfg1_l0.json 2> $O/screen_cfg1.err
