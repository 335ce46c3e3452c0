#!/bin/bash
O=gpurun_out/c17; mkdir -p $O
timeout 300 python tools/time_screen.py cfg1 20 > $O/screen_cfg1.json 2>> $O/err.txt
timeout 600 python tools/time_screen.py cfg2 20 100000 > $O/screen_cfg2_p100k.json 2>> $O/err.txt
timeout 900 python tools/time_screen.py cfg3 20 > $O/screen_cfg3.json 2>> $O/err.txt
timeout 2400 python tools/run_cfg2_full.py 1000000 > $O/cfg2_full.json 2> $O/cfg2_full.err; echo "rc=$?" >> $O/cfg2_full.err
