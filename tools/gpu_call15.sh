#!/bin/bash
O=gpurun_out/c15; mkdir -p $O
for v in "1 1" "0 1" "1 0" "0 0"; do set -- $v
GS_L2_HINT=$1 GS_LDS_EXPLICIT=$2 timeout 300 python tools/time_screen.py cfg1 20 > $O/screen_cfg1_h$1_l$2.json 2>> $O/err.txt
done
for h in 1 0; do
GS_L2_HINT=$h timeout 600 python tools/time_screen.py cfg2 20 100000 > $O/screen_cfg2_h$h.json 2>> $O/err.txt
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_screen_full -s 2 -c 1 -o $O/screen_cfg3 -f \
   python tools/time_screen.py cfg3 3 > $O/ncu_screen_cfg3.log 2>&1; echo "rc=$?" >> $O/ncu_screen_cfg3.log
python tools/ncu_summary.py $O/screen_cfg3.ncu-rep > $O/screen_cfg3_summary.md 2>&1
python tools/ncu_lines.py $O/screen_cfg3.ncu-rep gs_solve.cuh 400 900 40 > $O/screen_cfg3_lines.txt 2>&1
