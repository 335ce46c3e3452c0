#!/bin/bash
O=gpurun_out/c5; mkdir -p $O
GS_CD_PROF=1 timeout 600 python tools/time_path.py cfg1 --once --lambdas 80 > $O/cfg1_prof.txt 2> $O/cfg1_prof.err
GS_CD_PROF=1 timeout 600 python tools/time_path.py cfg0 --once --lambdas 60 > $O/cfg0_prof.txt 2> $O/cfg0_prof.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_screen_full -s 2 -c 1 -o $O/screen_cfg2 -f \
   python tools/time_screen.py cfg2 3 100000 > $O/ncu_screen_cfg2.log 2>&1; echo "rc=$?" >> $O/ncu_screen_cfg2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_screen_full -s 2 -c 1 -o $O/screen_cfg3 -f \
   python tools/time_screen.py cfg3 3 > $O/ncu_screen_cfg3.log 2>&1; echo "rc=$?" >> $O/ncu_screen_cfg3.log
for c in cfg2 cfg3; do
python tools/ncu_summary.py $O/screen_$c.ncu-rep > $O/screen_${c}_summary.md 2>&1
python tools/ncu_lines.py $O/screen_$c.ncu-rep gs_solve.cuh 270 520 40 > $O/screen_${c}_lines.txt 2>&1
done
