#!/bin/bash
# Round-2 evidence on one B200: full GPU suite, bench (ours + reference arm),
# ncu launch list, ncu --set full captures (screens of cfg1/cfg2/cfg3, one
# late-lambda solve of cfg1), other-config path times.   usage: tools/gpu_round_r02.sh TAG
TAG=${1:-r02d}; O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 1500 python bench.py --impl reference --steps 1 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?" >> $O/bench_reference.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $O/ncu_launch.log
for c in "cfg1 " "cfg2 100000" "cfg3 "; do set -- $c
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_screen_full -s 2 -c 1 -o $O/screen_$1 -f \
   python tools/time_screen.py $1 3 $2 > $O/ncu_screen_$1.log 2>&1; echo "rc=$?" >> $O/ncu_screen_$1.log
python tools/ncu_summary.py $O/screen_$1.ncu-rep > $O/ncu_screen_full_$1.md 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -s 88 -c 1 -o $O/solve_cfg1 -f \
   python tools/prof_path.py cfg1 92 > $O/ncu_solve.log 2>&1; echo "ncu solve rc=$?" >> $O/ncu_solve.log
python tools/ncu_summary.py $O/solve_cfg1.ncu-rep > $O/ncu_solve_cfg1_late_lambda.md 2>&1
python tools/ncu_lines.py $O/solve_cfg1.ncu-rep gs_cd_blk 1 500 50 > $O/ncu_solve_cfg1_blk_lines.txt 2>&1
timeout 600 python tools/time_batch.py 256 > $O/cfg4_256.json 2> $O/cfg4_256.err
timeout 600 python tools/time_path.py cfg0 --once > $O/cfg0.json 2> $O/cfg0.err
for h in "1 1" "0 0"; do set -- $h
GS_L2_HINT=$1 GS_LDS_EXPLICIT=$2 timeout 300 python tools/time_screen.py cfg1 20 > $O/screen_cfg1_h$1_l$2.json 2>> $O/err.txt
done
rm -f $O/*.ncu-rep.tmp
