# ncu source-level capture of one cfg1 lambda solve (k_solve launch #40)
O=gpurun_out/${1:-p1}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -s 40 -c 1 -o $O/solve_cfg1 -f \
   python tools/prof_path.py cfg1 45 > $O/ncu_solve.log 2>&1; echo "ncu solve rc=$?" >> $O/ncu_solve.log
