#!/bin/bash
O=gpurun_out/c10; mkdir -p $O
for v in "1 1" "0 1" "1 0" "0 0"; do set -- $v
GS_L2_HINT=$1 GS_LDS_EXPLICIT=$2 timeout 300 python tools/time_path.py cfg0 600 --once > $O/cfg0_p600_h$1_l$2.json 2> $O/cfg0_p600_h$1_l$2.err; echo "rc=$?" >> $O/cfg0_p600_h$1_l$2.err
done
for v in "0 1" "0 0" "1 0"; do set -- $v
GS_L2_HINT=$1 GS_LDS_EXPLICIT=$2 GS_CD_PROF=1 timeout 600 python tools/time_path.py cfg1 --once --lambdas 92 > $O/cfg1_h$1_l$2.txt 2> $O/cfg1_h$1_l$2.err
done
