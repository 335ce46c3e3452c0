#!/bin/bash
O=gpurun_out/c19; mkdir -p $O
for ch in 8192 16384 32768; do
GS_CD_CHUNK=$ch timeout 900 python tools/time_path.py cfg3 --once --lambdas 70 > $O/cfg3_l70_chunk$ch.json 2> $O/cfg3_chunk$ch.err
done
for g in 1 2 4 8; do
GS_GROUP_CTAS=$g timeout 300 python tools/time_path.py cfg0 --once > $O/cfg0_G$g.json 2> $O/cfg0_G$g.err
done
timeout 600 python tools/time_path.py cfg1 --once > $O/cfg1.json 2> $O/cfg1.err
