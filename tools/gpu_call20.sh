#!/bin/bash
O=gpurun_out/c20; mkdir -p $O
for g in 16 32 64; do
GS_GROUP_CTAS=$g timeout 300 python tools/time_path.py cfg0 --once > $O/cfg0_G$g.json 2> $O/cfg0_G$g.err
done
GS_CD_CHUNK=16384 timeout 1500 python tools/time_path.py cfg3 --once > $O/cfg3_chunk16384.json 2> $O/cfg3_chunk16384.err
