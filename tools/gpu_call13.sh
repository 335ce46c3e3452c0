#!/bin/bash
O=gpurun_out/c13; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,clocks.max.mem,power.draw,power.limit,temperature.gpu,clocks_event_reasons.active --format=csv > $O/smi_before.txt 2>&1
(while true; do nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.active --format=csv,noheader; sleep 2; done) > $O/smi_trace.txt 2>&1 &
SMI=$!
timeout 900 python bench.py --steps 2 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
GS_CD_PROF=1 timeout 600 python tools/time_path.py cfg1 --once --lambdas 92 > $O/cfg1_prof.txt 2> $O/cfg1_prof.err
timeout 600 python tools/time_path.py cfg0 --once > $O/cfg0.json 2> $O/cfg0.err
timeout 600 python tools/time_batch.py 256 > $O/cfg4_256.json 2> $O/cfg4_256.err
kill $SMI
