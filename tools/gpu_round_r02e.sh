#!/bin/bash
# Final checks of round 2 on the last build: smoke, full GPU suite, bench line, other-config path times.
TAG=${1:-r02e}; O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > $O/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 300 python tools/time_path.py cfg0 --once > $O/cfg0.json 2> $O/cfg0.err
timeout 1500 python tools/time_path.py cfg3 --once > $O/cfg3.json 2> $O/cfg3.err
timeout 600 python tools/time_batch.py 256 > $O/cfg4_256.json 2> $O/cfg4_256.err
timeout 300 python tools/time_screen.py cfg1 20 > $O/screen_cfg1.json 2>> $O/err.txt
timeout 600 python tools/time_screen.py cfg2 20 100000 > $O/screen_cfg2_p100k.json 2>> $O/err.txt
timeout 900 python tools/time_screen.py cfg3 20 > $O/screen_cfg3.json 2>> $O/err.txt
timeout 900 python bench.py --config cfg4 --problems 148 --steps 1 --quick --cpu-budget 10 > $O/bench_cfg4_148.json 2> $O/bench_cfg4.err; echo "rc=$?" >> $O/bench_cfg4.err
