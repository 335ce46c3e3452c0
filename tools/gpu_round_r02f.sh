#!/bin/bash
# Final checks of round 2 on the last build: smoke, full GPU suite, bench line, other-config
# path times, configs[2] at full size.
TAG=${1:-r02f}; O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > $O/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 300 python tools/time_path.py cfg0 --once > $O/cfg0.json 2> $O/cfg0.err
timeout 1500 python tools/time_path.py cfg3 --once > $O/cfg3.json 2> $O/cfg3.err
timeout 900 python tools/time_path.py cfg2 200000 --once > $O/cfg2_p200k.json 2> $O/cfg2_p200k.err
timeout 2400 python tools/run_cfg2_full.py 1000000 --check 1 > $O/cfg2_full.json 2> $O/cfg2_full.err; echo "rc=$?" >> $O/cfg2_full.err
