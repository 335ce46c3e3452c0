#!/bin/bash
# CPU reference arm (oracle, complete paths) for cfg0 and cfg3 on the GPU box's host cores,
# and the cfg2 200,000-column prefix path for comparison with round 1.
O=gpurun_out/${1:-refs}; mkdir -p $O
timeout 600 python bench.py --impl reference --config cfg0 --steps 1 --warmup 3 > $O/bench_reference_cfg0.json 2> $O/ref_cfg0.err
timeout 1500 python bench.py --impl reference --config cfg3 --steps 1 --warmup 3 --ref-budget 60 > $O/bench_reference_cfg3.json 2> $O/ref_cfg3.err
timeout 900 python tools/time_path.py cfg2 200000 --once > $O/cfg2_p200k.json 2> $O/cfg2_p200k.err
