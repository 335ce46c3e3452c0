#!/bin/bash
O=gpurun_out/c6; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_path.py tests/test_gpu_kernels.py tests/test_gpu_batch.py tests/test_sharded.py -m gpu -q -rf -x \
    -k "blocked or cd_modes or certify or cfg0_full or cd_pass or stress or cfg1_shape or batch or deterministic or sharded" > $O/pytest_blk.log 2>&1
echo "pytest rc=$?" >> $O/pytest_blk.log
GS_CD_PROF=1 timeout 600 python tools/time_path.py cfg1 --once > $O/cfg1_prof.txt 2> $O/cfg1_prof.err
GS_CD_PROF=1 timeout 600 python tools/time_path.py cfg0 --once > $O/cfg0_prof.txt 2> $O/cfg0_prof.err
timeout 600 python tools/time_path.py cfg1 --once --per-lambda > $O/cfg1.json 2> $O/cfg1.err
timeout 600 python tools/time_path.py cfg0 --once > $O/cfg0.json 2> $O/cfg0.err
