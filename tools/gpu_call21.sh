#!/bin/bash
O=gpurun_out/c21; mkdir -p $O
for nap in 0 20 100; do
GS_BLK_NAP=$nap timeout 600 python tools/time_path.py cfg1 --once > $O/cfg1_nap$nap.json 2> $O/cfg1_nap$nap.err
done
timeout 300 python tools/time_path.py cfg0 --once > $O/cfg0.json 2> $O/cfg0.err
timeout 900 python -m pytest tests/test_gpu_path.py tests/test_gpu_kernels.py -m gpu -q -rf -x -k "blocked or cd_modes or certify or deterministic or cfg0 or cfg1_shape or sparse_csc or hooks or budget" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
