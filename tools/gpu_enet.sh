#!/bin/bash
# Elastic-Net (F2) GPU parity tests, then smoke().
O=gpurun_out/enet; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_path.py -m gpu -q -k "elastic or tail" > $O/pytest_enet.log 2>&1; echo "pytest rc=$?" >> $O/pytest_enet.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
