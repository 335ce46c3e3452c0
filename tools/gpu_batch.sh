O=gpurun_out/bt; mkdir -p $O
timeout 600 compute-sanitizer --tool memcheck python tools/time_batch.py 160 2000 > $O/sanitize_160.log 2>&1; echo "rc=$?" >> $O/sanitize_160.log
timeout 600 python -m pytest tests/test_gpu_batch.py tests/test_sharded.py -q -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python tools/time_batch.py 256 > $O/cfg4_256.json 2>&1
