# quick GPU cycle: gpu tests + path timings (tag as $1)
O=gpurun_out/${1:-q}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/time_path.py cfg1 --once --lambdas 60 > $O/cfg1_60.json 2>&1
