# quick GPU cycle: gpu tests + path timings (tag as $1)
O=gpurun_out/${1:-q}; mkdir -p $O
timeout 300 python tools/time_path.py cfg1 --once --lambdas 60 > $O/cfg1_60.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/time_path.py cfg1 --once > $O/cfg1.json 2>&1
timeout 300 python tools/time_path.py cfg0 --once > $O/cfg0.json 2>&1
