timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "tuned or core or tiny" 2>&1 | tail -15
