set -x
timeout 900 python -m pytest tests/test_boundary.py -q -m gpu -k "timeout or binary_contract" > gpurun_out/boundary.txt 2>&1; tail -5 gpurun_out/boundary.txt
bash scripts/gpu_sanitize.sh > /dev/null 2>&1; cat gpurun_out/sanitize/summary.txt
bash scripts/gpu_c5_edp.sh
