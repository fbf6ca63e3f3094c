# GPU test pass: the -m gpu suite (parity vs the oracle, analytic pin, evaluator) + smoke.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests/ -q -m gpu --durations=20 > gpurun_out/gputests.txt 2>&1
tail -30 gpurun_out/gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
tail -2 gpurun_out/smoke.txt
