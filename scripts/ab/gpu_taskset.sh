nproc; lscpu | grep -i "numa\|model name" | head -4
python scripts/e2e_noise3.py free
taskset -c 0-7 python scripts/e2e_noise3.py taskset0-7
python scripts/e2e_noise3.py free
taskset -c 0-7 python scripts/e2e_noise3.py taskset0-7
