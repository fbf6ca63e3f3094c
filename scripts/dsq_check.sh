# device_schedule A/B on C2 (run_c2.py, 5 active batches), interleaved
for r in 1 2 3; do
for ds in 0 1; do timeout 300 python scripts/run_c2.py 7 2 device_schedule=$ds 2>&1 | grep -v "^$" | head -2; done
done
