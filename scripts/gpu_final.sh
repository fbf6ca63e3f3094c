# Round-end evidence: core pass (tests, smoke, bench, ncu, C4, C3) then C5 at the reference's budget.
bash scripts/gpu_evidence_core.sh
bash scripts/gpu_c5_full.sh
