# Round-2 evidence pass on one B200 (outputs under gpurun_out/r02/):
#  1. compute-sanitizer re-runs (queueless racecheck after the syncwarp fix; the
#     move-cap/P5 case at a size racecheck finishes)
#  2. the one-rank NCCL data plane through bench.py (--force-nccl), plain and under torchrun
#  3. the in-process `gpu` evaluator kind under the reference's campaign loop (C2 size, 4 workers)
#  4. the C5 EDP campaign (256 evaluations, 1 worker) + elapsed-vs-standalone check
set -x
mkdir -p gpurun_out/r02
bash scripts/gpu_sanitize_subset.sh "racecheck:pincell_queueless racecheck:assembly_queueless memcheck:pincell_cap1_p5 racecheck:pincell_cap1_p5 synccheck:pincell_cap1_p5 initcheck:pincell_cap1_p5"
timeout 600 python bench.py --force-nccl --steps 5 --warmup 3 > gpurun_out/r02/bench_force_nccl.json 2> gpurun_out/r02/bench_force_nccl.err
tail -c 600 gpurun_out/r02/bench_force_nccl.json
NCCL_DEBUG=INFO timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --force-nccl --steps 5 --warmup 3 > gpurun_out/r02/bench_torchrun_nccl.json 2> gpurun_out/r02/bench_torchrun_nccl.err
tail -c 600 gpurun_out/r02/bench_torchrun_nccl.json; grep -c "NCCL INFO" gpurun_out/r02/bench_torchrun_nccl.err
rm -rf /tmp/c5_inproc
OMCG_PARTICLES=1000000 OMCG_BATCHES=6 OMCG_INACTIVE=2 timeout 1200 oracle/_ref/atune_gpu_campaign oracle/_ref/campaigns/openmc/campaign.json /tmp/c5_inproc 64 4 > gpurun_out/r02/c5_inprocess_fom_report.txt 2>&1
cp /tmp/c5_inproc/results.csv gpurun_out/r02/c5_inprocess_fom_results.csv; head -20 gpurun_out/r02/c5_inprocess_fom_report.txt
bash scripts/gpu_c5_edp.sh
mv gpurun_out/c5_edp_* gpurun_out/r02/
