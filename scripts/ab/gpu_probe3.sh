timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
run() {
python - <<PY
import sys; sys.path.insert(0,'.')
import paper_2402_09222_b200 as P
p = P.Problem("assembly")
for prof in (0, 1):
    r = P.run(p, n_particles=1000000, n_batches=7, n_inactive=2, profile=prof).result
    names=["xs_fuel","xs_nonfuel","adv","cross","coll","sort","refill","tail"]
    print(f"$1 prof={prof} FoM={r.fom:.4e} t_active={r.t_active:.3f} k={r.k_mean:.6f}", " ".join(f"{n}={r.prof_ms[i]/5:.1f}ms" for i,n in enumerate(names)) if prof else "")
PY
}
OMCG_TAIL_WARP=0 run tail_thread
OMCG_TAIL_WARP=1 run tail_warp
