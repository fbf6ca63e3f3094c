"""CPU tests of the oracle (oracle/omc_oracle.c) against the golden fixtures.

ref_derive_seed.json pins the seed derivation against the REFERENCE
(proj/src/rng.hpp:10-25, compiled by oracle/build_ref.sh). The oracle_*.json
vectors freeze the oracle's own outputs; the
transport arithmetic is "parity unpinned" against the reference (it ships
no transport code) — see oracle/omc_oracle.h.
"""
import ctypes
import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
sys.path.insert(0, GOLD)
import make_golden as G  # noqa: E402


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_derive_seed_matches_reference_golden():
    ref = load("ref_derive_seed.json")
    L = O.lib()
    for b, s, want in ref["derive_seed"]:
        assert L.orc_derive_seed(int(b), int(s)) == int(want)


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(HERE), "oracle", "_ref", "ref_rng")),
                    reason="oracle/_ref not built (needs /root/reference)")
def test_derive_seed_matches_live_reference():
    exe = os.path.join(os.path.dirname(HERE), "oracle", "_ref", "ref_rng")
    live = json.loads(subprocess.run([exe], capture_output=True, text=True, check=True).stdout)
    L = O.lib()
    for b, s, want in live["derive_seed"]:
        assert L.orc_derive_seed(int(b), int(s)) == int(want)


def test_rng_golden_and_skip_ahead():
    g = load("oracle_rng.json")
    L = O.lib()
    for pid, vals in g["particle_streams"].items():
        s = ctypes.c_uint64(L.orc_particle_seed(1, int(pid)))
        assert [G.hexbits(L.orc_prn(ctypes.byref(s))) for _ in range(16)] == vals
    for n, seed, want in g["future_seed"]:
        assert L.orc_future_seed(int(n), int(seed)) == int(want)
    # skip-ahead equals sequential stepping (O(log n) vs O(n))
    M, A, MASK = 6364136223846793005, 1442695040888963407, (1 << 64) - 1
    for seed in (0, 1, 12345):
        x = seed
        for n in range(0, 300):
            assert L.orc_future_seed(n, seed) == x
            x = (M * x + A) & MASK


def test_prn_range_and_moments():
    L = O.lib()
    s = ctypes.c_uint64(L.orc_particle_seed(7, 1))
    v = np.array([L.orc_prn(ctypes.byref(s)) for _ in range(20000)])
    assert v.min() >= 0.0 and v.max() < 1.0
    assert abs(v.mean() - 0.5) < 0.01 and abs(v.var() - 1 / 12) < 0.005


def test_deterministic_log_exp_accuracy():
    g = load("oracle_rng.json")
    L = O.lib()
    for x, want in g["log"]:
        assert G.hexbits(L.orc_log(float(np.uint64(int(x, 16)).view(np.float64)))) == want
    for y, want in g["exp"]:
        assert G.hexbits(L.orc_exp(float(np.uint64(int(y, 16)).view(np.float64)))) == want
    rng = np.random.default_rng(5)
    xs = np.exp(rng.uniform(-700, 700, 20000))
    got = np.array([L.orc_log(float(x)) for x in xs])
    ulp = np.abs(got - np.log(xs)) / np.spacing(np.abs(np.log(xs)) + 1e-300)
    assert np.max(ulp[np.abs(np.log(xs)) > 1e-3]) <= 4
    ys = rng.uniform(-700, 700, 20000)
    got = np.array([L.orc_exp(float(y)) for y in ys])
    rel = np.abs(got - np.exp(ys)) / np.exp(ys)
    assert rel.max() < 2e-15


@pytest.mark.parametrize("entry", range(3))
def test_lookup_vectors_golden(entry):
    g = load("oracle_lookup.json")[entry]
    _, got = G.lookup_vectors(g["kind"], g["bins"])
    for k in ("library_checksum", "hash_checksum", "bin_sha256", "index_sha256", "micro_sha256", "macro_sha256",
              "first"):
        assert got[k] == g[k], k


def test_grid_index_independent_of_hash_bins():
    """bins only narrow the search; the found interval is the same."""
    probs = {b: O.Problem(O.ASSEMBLY, 1234, b) for b in (1, 100, 4000, 100000)}
    rng = np.random.default_rng(3)
    for _ in range(400):
        nuc = int(rng.integers(0, 272))
        E = float(np.exp(rng.uniform(np.log(1e-5), np.log(2e7))))
        ref = probs[4000].micro(nuc, E)
        for b, p in probs.items():
            assert p.micro(nuc, E) == ref


def test_micro_interpolation_brackets():
    p = O.Problem(O.PINCELL, 1234, 4000)
    for nuc in range(p.info.n_nuclides):
        E, xs = p.grid(nuc)
        assert E[0] == 1e-5 and E[-1] == 2e7 and np.all(np.diff(E) > 0)
        assert np.all(xs[:, 0] > 0) and np.all(xs[:, 1] >= 0)
        assert np.all(xs[:, 0] >= xs[:, 1]) and np.all(xs[:, 1] >= xs[:, 2])
        for k in (0, len(E) // 3, len(E) - 2):
            idx, m = p.micro(nuc, float(E[k]))
            assert idx == k and m == list(xs[k])


def test_transport_c1_golden():
    g = load("oracle_transport_c1.json")
    got = G.transport_vectors()
    assert got == g


def test_transport_thread_count_invariance():
    p = O.Problem(O.ASSEMBLY, 1234, 4000)
    a = p.run(600, 3, 1, seed=3, threads=1, record_batch=2, record_n=600)
    b = p.run(600, 3, 1, seed=3, threads=7, record_batch=2, record_n=600)
    assert [a[0].k_coll[i] for i in range(3)] == [b[0].k_coll[i] for i in range(3)]
    assert np.array_equal(a[1], b[1])
    assert bytes(a[2]) == bytes(b[2])


def test_pincell_physics_sanity():
    p = O.Problem(O.PINCELL, 1234, 4000)
    res, tally, _ = p.run(20000, 6, 2, seed=11, threads=0)
    assert res.n_lost == 0 and res.n_leaked == 0  # fully reflective pin cell
    k = [res.k_coll[i] for i in range(2, 6)]
    assert 1.0 < np.mean(k) < 1.2
    # the three k estimators agree statistically
    for est in (res.k_abs, res.k_track):
        assert abs(np.mean([est[i] for i in range(2, 6)]) - np.mean(k)) < 0.02
    flux, absr, fis, nufis = (tally.reshape(-1, 4)[0] / 2**28)
    assert flux > 0 and absr > 0 and fis > 0 and nufis > 2 * fis
    # absorption rate per source particle ~ 1 (every history ends absorbed) within tally noise
    assert abs(absr / (4 * 20000) - 1.0) < 0.05


@pytest.mark.parametrize("kind", [O.PINCELL, O.ASSEMBLY])
def test_queue_trace_consistent_with_history_transport(kind):
    """Two independent oracle code paths agree: with one kernel per event and no
    tail, the queued emulation (orc_queue_trace) visits the advance, crossing
    and collision queues exactly as often as the history-based transport
    (orc_run) counts those events; with event fusion only the fuel lookup,
    move and collision queues (and the tail) ever run, and fewer iterations."""
    n = 3000
    p = O.Problem(kind, 1234, 4000)
    res, _, _ = p.run(n, 1, 0, seed=1, threads=0)
    t0 = p.queue_trace(n, n, 0, seed=1, event_fusion=False)
    tot = {q: int(t0[t0[:, 0] == q, 1].sum()) for q in range(6)}
    assert tot[2] == res.n_events[1]  # advance
    assert tot[3] == res.n_events[2]  # crossing
    assert tot[4] == res.n_events[3]  # collision
    assert tot[0] + tot[1] <= res.n_events[0]  # lookups (cache hits skip the queue)
    t1 = p.queue_trace(n, n, 0, seed=1, event_fusion=True)
    assert set(np.unique(t1[:, 0])) <= {0, 2, 4}
    assert len(t1) < len(t0)
    assert int(t1[t1[:, 0] == 4, 1].sum()) <= res.n_events[3]
    # every history enters the move queue at least once; id checksums are order-free sums
    assert int(t1[t1[:, 0] == 2, 1].sum()) >= n
    # move-kernel event cap: 1 -> every flight and every crossing takes its own
    # move-queue entry; a cap no history reaches -> the uncapped trace
    t_c1 = p.queue_trace(n, n, 0, seed=1, event_fusion=True, move_cap=1)
    assert int(t_c1[t_c1[:, 0] == 2, 1].sum()) >= res.n_events[1] + res.n_events[2]
    assert set(np.unique(t_c1[:, 0])) <= {0, 2, 4}
    t_off = p.queue_trace(n, n, 0, seed=1, event_fusion=True, move_cap=0)
    assert np.array_equal(p.queue_trace(n, n, 0, seed=1, event_fusion=True, move_cap=10**6), t_off)
    assert len(t_c1) > len(t_off)


def test_oracle_matches_infinite_medium_analytic():
    """Independent physics pin of the oracle: the analytic infinite medium
    (k_inf = nu*Sigma_f/Sigma_a = 1.5625, Sigma_t/Sigma_a collisions and
    1/Sigma_a track length per history), tests/analytic.py."""
    import analytic
    p = O.Problem(O.INFINITE, 1234, 4000)
    n, b, i = 50_000, 22, 2
    res, tally, _ = p.run(n, b, i, seed=1, threads=0)
    analytic.check(res, tally, n, b, i)
