"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Bar: bit-exact for every integer output (hash grid, grid
indices, per-history event counts, termination, sites, queue lengths) and —
because the device code follows the oracle operation-for-operation with FMA
contraction disabled and tallies are int64 fixed point — bit-exact for the
floating-point outputs too (macroscopic XS, final energies/positions, k-eff
per batch, tally sums). The stated statistical tolerance (k within 3 sigma of
the oracle's independent run) is only used for cross-configuration checks
whose histories differ by construction.
"""
import numpy as np
import pytest

import oracle as O
import paper_2402_09222_b200 as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", [P.PINCELL, P.ASSEMBLY])
@pytest.mark.parametrize("bins", [1, 100, 4000, 100000])
def test_hash_grid_bit_exact(kind, bins):
    o = O.Problem(kind, 1234, bins)
    p = P.Problem(kind, 1234)
    chk, _ = p.hash_build(bins)
    assert chk == o.hash_checksum()


@pytest.mark.parametrize("kind", [P.PINCELL, P.ASSEMBLY])
@pytest.mark.parametrize("bins", [100, 4000])
def test_macro_xs_bit_exact(kind, bins):
    o = O.Problem(kind, 1234, bins)
    p = P.Problem(kind, 1234)
    rng = np.random.default_rng(1)
    n = 20000 if kind == P.PINCELL else 3000
    E = np.exp(rng.uniform(np.log(1e-6), np.log(3e7), n))  # includes out-of-grid energies
    E[:4] = [1e-5, 2e7, 1e-7, 5e7]
    mat = rng.integers(0, 3, n).astype(np.int32)
    got = p.xs_lookup(bins, mat, E)
    want = np.array([o.macro(int(m), float(e)) for m, e in zip(mat, E)])
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_branch_free_division_matches_ieee():
    """div_chk (the compiler's fast path for a / b without its slow-path
    branch, used by the flight, collision and lookup arithmetic): wherever it
    reports the fast path valid the quotient equals the device's '/' bit for
    bit, and the device's '/' equals the host's IEEE division. div_frac (the
    interpolation fraction and det_log's mantissa quotient, no fallback)
    equals '/' on both domains, including a = 0 (E on a grid point, m = 1)."""
    rng = np.random.default_rng(11)
    n = 2_000_000
    # arbitrary bit patterns: zeros, subnormals, huge, inf and NaN included
    bits = rng.integers(0, 2**63, (2, n), dtype=np.uint64) | (rng.integers(0, 2, (2, n), dtype=np.uint64) << 63)
    a, b = bits.view(np.float64)
    # the transport's ranges: distances / direction cosines, energies, sums of squares
    m = n // 4
    a[:m] = rng.uniform(-30.0, 30.0, m)
    b[:m] = rng.uniform(-1.0, 1.0, m) * np.exp(rng.uniform(-40, 0, m))
    a[m:2 * m] = np.exp(rng.uniform(np.log(1e-5), np.log(2e7), m))
    b[m:2 * m] = np.exp(rng.uniform(np.log(1e-5), np.log(2e7), m))
    specials = np.array([0.0, -0.0, 1.0, -1.0, 5e-324, 2.2250738585072014e-308, 1e-300, 1e300, 1.7976931348623157e308,
                         np.inf, -np.inf, np.nan, 1e-5, 2e7], np.float64)
    k = len(specials)
    a[2 * m:2 * m + k * k] = np.repeat(specials, k)
    b[2 * m:2 * m + k * k] = np.tile(specials, k)
    qf, ok, _, qi, sf, sok, si = P.div_check(a, b)
    with np.errstate(all="ignore"):
        host, hsqrt = a / b, np.sqrt(a)
    same = lambda x, y: (x.view(np.uint64) == y.view(np.uint64)) | (np.isnan(x) & np.isnan(y))
    assert same(qi, host).all()
    assert same(qf[ok], qi[ok]).all()
    assert ok[:2 * m].mean() > 0.999  # the fallback stays rare on the transport's ranges
    # sqrt_chk: the same contract for the square roots
    assert same(si, hsqrt).all()
    assert same(sf[sok], si[sok]).all()
    assert sok[m:2 * m].all() and sok.mean() > 0.45
    # div_frac on interpolation fractions: E_lo <= E < E_hi on the library grid
    lo = np.exp(rng.uniform(np.log(1e-5), np.log(2e7), n))
    hi = np.minimum(lo * np.exp(rng.uniform(1e-15, 0.5, n)), 2e7)
    hi = np.where(hi > lo, hi, np.nextafter(lo, np.inf))
    E = lo + (hi - lo) * rng.uniform(0.0, 1.0, n)
    E = np.where(E < hi, E, lo)
    E[: n // 8] = lo[: n // 8]  # on a grid point: numerator exactly 0
    num, den = E - lo, hi - lo
    _, _, qr, qi, _, _, _ = P.div_check(num, den)
    assert same(qr, qi).all()
    assert same(qi, num / den).all()
    # det_log's (m - 1) / (m + 1) on its reduced mantissa m in [sqrt(2)/2, sqrt(2)], m = 1 included
    m = np.concatenate([rng.uniform(np.sqrt(0.5), np.sqrt(2.0), n), [1.0, np.nextafter(1.0, 0), np.nextafter(1.0, 2)]])
    _, _, qr, qi, _, _, _ = P.div_check(m - 1.0, m + 1.0)
    assert same(qr, qi).all()


@pytest.mark.parametrize("bins", [100, 4000])
@pytest.mark.parametrize("sort", [None, 20000])
@pytest.mark.parametrize("mix", ["fuel", "mixed"])
def test_fuel_lookup_kernel_bit_exact(bins, sort, mix):
    """The production fuel calculate_xs (k_xs_fuel_fused: 4 warps share the
    17 segments of the 261-nuclide fuel, partials folded in shared memory) on a
    queue of 1.2e5 histories, unsorted and sorted by (material, energy) as the
    queued loop sorts at P3 — macroscopic XS and the 16 segment checkpoints the
    collision samples from, bit for bit against the oracle."""
    kind = P.ASSEMBLY
    o = O.Problem(kind, 1234, bins)
    p = P.Problem(kind, 1234)
    rng = np.random.default_rng(7)
    n = 120_000
    E = np.exp(rng.uniform(np.log(1e-6), np.log(3e7), n))  # includes out-of-grid energies
    E[:6] = [1e-5, 2e7, 1e-7, 5e7, 1e-5 * (1 + 1e-15), 2e7 * (1 - 1e-15)]
    E[6:1000] = E[6]  # one energy many times (a sorted bucket of equal keys)
    fuel = o.info.fuel_material
    mat = np.full(n, fuel, np.int32) if mix == "fuel" else rng.integers(0, o.info.n_materials, n).astype(np.int32)
    got, gck = p.xs_lookup_queue(bins, mat, E, sort_threshold=sort)
    want, wck, nck = o.macro_ckpt_n(mat, E)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    for k in range(16):
        sel = nck > k
        assert np.array_equal(gck[sel, k].view(np.uint64), wck[sel, k].view(np.uint64)), k
    if mix == "fuel":
        assert (nck == 16).all()


def _oracle_run(kind, n, batches, inactive, rec_n, bins):
    key = (kind, n, batches, inactive, rec_n, bins)
    if key not in _ORACLE_CACHE:
        o = O.Problem(kind, 1234, bins)
        ores, otally, orecs = o.run(n, batches, inactive, seed=1, record_batch=2, record_n=rec_n)
        _ORACLE_CACHE[key] = (ores, otally, O.records_array(orecs, rec_n))
    return _ORACLE_CACHE[key]


_ORACLE_CACHE = {}


def _compare_runs(kind, n, batches, inactive, rec_n, **kw):
    # the oracle's results do not depend on P2 (its hash bracket is repaired
    # like the GPU's), so one oracle run per problem size serves every variant
    ores, otally, orec = _oracle_run(kind, n, batches, inactive, rec_n, kw.get("n_bins", 4000))
    p = P.Problem(kind, 1234)
    out = P.run(p, n_particles=n, n_batches=batches, n_inactive=inactive, seed=1, record_batch=2,
                record_n=rec_n, **kw)
    r = out.result
    assert r.n_lost == ores.n_lost == 0
    for f in ("n_xs", "n_adv", "n_cross", "n_coll", "n_sites", "term"):
        assert np.array_equal(out.records[f], orec[f]), f
    assert np.array_equal(out.records["e_final"].view(np.uint64), orec["e_final"].view(np.uint64))
    assert np.array_equal(out.records["x_final"].view(np.uint64), orec["x_final"].view(np.uint64))
    for b in range(batches):
        assert r.k_coll[b] == ores.k_coll[b], b
        assert r.k_abs[b] == ores.k_abs[b], b
        assert r.k_track[b] == ores.k_track[b], b
        assert r.n_sites[b] == ores.n_sites[b], b
    assert list(r.n_events) == list(ores.n_events)
    assert (r.n_leaked, r.n_absorbed) == (ores.n_leaked, ores.n_absorbed)
    assert np.array_equal(out.tally, otally)
    return out


def test_pincell_transport_bit_exact():
    _compare_runs(P.PINCELL, 20000, 4, 2, 2000, particles_in_flight=20000)


@pytest.mark.parametrize("fusion", [1, 0])
def test_assembly_transport_bit_exact(fusion):
    _compare_runs(P.ASSEMBLY, 4000, 3, 1, 1000, particles_in_flight=4000, tail_threshold=100, event_fusion=fusion)


@pytest.mark.parametrize("fusion,cap,dsched", [(1, 20, 0), (1, 0, 0), (1, 3, 0), (0, 20, 0), (1, 20, 1), (1, 0, 1),
                                               (1, 3, 1)])
@pytest.mark.parametrize("kind,n,in_flight,tail,sort", [
    (P.PINCELL, 6000, 1500, 300, 0),       # refill active, sorted fuel queue, tail
    (P.PINCELL, 4000, 4000, 0, -1),        # all in flight, no tail
    (P.ASSEMBLY, 3000, 1000, 200, 500),
])
def test_queue_contents_bit_exact(kind, n, in_flight, tail, sort, fusion, cap, dsched):
    """North star: queue contents match. Per queued-mode iteration, the chosen
    queue, its length and the order-free checksum of its history ids equal the
    oracle's emulation of the same scheduling policy (batch 1), with and
    without event fusion (the move kernel), with the move kernel's
    per-launch event cap at its default, off, and small, and with the queue
    choice made on the host or by the GPU itself (device_schedule)."""
    o = O.Problem(kind, 1234, 4000)
    want = o.queue_trace(n, in_flight, tail, seed=1, event_fusion=bool(fusion), move_cap=cap)
    p = P.Problem(kind, 1234)
    out = P.run(p, n_particles=n, n_batches=1, n_inactive=0, seed=1, particles_in_flight=in_flight,
                tail_threshold=tail, sort_threshold=sort, trace_queues=True, event_fusion=fusion,
                move_event_cap=cap, device_schedule=dsched)
    got = out.queue_trace
    assert got.shape == want.shape
    assert np.array_equal(got, want)


def test_c2_bench_configuration_bit_exact():
    """Parity where the benchmark runs (BASELINE.json configs[1], bench.py's
    defaults): 17x17 assembly, 261-nuclide depleted fuel, 1e6 histories per
    batch, P1 = 1e6 in flight, P2 = 4000, P3 = 20000 (the fuel-queue sort fires:
    checked below), queued with event fusion, move cap 20, tail threshold
    16384 — 3 batches (1 inactive). k per batch, int64 tallies, event totals
    and the records of the first 1e4 histories of batch 2, bit for bit."""
    n = 1_000_000
    out = _compare_runs(P.ASSEMBLY, n, 3, 1, 10_000, particles_in_flight=n, n_bins=4000, sort_threshold=20_000)
    assert out.result.sorts > 0
    assert out.result.tail_launches == 3


def test_c2_bench_configuration_device_schedule_bit_exact():
    """The same bench configuration with the queue choice made on the GPU
    (device-driven loop): identical results, and the same
    number of queue iterations and sorts as the host-driven loop."""
    n = 1_000_000
    kw = dict(particles_in_flight=n, n_bins=4000, sort_threshold=20_000)
    dev = _compare_runs(P.ASSEMBLY, n, 3, 1, 10_000, device_schedule=1, **kw)
    host = P.run(P.Problem(P.ASSEMBLY, 1234), n_particles=n, n_batches=3, n_inactive=1, seed=1, **kw)
    assert dev.result.queue_iterations == host.result.queue_iterations
    assert dev.result.sorts == host.result.sorts


TUNED_VARIANTS = [
    dict(particles_in_flight=1000),                       # P1 < N: dynamic refill
    dict(particles_in_flight=5000, sort_threshold=0),     # always sort
    dict(particles_in_flight=5000, sort_threshold=-1),    # never sort
    dict(particles_in_flight=5000, n_bins=100),           # P2
    dict(particles_in_flight=5000, n_bins=100000),
    dict(mode="openmc-queueless", particles_in_flight=3000),  # P0
    dict(particles_in_flight=2000, tasks_per_gpu=2),      # P5
    dict(particles_in_flight=5000, tail_threshold=0),     # pure event-by-event (move kernel)
    dict(particles_in_flight=5000, tail_threshold=0, event_fusion=0),  # one kernel per event type
    dict(particles_in_flight=1000, event_fusion=0),
    dict(particles_in_flight=5000, tail_threshold=10**9),  # history-per-thread tail right after refill
    dict(mode="openmc-queueless", particles_in_flight=3000, tail_threshold=0),
    dict(mode="openmc-queueless", particles_in_flight=3000, tail_threshold=0, event_fusion=0),
    dict(mode="openmc-queueless", particles_in_flight=1000, tail_threshold=200, event_fusion=0),
    # multi-rank path (partition, int64 reductions, fission-bank exchange plan)
    # with ranks sharing GPU 0 through the in-process loopback transport
    dict(particles_in_flight=5000, n_gpus=2, devices=[0, 0]),
    dict(particles_in_flight=2000, n_gpus=3, devices=[0, 0, 0], tasks_per_gpu=2),
    # move-kernel event cap: every event of the move queue a separate visit; no cap
    dict(particles_in_flight=5000, tail_threshold=0, move_event_cap=1),
    dict(particles_in_flight=5000, tail_threshold=0, move_event_cap=0),
    # one history in flight at a time; more slots than histories
    dict(particles_in_flight=1, tail_threshold=0),
    dict(particles_in_flight=50000),
    # the per-batch exchanges through a one-rank NCCL communicator
    dict(particles_in_flight=5000, force_nccl=True),
    # the queue choice made by the GPU itself (device-driven loop), with refill first and all in flight
    dict(particles_in_flight=2000, device_schedule=1),
    dict(particles_in_flight=10000, tail_threshold=0, device_schedule=1),
]
ASSEMBLY_VARIANTS = TUNED_VARIANTS + [
    dict(particles_in_flight=10000, sort_threshold=500),  # the sort fires on the depleted fuel queue
    dict(particles_in_flight=2500, sort_threshold=500, tail_threshold=100),
    dict(mode="openmc-queueless", particles_in_flight=10000, tasks_per_gpu=2),
    dict(particles_in_flight=10000, sort_threshold=500, device_schedule=1, tasks_per_gpu=2),
]


@pytest.mark.parametrize("kw", TUNED_VARIANTS)
def test_tuned_parameters_do_not_change_results(kw):
    """in-flight count (and every other tuned knob) changes time only."""
    _compare_runs(P.PINCELL, 10000, 3, 1, 1000, **kw)


@pytest.mark.parametrize("kw", [k for k in ASSEMBLY_VARIANTS if k.get("particles_in_flight") != 1])
def test_tuned_parameters_do_not_change_results_assembly(kw):
    """The same invariance on the 261-nuclide depleted-fuel assembly (17
    segments per fuel lookup: the split-K lookup, the collision checkpoints,
    the fuel-queue sort at P3 = 500 and 0)."""
    _compare_runs(P.ASSEMBLY, 10000, 3, 1, 1000, **kw)


def test_core_transport_bit_exact():
    """C4 geometry (37 assemblies, water reflector, vacuum boundaries: leakage)."""
    out = _compare_runs(P.CORE, 3000, 2, 1, 500, particles_in_flight=3000, tail_threshold=100)
    assert out.result.n_leaked > 0


def test_core_transport_at_scale_bit_exact():
    """C4 at 2e5 histories per batch with the library defaults (sorted fuel
    queue, warp-cooperative lookups, move cap, tail), 2 batches."""
    out = _compare_runs(P.CORE, 200_000, 2, 1, 2000, particles_in_flight=200_000)
    assert out.result.n_leaked > 0 and out.result.sorts > 0


@pytest.mark.parametrize("kw", [
    dict(n_gpus=3, devices=[0, 0, 0], tasks_per_gpu=4),   # ragged: 7 histories over 12 sub-banks
    dict(particles_in_flight=2),
    dict(mode="openmc-queueless", particles_in_flight=3),
])
def test_tiny_ragged_runs_bit_exact(kw):
    """Edge sizes: fewer histories than ranks x sub-banks, a 2-slot bank."""
    _compare_runs(P.PINCELL, 7, 3, 1, 7, **kw)


def test_infinite_medium_bit_exact_vs_oracle():
    _compare_runs(P.INFINITE, 20000, 3, 1, 1000, particles_in_flight=5000)


@pytest.mark.parametrize("mode", ["openmc", "openmc-queueless"])
def test_infinite_medium_analytic(mode):
    """Independent physics pin of the GPU path (not through the oracle): the
    analytic infinite medium at 1e6 histories per batch — k_inf =
    nu*Sigma_f/Sigma_a within 3 sigma (collision and track-length estimators)
    and exactly (absorption estimator), Sigma_t/Sigma_a collisions and
    1/Sigma_a track length per history, no leakage (tests/analytic.py)."""
    import analytic
    p = P.Problem("infinite")
    n, b, i = 1_000_000, 12, 2
    out = P.run(p, mode=mode, n_particles=n, n_batches=b, n_inactive=i, particles_in_flight=n)
    analytic.check(out.result, out.tally, n, b, i)
