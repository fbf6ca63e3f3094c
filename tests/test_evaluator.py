"""The in-process evaluator (paper_2402_09222_b200.evaluate) against the
reference's Evaluator contract (proj/src/harness.hpp:92-102): it never raises;
any failure — including a non-finite objective — is status 'fail' with the
penalty as objective (proj/src/ensemble.cpp:182-191); it is called
concurrently from n_workers threads (proj/src/ensemble.cpp:163-197)."""
import threading

import numpy as np
import pytest

import paper_2402_09222_b200 as P

from conftest import _has_gpu

SMALL = dict(n_particles=2000, n_batches=3, n_inactive=1)
CFG = {"P0": "openmc", "P1": 1000, "P2": 4000, "P3": 20000, "P4": 2, "P5": 1, "P6": "threads"}


@pytest.mark.skipif(_has_gpu(), reason="CPU-only: the no-device failure path")
def test_evaluate_without_gpu_is_fail_with_penalty():
    r = P.evaluate(CFG, problem=P.Problem("pincell"), penalty=-7.5, **SMALL)
    assert r["status"] == "fail" and r["objective"] == -7.5 and r["elapsed"] >= 0
    assert "CUDA" in r["message"] or "device" in r["message"]


def test_evaluate_bad_configuration_is_fail_with_penalty():
    """Invalid parameters are rejected before any device work (no GPU needed)."""
    for bad in ({**CFG, "P1": 0}, {**CFG, "P2": 0}, {**CFG, "P5": 99}, {**CFG, "P0": "openmc-bogus"}):
        r = P.evaluate(bad, problem=P.Problem("pincell"), **SMALL)
        assert r["status"] == "fail" and r["objective"] == -1.0, bad


@pytest.mark.gpu
def test_evaluate_ok_and_deterministic():
    p = P.Problem("pincell")
    a = P.evaluate(CFG, problem=p, **SMALL)
    b = P.evaluate({**CFG, "P0": "openmc-queueless", "P3": float("nan"), "P1": 500}, problem=p, **SMALL)
    assert a["status"] == b["status"] == "ok"
    assert a["objective"] > 0 and b["objective"] > 0
    assert a["k_eff"] == b["k_eff"]  # tuned parameters change time only


@pytest.mark.gpu
def test_evaluate_concurrent_workers():
    """Four worker threads evaluate at once on one GPU (the ensemble's n_workers
    pattern): every call succeeds, results equal the serial ones, and a failing
    call in the mix does not disturb the others."""
    p = P.Problem("pincell")
    cfgs = [{**CFG, "P1": 500 * (w + 1)} for w in range(4)] + [{**CFG, "P1": 0}]
    serial = P.evaluate(CFG, problem=p, **SMALL)
    out = [None] * len(cfgs)

    def work(i):
        out[i] = P.evaluate(cfgs[i], problem=p, **SMALL)

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(cfgs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert [o["status"] for o in out] == ["ok"] * 4 + ["fail"]
    assert all(o["k_eff"] == serial["k_eff"] for o in out[:4])
    assert np.isfinite([o["objective"] for o in out]).all()
