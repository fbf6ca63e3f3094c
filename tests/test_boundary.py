"""The process-level drop-in boundary: bin/openmc under the reference's own,
unchanged tuner (oracle/_ref/libautotune.so built from /root/reference/proj/src)
and unchanged campaign (proj/campaigns/openmc: space.json, openmc.sh.in,
launcher.in, campaign.json; copied to oracle/_ref/campaigns by build_ref.sh).

Pins: argv `--event -i P1 -b P2 [-m P3]`, mode from argv[0]
(openmc / openmc-queueless), "FOM: <x> particles/s" on stdout (last match,
proj/src/harness.cpp:150-171), metrics.txt "<package_J> <dram_J>"
(harness.cpp:117-136), nonzero exit -> status fail + penalty (harness.cpp:292).
"""
import csv
import json
import os
import subprocess
import time

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "bin")
REF = os.path.join(ROOT, "oracle", "_ref")
CAMPAIGN = os.path.join(REF, "campaigns", "openmc", "campaign.json")
have_ref = pytest.mark.skipif(not os.path.exists(os.path.join(REF, "atune_run")),
                              reason="reference tuner not built (oracle/build_ref.sh needs /root/reference)")


def has_gpu():
    from conftest import _has_gpu
    return _has_gpu()


def run_openmc(args, env=None, cwd=None, name="openmc"):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([os.path.join(BIN, name)] + args, capture_output=True, text=True, env=e, cwd=cwd,
                          timeout=600)


def test_usage_errors_exit_2(tmp_path):
    assert run_openmc(["--event", "-i"], cwd=tmp_path).returncode == 2
    assert run_openmc(["--event", "-q", "5"], cwd=tmp_path).returncode == 2
    r = run_openmc(["-i", "100", "-b", "100"], cwd=tmp_path)
    assert r.returncode == 2 and "--event" in r.stderr


@pytest.mark.skipif(has_gpu(), reason="GPU visible")
def test_no_gpu_fails_loudly(tmp_path):
    r = run_openmc(["--event", "-i", "1000", "-b", "100", "-m", "0"], cwd=tmp_path)
    assert r.returncode == 3
    assert "CUDA" in r.stderr or "cuda" in r.stderr
    assert "FOM" not in r.stdout


def read_results(path):
    with open(path) as f:
        return list(csv.DictReader(f))


def run_campaign(campaign, out, evals, workers, env):
    e = dict(os.environ)
    e["PATH"] = BIN + os.pathsep + e["PATH"]
    e.update(env)
    r = subprocess.run([os.path.join(REF, "atune_run"), campaign, str(out), str(evals), str(workers)],
                       capture_output=True, text=True, env=e, timeout=1800)
    return r, read_results(os.path.join(out, "results.csv"))


@have_ref
@pytest.mark.skipif(has_gpu(), reason="GPU visible")
def test_reference_harness_records_failures_without_gpu(tmp_path):
    r, rows = run_campaign(CAMPAIGN, tmp_path / "run", 3, 2, {})
    assert len(rows) == 3
    assert all(row["status"] == "fail" and float(row["objective"]) == -1.0 for row in rows)
    # the unchanged mold called our binary with the documented argv
    script = open(tmp_path / "run" / "evals" / "0" / "script").read()
    assert "openmc --event -i" in script or "openmc-queueless --event -i" in script


SMALL = {"OMCG_PARTICLES": "20000", "OMCG_BATCHES": "3", "OMCG_INACTIVE": "1", "OMCG_LEASE_DIR": "/tmp"}


@pytest.mark.gpu
def test_openmc_binary_contract(tmp_path):
    for name, args in (("openmc", ["--event", "-i", "20000", "-b", "4000", "-m", "20000"]),
                       ("openmc-queueless", ["--event", "-i", "20000", "-b", "4000"]),
                       ("openmc", ["--event", "-i", "5000", "-b", "100", "-m", "nan"])):
        d = tmp_path / name / args[2]
        d.mkdir(parents=True)
        r = run_openmc(args, env=dict(SMALL, AUTOTUNE_LAUNCHER_ARGS="-c 4 --ntasks-per-gpu=2 --cpu-bind=cores"),
                       cwd=d, name=name)
        assert r.returncode == 0, r.stderr
        fom = [l for l in r.stdout.splitlines() if l.startswith("FOM:")]
        assert len(fom) == 1 and fom[0].endswith("particles/s") and float(fom[0].split()[1]) > 0
        pkg, dram = open(d / "metrics.txt").read().split()
        assert float(pkg) >= 0 and float(dram) >= 0
        assert ("queueless" in r.stderr) == (name == "openmc-queueless")
        assert "P5=2" in r.stderr and "P4=4" in r.stderr


@have_ref
@pytest.mark.gpu
def test_unchanged_reference_campaign_runs_on_gpu_fom(tmp_path):
    r, rows = run_campaign(CAMPAIGN, tmp_path / "fom", 6, 2, SMALL)
    assert r.returncode == 0, r.stderr
    assert len(rows) == 6 and all(row["status"] == "ok" for row in rows), rows
    for row in rows:
        out = open(tmp_path / "fom" / "evals" / row["eval_id"] / "stdout.log").read()
        last = [l for l in out.splitlines() if l.startswith("FOM:")][-1]
        assert float(row["objective"]) == pytest.approx(float(last.split()[1]), rel=1e-9)


@have_ref
@pytest.mark.gpu
def test_unchanged_reference_campaign_runs_on_gpu_edp(tmp_path):
    src = json.load(open(CAMPAIGN))
    d = os.path.dirname(CAMPAIGN)
    src.update(space_file=os.path.join(d, src["space_file"]), mold_file=os.path.join(d, src["mold_file"]),
               launcher_file=os.path.join(d, src["launcher_file"]), metric={"kind": "edp"})
    src.pop("baseline", None)
    cj = tmp_path / "edp_campaign.json"
    cj.write_text(json.dumps(src))
    r, rows = run_campaign(str(cj), tmp_path / "edp", 4, 2, SMALL)
    assert r.returncode == 0, r.stderr
    assert all(row["status"] == "ok" and float(row["objective"]) > 0 for row in rows), rows


def _abs_campaign(tmp_path, name, **overrides):
    src = json.load(open(CAMPAIGN))
    d = os.path.dirname(CAMPAIGN)
    for k in ("space_file", "mold_file", "launcher_file"):
        src[k] = os.path.join(d, src[k])
    src.pop("baseline", None)
    src.update(overrides)
    cj = tmp_path / name
    cj.write_text(json.dumps(src))
    return str(cj)


@have_ref
@pytest.mark.gpu
def test_timeout_sigkill_releases_gpu_lease(tmp_path):
    """The harness SIGKILLs the whole process group at the timeout with no
    grace period (proj/src/harness.cpp:267-283). A killed bin/openmc must leave
    no state behind: its flock GPU lease is released by the kernel, no process
    of the evaluation survives, and the next evaluations lease the GPU and
    finish ok."""
    import fcntl
    lease = tmp_path / "lease"
    lease.mkdir()
    # long runs (1e6 histories x 40 batches, ~3 s on the GPU) against a 1.5 s timeout
    killer = _abs_campaign(tmp_path, "timeout.json", timeout=1.5)
    big = {"OMCG_PARTICLES": "1000000", "OMCG_BATCHES": "40", "OMCG_INACTIVE": "1", "OMCG_LEASE_DIR": str(lease)}
    r, rows = run_campaign(killer, tmp_path / "killed", 3, 1, big)
    assert r.returncode == 0, r.stderr
    assert [row["status"] for row in rows] == ["timeout"] * 3, rows
    for row in rows:  # the binary was inside its GPU run when it was killed (it had leased the GPU)
        err = open(tmp_path / "killed" / "evals" / row["eval_id"] / "stdout.log").read()
        assert "FOM:" not in err
    # No holder of the lease survives the SIGKILL. The harness reaps the
    # evaluation's /bin/sh at once, while the killed bin/openmc (its child, in
    # the same process group) may still be tearing down its CUDA context; its
    # descriptors -- the flock lease among them -- close when that exit
    # completes. So the contract is "released once the killed processes are
    # gone", checked with a bounded wait.
    deadline = time.time() + 30.0
    while True:
        ps = subprocess.run(["ps", "-eo", "comm="], capture_output=True, text=True).stdout.split()
        alive = [c for c in ps if c.startswith("openmc")]
        fd = os.open(str(lease / "omcg-gpu-0.lock"), os.O_RDWR)
        try:
            fcntl.flock(fd, fcntl.LOCK_EX | fcntl.LOCK_NB)  # raises if any process still holds it
            fcntl.flock(fd, fcntl.LOCK_UN)
            held = False
        except BlockingIOError:
            held = True
        finally:
            os.close(fd)
        if not alive and not held:
            break
        assert time.time() < deadline, f"lease held={held}, surviving processes {alive} 30 s after the kill"
        time.sleep(0.1)
    # the next evaluations lease the same GPU and complete
    ok = _abs_campaign(tmp_path, "ok.json")
    r, rows = run_campaign(ok, tmp_path / "after", 3, 2, dict(SMALL, OMCG_LEASE_DIR=str(lease)))
    assert r.returncode == 0, r.stderr
    assert all(row["status"] == "ok" and float(row["objective"]) > 0 for row in rows), rows


GPU_CAMPAIGN = os.path.join(REF, "atune_gpu_campaign")
have_gpu_campaign = pytest.mark.skipif(not os.path.exists(GPU_CAMPAIGN),
                                       reason="in-process GPU evaluator driver not built (oracle/build_ref.sh)")


def run_gpu_campaign(campaign, out, evals, workers, env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([GPU_CAMPAIGN, campaign, str(out), str(evals), str(workers)], capture_output=True,
                       text=True, env=e, timeout=1800)
    return r, read_results(os.path.join(out, "results.csv"))


@have_gpu_campaign
@pytest.mark.skipif(has_gpu(), reason="GPU visible")
def test_inprocess_gpu_evaluator_failures_without_gpu(tmp_path):
    """The in-process evaluator (integration/gpu_evaluator.cpp) under the
    reference's own campaign loop: without a device every evaluation is
    status fail with the penalty, and the campaign still completes."""
    r, rows = run_gpu_campaign(CAMPAIGN, tmp_path / "g", 4, 2, {})
    assert r.returncode == 0, r.stderr
    assert len(rows) == 4 and all(row["status"] == "fail" and float(row["objective"]) == -1.0 for row in rows)


@have_gpu_campaign
@pytest.mark.gpu
@pytest.mark.parametrize("metric", ["fom", "edp"])
def test_inprocess_gpu_evaluator_campaign(tmp_path, metric):
    """A 4-worker campaign over the unchanged campaigns/openmc space through the
    in-process `gpu` evaluator kind: the reference's
    run_campaign calls the evaluator from 4 threads at once; every evaluation
    leases the GPU in-process and succeeds."""
    camp = CAMPAIGN if metric == "fom" else _abs_campaign(tmp_path, "edp.json", metric={"kind": "edp"})
    small = {"OMCG_PARTICLES": "20000", "OMCG_BATCHES": "3", "OMCG_INACTIVE": "1"}
    r, rows = run_gpu_campaign(camp, tmp_path / metric, 12, 4, small)
    assert r.returncode == 0, r.stderr
    assert len(rows) == 12 and all(row["status"] == "ok" and float(row["objective"]) > 0 for row in rows), \
        [(row["status"], row["objective"], row.get("elapsed")) for row in rows]
    assert len({row["worker_id"] for row in rows}) == 4
