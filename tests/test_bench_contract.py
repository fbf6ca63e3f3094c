"""CPU check of bench.py's reference arm: `bench.py --impl reference` times the
CPU oracle (the reference ships no transport code) and prints one JSON line
with the contract's keys; under torchrun only rank 0 prints."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--problem", "pincell", "--cpu-sample", "2000"],
                         capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return [l for l in out.stdout.splitlines() if l.strip()]


def test_reference_arm_json_line():
    lines = _run({})
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"]


def test_reference_arm_other_ranks_silent():
    assert _run({"RANK": "1", "WORLD_SIZE": "2"}) == []


def test_clock_sampler_degrades_without_a_gpu():
    """The clocks key is always a dict with the contract's fields; on a host
    without NVML / nvidia-smi it says so instead of failing the bench."""
    sys.path.insert(0, ROOT)
    import bench
    s = bench.clock_sampler(0)
    s.wait_ready(timeout=0.2)
    s.mark()
    d = s.stop()
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in d, k
    assert isinstance(d["reasons"], list)


def test_roofline_fields_from_committed_ncu():
    """bench.py's roofline extras come from the committed ncu summary: the fuel
    lookup's DRAM rate is a true HBM fraction (well below 1, unlike the
    algorithmic-byte `frac`), and the binding roof is the L1 data pipe."""
    sys.path.insert(0, ROOT)
    import bench
    roofs = bench.ncu_roofs()
    k = roofs["k_xs_fuel_fused"]
    f = bench.roof_fields(k, 1e6, 1.3, 6554.9)
    assert 0.0 < f["dram_frac"] < 0.2
    br = f["binding_roof"]
    assert br["name"] == "L1/TEX throughput"
    assert br["l1_data_pipe_wavefronts_pct"] > 50.0
    assert br["source"].startswith("profiles/")
    assert os.path.exists(os.path.join(ROOT, br["source"].split(" ")[0]))
