"""CPU tests of the C-ABI library (libomcg.so) — no compute calls need a GPU here.

* libomcg.so loads and exports exactly the symbols include/omcg.h declares
* struct layouts seen by Python (ctypes) match the C header (sizeof/offsetof)
* the product's host-side synthetic-library generator reproduces the oracle's
  library bit-for-bit (independent restatements of the same specification)
* without a GPU, device entry points fail loudly (OMCG_ECUDA), never fall back
* argument validation returns OMCG_EINVAL before touching the device
* the multi-GPU fission-bank exchange plan is consistent (host logic)
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O
import paper_2402_09222_b200 as P
from paper_2402_09222_b200 import _omcg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "omcg.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"OMCG_API\s+[\w\s\*]+?\b(omcg_\w+)\s*\(", txt)))


def test_exports_match_header():
    out = subprocess.run(["nm", "-D", "--defined-only", _omcg.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = sorted(l.split()[-1] for l in out.splitlines() if " T " in l)
    assert exported == header_symbols()
    assert sorted(_omcg.EXPORTS) == header_symbols()
    lib = ctypes.CDLL(_omcg.LIB_PATH)
    for s in header_symbols():
        assert hasattr(lib, s)


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "omcg.h"\nint main(void){'
                   'printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(omcg_run_config), sizeof(omcg_run_result),'
                   ' sizeof(omcg_record), sizeof(omcg_problem_info), offsetof(omcg_run_config, tail_threshold),'
                   ' offsetof(omcg_run_result, tail_launches), offsetof(omcg_run_config, nccl_id));return 0;}')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(_omcg.RunConfig), ctypes.sizeof(_omcg.RunResult), ctypes.sizeof(_omcg.Record),
            ctypes.sizeof(_omcg.ProblemInfo), _omcg.RunConfig.tail_threshold.offset,
            _omcg.RunResult.tail_launches.offset, _omcg.RunConfig.nccl_id.offset]
    assert got == want


@pytest.mark.parametrize("kind", [O.PINCELL, O.ASSEMBLY, O.CORE])
def test_host_library_matches_oracle(kind):
    o = O.Problem(kind, 1234, 4000)
    p = P.Problem(kind, 1234, host_threads=3)
    assert p.library_checksum() == o.library_checksum()
    assert p.info.n_nuclides == o.info.n_nuclides
    assert p.info.n_grid_total == o.info.n_grid_total
    assert p.info.n_tally_bins == o.info.n_tally_bins
    assert p.info.fuel_nuclides == o.info.fuel_nuclides


def test_library_generation_thread_invariant_and_seeded():
    a = P.Problem("assembly", 1234, host_threads=1).library_checksum()
    b = P.Problem("assembly", 1234, host_threads=16).library_checksum()
    c = P.Problem("assembly", 4321, host_threads=8).library_checksum()
    assert a == b != c


def test_problem_sizes():
    p = P.Problem("assembly")
    assert p.info.n_nuclides == 272          # PAPER.md:190 (HM-Large total)
    assert p.info.fuel_nuclides == 261       # depleted fuel
    assert 100e6 < p.info.lib_bytes < 130e6  # ~122 MB: E + 4 channels, f64
    assert P.Problem("pincell").info.n_nuclides == 10


def _no_gpu():
    try:
        P.device_count()
        return False
    except P.OmcgError as e:
        return e.code == _omcg.OMCG_ECUDA


@pytest.mark.skipif(not _no_gpu(), reason="a GPU is visible")
def test_device_entry_points_fail_loudly_without_gpu():
    p = P.Problem("pincell")
    with pytest.raises(P.OmcgError) as e:
        P.run(p, n_particles=100, n_batches=2, n_inactive=1)
    assert e.value.code == _omcg.OMCG_ECUDA
    with pytest.raises(P.OmcgError) as e:
        p.hash_build(100)
    assert e.value.code == _omcg.OMCG_ECUDA


@pytest.mark.parametrize("kw", [dict(n_batches=0), dict(n_inactive=5, n_batches=5), dict(particles_in_flight=0),
                                dict(n_bins=0), dict(tasks_per_gpu=0), dict(mode=7), dict(n_particles=0)])
def test_invalid_config_is_einval(kw):
    p = P.Problem("pincell")
    args = dict(n_particles=100, n_batches=2, n_inactive=1)
    args.update(kw)
    with pytest.raises(P.OmcgError) as e:
        P.run(p, **args)
    assert e.value.code == _omcg.OMCG_EINVAL


def test_null_arguments():
    lib = P._lib
    assert lib.omcg_run(None, None, None, None, None) == _omcg.OMCG_EINVAL
    assert b"null" in lib.omcg_last_error()
    assert lib.omcg_problem_create(9, 1, 1, ctypes.byref(ctypes.c_void_p())) == _omcg.OMCG_EINVAL


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_bank_exchange_plan_is_a_partition(world):
    rng = np.random.default_rng(world)
    N = 1000 + world
    for _ in range(20):
        S_all = rng.integers(0, 700, world).astype(np.uint64)
        S_all[rng.integers(0, world)] += 1
        S = int(S_all.sum())
        off = int(rng.integers(0, S))
        plans = [P.bank_exchange_plan(S_all, N, off, r) for r in range(world)]
        G = np.concatenate([[0], np.cumsum(S_all)])
        for r in range(world):
            W = world
            need_first, need_count = plans[r][4 * W], plans[r][4 * W + 1]
            lo, hi = N * r // W, N * (r + 1) // W
            if hi > lo:
                assert need_first == (lo * S + off) // N
                assert need_first + need_count - 1 == ((hi - 1) * S + off) // N
            covered = 0
            for q in range(W):
                # what r receives from q equals what q sends to r, at consistent offsets
                rc, rf = plans[r][3 * W + q], plans[r][2 * W + q]
                sc, sf = plans[q][W + r], plans[q][r]
                assert rc == sc
                if rc:
                    assert G[q] + sf == need_first + rf
                covered += rc
            assert covered == need_count
