"""ctypes binding of the CPU oracle (oracle/_build/liboracle.so).

TEST / BASELINE INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs, never by the product
package. See omc_oracle.h for the parity status ("parity unpinned" for the
transport arithmetic; the reference ships no transport code).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")
CLI_PATH = os.path.join(HERE, "_build", "openmc-oracle")

PINCELL, ASSEMBLY, CORE, INFINITE = 0, 1, 2, 3
# the analytic infinite medium (omc_oracle.h ORC_INF_*)
INF_SIGMA_T, INF_SIGMA_A, INF_SIGMA_F, INF_NU = 1.0, 0.4, 0.25, 2.5
MAX_BATCHES = 512


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class Info(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("n_nuclides", C.c_int), ("n_materials", C.c_int), ("n_bins", C.c_int),
        ("nx", C.c_int), ("ny", C.c_int), ("n_tally_bins", C.c_int), ("fuel_material", C.c_int),
        ("fuel_nuclides", C.c_int), ("n_grid_total", C.c_int64), ("lib_bytes", C.c_int64),
        ("hash_bytes", C.c_int64),
    ]


class RunConfig(C.Structure):
    _fields_ = [
        ("n_particles", C.c_int64), ("n_batches", C.c_int), ("n_inactive", C.c_int),
        ("seed", C.c_uint64), ("n_threads", C.c_int), ("record_batch", C.c_int),
        ("record_n", C.c_int64), ("stop_after_batch", C.c_int),
    ]


class Record(C.Structure):
    _fields_ = [
        ("n_xs", C.c_int32), ("n_adv", C.c_int32), ("n_cross", C.c_int32), ("n_coll", C.c_int32),
        ("n_sites", C.c_int32), ("term", C.c_int32), ("e_final", C.c_double), ("x_final", C.c_double),
    ]


class RunResult(C.Structure):
    _fields_ = [
        ("n_batches_run", C.c_int),
        ("k_coll", C.c_double * MAX_BATCHES), ("k_abs", C.c_double * MAX_BATCHES),
        ("k_track", C.c_double * MAX_BATCHES), ("n_sites", C.c_int64 * MAX_BATCHES),
        ("n_events", C.c_int64 * 4), ("n_leaked", C.c_int64), ("n_absorbed", C.c_int64),
        ("n_lost", C.c_int64), ("k_mean", C.c_double), ("k_std", C.c_double),
        ("t_active", C.c_double), ("t_total", C.c_double), ("fom", C.c_double),
    ]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.orc_problem_create.argtypes = [C.c_int, C.c_uint64, C.c_int, C.POINTER(P)]
        L.orc_problem_free.argtypes = [P]
        L.orc_problem_free.restype = None
        L.orc_problem_get_info.argtypes = [P, C.POINTER(Info)]
        L.orc_library_checksum.argtypes = [P]
        L.orc_library_checksum.restype = C.c_uint64
        L.orc_hash_checksum.argtypes = [P]
        L.orc_hash_checksum.restype = C.c_uint64
        L.orc_nuclide_grid_size.argtypes = [P, C.c_int]
        L.orc_nuclide_copy.argtypes = [P, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_hash_copy.argtypes = [P, C.c_int, C.c_void_p]
        L.orc_hash_bin.argtypes = [P, C.c_double]
        L.orc_micro_xs.argtypes = [P, C.c_int, C.c_double, C.POINTER(C.c_int32), C.c_double * 4]
        L.orc_macro_xs.argtypes = [P, C.c_int, C.c_double, C.c_double * 4]
        L.orc_macro_xs_ckpt.argtypes = [P, C.c_int, C.c_double, C.c_double * 4, C.c_double * 16,
                                        C.POINTER(C.c_int)]
        L.orc_macro_xs_ckpt_n.argtypes = [P, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p]
        L.orc_log.argtypes = [C.c_double]
        L.orc_log.restype = C.c_double
        L.orc_exp.argtypes = [C.c_double]
        L.orc_exp.restype = C.c_double
        L.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_future_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_future_seed.restype = C.c_uint64
        L.orc_prn.argtypes = [C.POINTER(C.c_uint64)]
        L.orc_prn.restype = C.c_double
        L.orc_particle_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_particle_seed.restype = C.c_uint64
        L.orc_run.argtypes = [P, C.POINTER(RunConfig), C.POINTER(RunResult), C.c_void_p, C.c_void_p]
        L.orc_last_error.restype = C.c_char_p
        L.orc_queue_trace.argtypes = [P, C.c_int64, C.c_uint64, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_void_p,
                                      C.c_int64, C.POINTER(C.c_int64)]
        _lib = L
    return _lib


class Problem:
    """Oracle problem (synthetic library + hash grid + geometry)."""

    def __init__(self, kind: int, xs_seed: int = 1234, n_bins: int = 4000):
        L = lib()
        self._p = C.c_void_p()
        if L.orc_problem_create(kind, xs_seed, n_bins, C.byref(self._p)) != 0:
            raise RuntimeError(L.orc_last_error().decode())
        self.info = Info()
        L.orc_problem_get_info(self._p, C.byref(self.info))
        self.kind, self.n_bins = kind, n_bins

    def __del__(self):
        if getattr(self, "_p", None):
            lib().orc_problem_free(self._p)
            self._p = None

    def library_checksum(self) -> int:
        return lib().orc_library_checksum(self._p)

    def hash_checksum(self) -> int:
        return lib().orc_hash_checksum(self._p)

    def hash_bin(self, E: float) -> int:
        return lib().orc_hash_bin(self._p, E)

    def micro(self, nuc: int, E: float):
        idx = C.c_int32()
        out = (C.c_double * 4)()
        if lib().orc_micro_xs(self._p, nuc, E, C.byref(idx), out) != 0:
            raise RuntimeError(lib().orc_last_error().decode())
        return idx.value, list(out)

    def macro(self, mat: int, E: float):
        out = (C.c_double * 4)()
        if lib().orc_macro_xs(self._p, mat, E, out) != 0:
            raise RuntimeError(lib().orc_last_error().decode())
        return list(out)

    def macro_ckpt(self, mat: int, E: float):
        """(macro XS[4], segment checkpoints[:nck]) as calculate_xs stores them."""
        out = (C.c_double * 4)()
        ck = (C.c_double * 16)()
        nck = C.c_int()
        if lib().orc_macro_xs_ckpt(self._p, mat, E, out, ck, C.byref(nck)) != 0:
            raise RuntimeError(lib().orc_last_error().decode())
        return list(out), list(ck)[: nck.value]

    def macro_ckpt_n(self, mat, E):
        """Vectorised macro_ckpt: (xs [n, 4], ck [n, 16] (NaN past nck), nck [n])."""
        import numpy as np
        mat = np.ascontiguousarray(mat, np.int32)
        E = np.ascontiguousarray(E, np.float64)
        n = len(E)
        xs = np.empty((n, 4), np.float64)
        ck = np.full((n, 16), np.nan)
        nck = np.empty(n, np.int32)
        if lib().orc_macro_xs_ckpt_n(self._p, n, mat.ctypes.data, E.ctypes.data, xs.ctypes.data, ck.ctypes.data,
                                     nck.ctypes.data) != 0:
            raise RuntimeError(lib().orc_last_error().decode())
        return xs, ck, nck

    def grid(self, nuc: int):
        import numpy as np
        n = lib().orc_nuclide_grid_size(self._p, nuc)
        E = np.empty(n, np.float64)
        xs = np.empty((n, 4), np.float64)
        lib().orc_nuclide_copy(self._p, nuc, E.ctypes.data, xs.ctypes.data)
        return E, xs

    def queue_trace(self, n_particles: int, in_flight: int, tail_threshold: int, seed: int = 1,
                    event_fusion: bool = True, move_cap: int = 20):
        """Queued event-loop emulation of batch 1: array of (queue, length, id-checksum).
        move_cap mirrors omcg_run_config.move_event_cap (used with event fusion only)."""
        import numpy as np
        n = C.c_int64()
        f = int(bool(event_fusion))
        if lib().orc_queue_trace(self._p, n_particles, seed, in_flight, tail_threshold, f, move_cap, None, 0,
                                 C.byref(n)) != 0:
            raise RuntimeError(lib().orc_last_error().decode())
        out = np.zeros((n.value, 3), np.int64)
        lib().orc_queue_trace(self._p, n_particles, seed, in_flight, tail_threshold, f, move_cap, out.ctypes.data,
                              n.value, C.byref(n))
        return out

    def run(self, n_particles: int, n_batches: int, n_inactive: int, seed: int = 1, threads: int = 0,
            record_batch: int = 0, record_n: int = 0, stop_after_batch: int = 0):
        """History-based transport; returns (RunResult, tally int64[n_tally_bins*4], records)."""
        import numpy as np
        cfg = RunConfig(n_particles, n_batches, n_inactive, seed, threads, record_batch, record_n,
                        stop_after_batch)
        res = RunResult()
        tally = np.zeros(self.info.n_tally_bins * 4, np.int64)
        recs = (Record * max(record_n, 1))()
        rc = lib().orc_run(self._p, C.byref(cfg), C.byref(res), tally.ctypes.data,
                           C.cast(recs, C.c_void_p) if record_n > 0 else None)
        if rc != 0:
            raise RuntimeError(lib().orc_last_error().decode())
        return res, tally, (recs if record_n > 0 else None)


def records_array(recs, n):
    """Structured numpy view of n records."""
    import numpy as np
    dt = np.dtype([("n_xs", "<i4"), ("n_adv", "<i4"), ("n_cross", "<i4"), ("n_coll", "<i4"),
                   ("n_sites", "<i4"), ("term", "<i4"), ("e_final", "<f8"), ("x_final", "<f8")])
    return np.frombuffer(bytes(recs)[: n * dt.itemsize], dtype=dt).copy()
