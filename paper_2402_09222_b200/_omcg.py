"""ctypes mirror of include/omcg.h (libomcg.so, built in-tree by __graft_entry__.build()).

The library is the product: sm_100a CUDA kernels behind a C ABI. There is no
CPU fallback — if libomcg.so is missing the import fails loudly, and on a
machine without a GPU every device entry point returns OMCG_ECUDA.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libomcg.so")

OMCG_OK, OMCG_EINVAL, OMCG_EIO, OMCG_ECUDA, OMCG_ENCCL, OMCG_EFAIL = range(6)
PINCELL, ASSEMBLY, CORE, INFINITE = 0, 1, 2, 3
QUEUED, QUEUELESS = 0, 1
BIND_CORES, BIND_THREADS, BIND_SOCKETS = 0, 1, 2
N_SCORES = 4
MAX_BATCHES = 512

#: symbols declared in include/omcg.h (checked by tests/test_capi.py)
EXPORTS = (
    "omcg_version", "omcg_last_error", "omcg_problem_create", "omcg_problem_free",
    "omcg_problem_get_info", "omcg_library_checksum", "omcg_hash_build", "omcg_xs_lookup",
    "omcg_xs_lookup_queue", "omcg_div_check",
    "omcg_run_config_default", "omcg_run", "omcg_queue_trace", "omcg_nccl_unique_id",
    "omcg_device_count", "omcg_bank_exchange_plan", "omcg_energy_counter_mj",
    "omcg_energy_mark", "omcg_energy_since_mark_j", "omcg_release_devices",
)


class ProblemInfo(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("n_nuclides", C.c_int), ("n_materials", C.c_int),
        ("nx", C.c_int), ("ny", C.c_int), ("n_tally_bins", C.c_int), ("fuel_nuclides", C.c_int),
        ("n_grid_total", C.c_int64), ("lib_bytes", C.c_int64), ("gen_seconds", C.c_double),
    ]


class RunConfig(C.Structure):
    _fields_ = [
        ("mode", C.c_int), ("particles_in_flight", C.c_int64), ("n_bins", C.c_int),
        ("sort_threshold", C.c_int64), ("host_threads", C.c_int), ("tasks_per_gpu", C.c_int),
        ("cpu_bind", C.c_int), ("n_particles", C.c_int64), ("n_batches", C.c_int),
        ("n_inactive", C.c_int), ("seed", C.c_uint64), ("n_gpus", C.c_int),
        ("devices", C.c_int * 8), ("world_size", C.c_int), ("rank", C.c_int),
        ("nccl_id", C.c_ubyte * 128), ("record_batch", C.c_int), ("record_n", C.c_int64),
        ("profile", C.c_int), ("trace_queues", C.c_int), ("tail_threshold", C.c_int64),
        ("event_fusion", C.c_int), ("move_event_cap", C.c_int), ("force_nccl", C.c_int),
        ("device_schedule", C.c_int),
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
        ("t_init", C.c_double), ("t_active", C.c_double), ("t_total", C.c_double),
        ("fom", C.c_double), ("energy_j", C.c_double), ("kernel_launches", C.c_int64),
        ("kernel_launches_total", C.c_int64), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
        ("prof_ms", C.c_double * 8), ("prof_launches", C.c_int64 * 8), ("prof_items", C.c_int64 * 8),
        ("xs_fuel_bytes", C.c_double), ("queue_iterations", C.c_int64), ("sorts", C.c_int64),
        ("tail_launches", C.c_int64),
    ]


def load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the transport path)")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    lib.omcg_version.restype = C.c_char_p
    lib.omcg_last_error.restype = C.c_char_p
    lib.omcg_problem_create.argtypes = [C.c_int, C.c_uint64, C.c_int, C.POINTER(P)]
    lib.omcg_problem_free.argtypes = [P]
    lib.omcg_problem_free.restype = None
    lib.omcg_problem_get_info.argtypes = [P, C.POINTER(ProblemInfo)]
    lib.omcg_library_checksum.argtypes = [P]
    lib.omcg_library_checksum.restype = C.c_uint64
    lib.omcg_hash_build.argtypes = [P, C.c_int, C.c_int, C.POINTER(C.c_uint64), C.c_void_p]
    lib.omcg_xs_lookup.argtypes = [P, C.c_int, C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.omcg_xs_lookup_queue.argtypes = [P, C.c_int, C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,
                                         C.c_void_p, C.c_void_p]
    lib.omcg_div_check.argtypes = [C.c_int, C.c_int64] + [C.c_void_p] * 6
    lib.omcg_run_config_default.argtypes = [C.POINTER(RunConfig)]
    lib.omcg_run_config_default.restype = None
    lib.omcg_run.argtypes = [P, C.POINTER(RunConfig), C.POINTER(RunResult), C.c_void_p, C.c_void_p]
    lib.omcg_queue_trace.argtypes = [C.c_void_p, C.c_int64]
    lib.omcg_queue_trace.restype = C.c_int64
    lib.omcg_nccl_unique_id.argtypes = [C.c_void_p]
    lib.omcg_device_count.argtypes = [C.POINTER(C.c_int)]
    lib.omcg_energy_counter_mj.argtypes = [C.c_int, C.POINTER(C.c_uint64)]
    lib.omcg_energy_since_mark_j.argtypes = [C.c_int, C.POINTER(C.c_double)]
    lib.omcg_bank_exchange_plan.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_int, C.c_void_p]
    return lib
