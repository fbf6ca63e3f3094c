// capi.cpp — extern "C" surface of libomcg.so (include/omcg.h).
// Error model mirrors the reference C ABI (proj/src/capi.cpp:24-76): every
// entry point returns an int code, exceptions never cross the boundary, and
// omcg_last_error() holds the calling thread's last message.
#define OMCG_BUILDING 1
#include "../../include/omcg.h"

#include <cstring>
#include <exception>
#include <new>
#include <string>

#include "problem.hpp"
#include "transport.hpp"

struct omcg_problem {
    omcg::Problem p;
};

namespace {
thread_local std::string g_err;

template <typename F>
int wrap(F&& f) {
    try {
        f();
        return OMCG_OK;
    } catch (const omcg::CudaError& e) {
        g_err = e.what();
        return OMCG_ECUDA;
    } catch (const omcg::NcclError& e) {
        g_err = e.what();
        return OMCG_ENCCL;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return OMCG_EINVAL;
    } catch (const omcg::IoError& e) {
        g_err = e.what();
        return OMCG_EIO;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return OMCG_EFAIL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return OMCG_EFAIL;
    } catch (...) {
        g_err = "unknown error";
        return OMCG_EFAIL;
    }
}
}  // namespace

extern "C" {

OMCG_API const char* omcg_version(void) { return "omcg 0.1 (sm_100a)"; }
OMCG_API const char* omcg_last_error(void) { return g_err.c_str(); }

OMCG_API int omcg_problem_create(int kind, uint64_t xs_seed, int host_threads, omcg_problem** out) {
    return wrap([&] {
        if (!out) throw std::invalid_argument("out is null");
        *out = nullptr;
        auto* h = new omcg_problem;
        try {
            omcg::build_problem(h->p, kind, xs_seed, host_threads);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

OMCG_API void omcg_problem_free(omcg_problem* p) { delete p; }

OMCG_API int omcg_problem_get_info(const omcg_problem* p, omcg_problem_info* info) {
    return wrap([&] {
        if (!p || !info) throw std::invalid_argument("null argument");
        std::memset(info, 0, sizeof *info);
        const omcg::Problem& P = p->p;
        info->kind = P.kind;
        info->n_nuclides = P.n_nuc;
        info->n_materials = (int)P.mat.size();
        info->nx = P.geo.nx;
        info->ny = P.geo.ny;
        info->n_tally_bins = P.geo.nx * P.geo.ny;
        info->fuel_nuclides = (int)P.mat[omcg::MAT_FUEL].nuc.size();
        info->n_grid_total = P.grid_points();
        info->lib_bytes = P.library_bytes();
        info->gen_seconds = P.gen_seconds;
    });
}

OMCG_API uint64_t omcg_library_checksum(const omcg_problem* p) {
    return p ? omcg::library_checksum(p->p) : 0;
}

OMCG_API int omcg_hash_build(const omcg_problem* p, int n_bins, int device, uint64_t* checksum, int32_t* hash_out) {
    return wrap([&] {
        if (!p || !checksum) throw std::invalid_argument("null argument");
        if (n_bins < 1 || n_bins > 1000000) throw std::invalid_argument("n_bins out of range [1, 1e6]");
        *checksum = omcg::device_hash_build(p->p, n_bins, device, hash_out);
    });
}

OMCG_API int omcg_div_check(int device, int64_t n, const double* a, const double* b, double* q_fast,
                            uint8_t* fast_ok, double* q_frac, double* q_ieee) {
    return wrap([&] {
        if (n < 0) throw std::invalid_argument("n < 0");
        if (n == 0) return;
        if (!a || !b || !q_fast || !fast_ok || !q_frac || !q_ieee) throw std::invalid_argument("null argument");
        omcg::device_div_check(device, n, a, b, q_fast, fast_ok, q_frac, q_ieee);
    });
}

OMCG_API int omcg_xs_lookup(const omcg_problem* p, int n_bins, int device, int64_t n, const int32_t* mat,
                            const double* E, double* out) {
    return wrap([&] {
        if (!p || (n > 0 && (!mat || !E || !out))) throw std::invalid_argument("null argument");
        if (n < 0) throw std::invalid_argument("n < 0");
        if (n == 0) return;
        omcg::device_xs_lookup(p->p, n_bins, device, n, mat, E, out);
    });
}

OMCG_API int omcg_xs_lookup_queue(const omcg_problem* p, int n_bins, int device, int64_t n, const int32_t* mat,
                                  const double* E, int64_t sort_threshold, double* out, double* ckpt_out) {
    return wrap([&] {
        if (!p || (n > 0 && (!mat || !E || !out))) throw std::invalid_argument("null argument");
        if (n < 0) throw std::invalid_argument("n < 0");
        if (n_bins < 1 || n_bins > 1000000) throw std::invalid_argument("n_bins out of range [1, 1e6]");
        if (n == 0) return;
        omcg::device_xs_lookup_queue(p->p, n_bins, device, n, mat, E, sort_threshold, out, ckpt_out);
    });
}
#ifndef OMCG_DEFAULT_DEVICE_SCHEDULE
#define OMCG_DEFAULT_DEVICE_SCHEDULE 0
#endif
OMCG_API void omcg_run_config_default(omcg_run_config* c) {
    if (!c) return;
    std::memset(c, 0, sizeof *c);
    // defaults of campaigns/openmc/space.json (Table 1)
    c->mode = OMCG_QUEUED;
    c->particles_in_flight = 1000000;
    c->n_bins = 4000;
    c->sort_threshold = 20000;
    c->host_threads = 8;
    c->tasks_per_gpu = 1;
    c->cpu_bind = OMCG_BIND_THREADS;
    // SMR-like assembly configuration C2
    c->n_particles = 1000000;
    c->n_batches = 15;
    c->n_inactive = 5;
    c->seed = 1;
    c->n_gpus = 1;
    for (int i = 0; i < 8; ++i) c->devices[i] = i;
    c->world_size = 1;
    c->rank = 0;
    c->tail_threshold = 16384;
    c->event_fusion = 1;
    c->move_event_cap = 20;
    c->device_schedule = OMCG_DEFAULT_DEVICE_SCHEDULE;
}

OMCG_API int omcg_run(const omcg_problem* p, const omcg_run_config* cfg, omcg_run_result* res, int64_t* tally_out,
                      omcg_record* records) {
    return wrap([&] {
        if (!p || !cfg || !res) throw std::invalid_argument("null argument");
        omcg::run_transport(p->p, *cfg, res, tally_out, records);
    });
}

OMCG_API int64_t omcg_queue_trace(int64_t* out, int64_t max_entries) {
    auto& t = omcg::last_queue_trace();
    int64_t n = (int64_t)t.size() / 3;
    if (out) {
        int64_t m = n < max_entries ? n : max_entries;
        std::memcpy(out, t.data(), sizeof(int64_t) * 3 * (size_t)m);
    }
    return n;
}

OMCG_API int omcg_nccl_unique_id(unsigned char out[128]) {
    return wrap([&] {
        if (!out) throw std::invalid_argument("null argument");
        omcg::nccl_unique_id(out);
    });
}

OMCG_API int omcg_energy_counter_mj(int device, uint64_t* mj) {
    return wrap([&] {
        if (!mj) throw std::invalid_argument("null argument");
        unsigned long long v = 0;
        if (!omcg::energy_counter_mj(device, &v)) throw omcg::IoError("NVML energy counter unavailable");
        *mj = (uint64_t)v;
    });
}
OMCG_API int omcg_release_devices(void) {
    return wrap([&] { omcg::release_devices(); });
}
OMCG_API int omcg_energy_mark(void) {
    return wrap([&] {
        if (!omcg::energy_mark()) throw omcg::IoError("NVML energy counters unavailable");
    });
}
OMCG_API int omcg_energy_since_mark_j(int device, double* joules) {
    return wrap([&] {
        if (!joules) throw std::invalid_argument("null argument");
        if (!omcg::energy_since_mark_j(device, joules))
            throw omcg::IoError("no NVML energy mark for this device (omcg_energy_mark not called, or NVML unavailable)");
    });
}
OMCG_API int omcg_bank_exchange_plan(const uint64_t* S_all, int world, int64_t n_batch, uint64_t off, int rank,
                                     int64_t* plan) {
    return wrap([&] {
        if (!S_all || !plan) throw std::invalid_argument("null argument");
        omcg::bank_exchange_plan(S_all, world, n_batch, off, rank, plan);
    });
}

OMCG_API int omcg_device_count(int* n) {
    return wrap([&] {
        if (!n) throw std::invalid_argument("null argument");
        *n = omcg::device_count();
    });
}

}  // extern "C"
