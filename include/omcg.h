/*
 * omcg.h — C ABI of the B200-native event-based Monte Carlo transport hot path
 * (libomcg.so). This is the "thin C-ABI layer" between the C++ host driver and
 * the sm_100a kernels named by BASELINE.json's north_star.
 *
 * What each entry point replaces in the reference (arxiv/paper_2402_09222,
 * /root/reference/proj):
 *   - The reference reaches the transport loop only through a process boundary:
 *     `openmc --event -i #P1 -b #P2 -m #P3` / `openmc-queueless --event -i #P1
 *     -b #P2` (campaigns/openmc/openmc.sh.in:5,7), FoM parsed from stdout with
 *     `FOM:\s*([0-9.eE+-]+)\s*particles/s` (campaigns/openmc/campaign.json:8,
 *     last match wins, src/harness.cpp:150-171), energy from metrics.txt
 *     (src/harness.cpp:117-136). omcg_run() is that binary's body: the
 *     `openmc` executable built from this repo (tools: bin/openmc) is a thin
 *     argv/env front end over it.
 *   - omcg_run_config mirrors the seven tuned parameters P0..P6
 *     (campaigns/openmc/space.json:3-9; Table 1).
 *   - Conventions follow the reference C ABI (include/autotune/autotune.h:13-41,
 *     src/capi.cpp:24-76): int return codes, no exception crosses the ABI,
 *     thread-local omcg_last_error(), opaque handles, only these symbols exported.
 *   - An in-process evaluator (the reference's Evaluator plugin type,
 *     src/harness.hpp:102) would call omcg_run() directly; see INTEGRATION.md.
 */
#ifndef OMCG_H
#define OMCG_H

#include <stddef.h>
#include <stdint.h>

#if defined(OMCG_BUILDING)
#define OMCG_API __attribute__((visibility("default")))
#else
#define OMCG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
    OMCG_OK = 0,
    OMCG_EINVAL = 1, /* invalid argument / configuration */
    OMCG_EIO = 2,    /* filesystem failure */
    OMCG_ECUDA = 3,  /* CUDA runtime / driver failure (no device, OOM, ...) */
    OMCG_ENCCL = 4,  /* NCCL failure */
    OMCG_EFAIL = 5   /* unexpected internal failure */
};

/* problem kinds: C1 pin cell, C2 17x17 assembly, C4 full core,
 * and an analytic infinite homogeneous medium of one energy-independent
 * nuclide (k_inf = nu*Sigma_f/Sigma_a = 1.5625) */
enum { OMCG_PINCELL = 0, OMCG_ASSEMBLY = 1, OMCG_CORE = 2, OMCG_INFINITE = 3 };
enum { OMCG_QUEUED = 0, OMCG_QUEUELESS = 1 };           /* P0 */
enum { OMCG_BIND_CORES = 0, OMCG_BIND_THREADS = 1, OMCG_BIND_SOCKETS = 2 }; /* P6 */
enum { OMCG_N_SCORES = 4 };   /* per pin: flux, absorption, fission, nu-fission */
enum { OMCG_MAX_BATCHES = 512 };

typedef struct omcg_problem omcg_problem;

typedef struct {
    int kind;
    int n_nuclides;
    int n_materials;
    int nx, ny;
    int n_tally_bins;      /* nx*ny pins; OMCG_N_SCORES scores each */
    int fuel_nuclides;
    int64_t n_grid_total;
    int64_t lib_bytes;     /* E + 4-channel rows, bytes */
    double gen_seconds;    /* host library generation time */
} omcg_problem_info;

typedef struct {
    /* tuned parameters (campaigns/openmc/space.json) */
    int mode;                     /* P0: OMCG_QUEUED ("openmc") or OMCG_QUEUELESS */
    int64_t particles_in_flight;  /* P1 (-i): in-flight bank slots per task */
    int n_bins;                   /* P2 (-b): log hash-grid bins */
    int64_t sort_threshold;       /* P3 (-m): sort fuel XS queue when len >= P3; <0 never */
    int host_threads;             /* P4 (-c): host threads for initialisation */
    int tasks_per_gpu;            /* P5 (--ntasks-per-gpu): concurrent sub-banks per GPU */
    int cpu_bind;                 /* P6 (--cpu-bind) */
    /* problem size */
    int64_t n_particles;          /* histories per batch (whole job) */
    int n_batches;
    int n_inactive;
    uint64_t seed;                /* transport master seed */
    /* placement: either n_gpus devices in this process (devices[] or 0..n-1),
     * or one rank of a multi-process job (world_size > 1, nccl_id set). */
    int n_gpus;
    int devices[8];
    int world_size;
    int rank;
    unsigned char nccl_id[128];
    /* diagnostics */
    int record_batch;             /* 1-based batch whose first record_n histories are recorded */
    int64_t record_n;
    int profile;                  /* CUDA-event timing: 1 every kernel class, 2 fuel calculate_xs only */
    int trace_queues;             /* record per-iteration (queue, length, id-checksum) */
    /* When the source is exhausted and at most tail_threshold histories are
     * alive, finish them in one history-per-thread launch instead of one
     * launch per event (results are identical; 0 disables). */
    int64_t tail_threshold;
    /* 0: one kernel per event type (advance, crossing, non-fuel and fuel
     * calculate_xs, collision): queued mode re-queues each history after every
     * event, queueless mode sweeps each of those kernels over all slots.
     * 1 (default): event fusion — the cheap events (advance, crossing,
     * non-fuel calculate_xs and collision) of a history run back to back in
     * one "move" kernel; only fuel calculate_xs and fuel collisions are
     * separate kernels (queued: separate queues; queueless: separate sweeps).
     * Results are identical either way. */
    int event_fusion;
    /* Event fusion, queued mode: a history runs at most this many events
     * (flights, crossings, non-fuel lookups) per move-kernel launch, then
     * rejoins the move queue for the next one; this bounds the launch's tail
     * of long flights through the moderator (default 20; 0: no cap). Results
     * are identical for every value; only the queue contents change. */
    int move_event_cap;
    /* 1: the per-batch exchanges (int64 tally/k all-reduce, bank-size
     * all-gather, fission-bank send/recv) go through NCCL even when this
     * process runs a single rank (a one-rank communicator), so the multi-GPU
     * data plane runs on one GPU. 0 (default): NCCL only between ranks on
     * different GPUs. Communicators are created once per placement and reused
     * by later calls in the same process. */
    int force_nccl;
    /* Queued mode with event fusion, once the source is exhausted: 1 (default)
     * lets the GPU apply the longest-queue rule itself — the kernel that ends
     * an iteration records the next choice, and the host enqueues candidate
     * kernels ahead without reading queue lengths back (a candidate that is
     * not the recorded choice returns at once). 0: the host reads the
     * lengths back and picks every iteration. Same iterations, same results. */
    int device_schedule;
} omcg_run_config;

typedef struct {
    int32_t n_xs, n_adv, n_cross, n_coll, n_sites, term;
    double e_final, x_final;
} omcg_record;

typedef struct {
    int n_batches_run;
    double k_coll[OMCG_MAX_BATCHES];
    double k_abs[OMCG_MAX_BATCHES];
    double k_track[OMCG_MAX_BATCHES];
    int64_t n_sites[OMCG_MAX_BATCHES];
    int64_t n_events[4];          /* xs, advance, cross, collision */
    int64_t n_leaked, n_absorbed, n_lost;
    double k_mean, k_std;
    double t_init;                /* upload + hash build + allocation, s */
    double t_active;              /* active batches, s (device-event timed, max over ranks) */
    double t_total;               /* all batches, s */
    double fom;                   /* n_particles * n_active / t_active */
    double energy_j;              /* NVML GPU energy over the call, J (0 if unavailable) */
    int64_t kernel_launches;      /* launches inside the active batches */
    int64_t kernel_launches_total;
    int64_t h2d_bytes, d2h_bytes; /* host<->device traffic of the call */
    /* profile (profile != 0): per kernel class, active batches */
    double prof_ms[8];            /* xs_fuel, xs_nonfuel, advance, cross, collision, sort, refill, tail */
    int64_t prof_launches[8];
    int64_t prof_items[8];        /* queue entries processed */
    double xs_fuel_bytes;         /* algorithmic bytes of the fuel XS launches */
    int64_t queue_iterations;     /* host event-loop iterations, all batches */
    int64_t sorts;                /* fuel-queue sorts performed */
    int64_t tail_launches;        /* history-per-thread tail launches */
} omcg_run_result;

OMCG_API const char* omcg_version(void);
OMCG_API const char* omcg_last_error(void);

/* ---- problem (host buffers) ---- */
OMCG_API int omcg_problem_create(int kind, uint64_t xs_seed, int host_threads, omcg_problem** out);
OMCG_API void omcg_problem_free(omcg_problem* p);
OMCG_API int omcg_problem_get_info(const omcg_problem* p, omcg_problem_info* info);
OMCG_API uint64_t omcg_library_checksum(const omcg_problem* p);

/* ---- device-side building blocks (parity hooks) ---- */
/* Build the log hash grid for n_bins on `device` and return its FNV-1a checksum
 * (same definition as the oracle's orc_hash_checksum); optionally copy it out
 * (n_nuclides*(n_bins+1) int32, nuclide-major). */
OMCG_API int omcg_hash_build(const omcg_problem* p, int n_bins, int device, uint64_t* checksum,
                             int32_t* hash_out);
/* Macroscopic XS for n (material, E) pairs through the calculate_xs kernel:
 * out = 4n doubles (total, absorption, fission, nu-fission). */
OMCG_API int omcg_xs_lookup(const omcg_problem* p, int n_bins, int device, int64_t n,
                            const int32_t* mat, const double* E, double* out);

/* The production fuel lookup (calculate_xs kernel k_xs_fuel_fused, the one
 * the queued loop launches) on a queue of n histories at (mat[i], E[i]),
 * queue entry i = history i; the queue is first sorted by (material, energy)
 * when n >= sort_threshold >= 0, as the queued loop does (P3). out: 4n doubles
 * (total, absorption, fission, nu-fission) as stored in each record;
 * ckpt_out (optional, 16n doubles): per history the folded running total
 * after each 16-nuclide segment but the last (the collision's sampling
 * checkpoints), unused entries NaN. Fails (OMCG_EFAIL) if the launch does not
 * hand every history on to the move queue exactly once. */
OMCG_API int omcg_xs_lookup_queue(const omcg_problem* p, int n_bins, int device, int64_t n, const int32_t* mat,
                                  const double* E, int64_t sort_threshold, double* out, double* ckpt_out);

/* Parity hook for the event kernels' branch-free fp64 divisions and square
 * roots: per pair on the device, q_fast[i] / fast_ok[i] = the
 * checked fast path a / b (div_chk) and its flag, q_frac[i] = the no-fallback
 * form (div_frac), q_ieee[i] = a / b; q_fast[n + i] / fast_ok[n + i] /
 * q_ieee[n + i] the same for sqrt(a) (sqrt_chk). q_fast, fast_ok and q_ieee
 * hold 2n entries, q_frac n. Contract: fast_ok => q_fast == q_ieee bit for
 * bit; q_frac == q_ieee on its domains (interpolation fractions, det_log).
 * No reference counterpart (test infrastructure, like omcg_xs_lookup). */
OMCG_API int omcg_div_check(int device, int64_t n, const double* a, const double* b, double* q_fast,
                            uint8_t* fast_ok, double* q_frac, double* q_ieee);

/* ---- the transport run (the `openmc --event` body) ---- */
OMCG_API void omcg_run_config_default(omcg_run_config* cfg);
OMCG_API int omcg_run(const omcg_problem* p, const omcg_run_config* cfg, omcg_run_result* res,
                      int64_t* tally_out, omcg_record* records);
/* Per-iteration queue trace of the last omcg_run with trace_queues != 0:
 * triples (queue id, length, checksum of particle ids). */
OMCG_API int64_t omcg_queue_trace(int64_t* out, int64_t max_entries);

/* Cumulative GPU energy counter of CUDA device `device` in millijoules (NVML
 * nvmlDeviceGetTotalEnergyConsumption). The `openmc` front end reads it right
 * after leasing its GPUs and again at exit, so metrics.txt covers the whole
 * evaluation process (library generation, upload, hash build, transport,
 * teardown) like the harness's elapsed time (proj/src/harness.cpp:311-323).
 * OMCG_EIO when NVML is unavailable. */
OMCG_API int omcg_energy_counter_mj(int device, uint64_t* mj);

/* Energy metering of a whole evaluation process. omcg_energy_mark() reads the
 * energy counter of every GPU NVML sees without initialising CUDA; the
 * `openmc` front end calls it first thing in main(), so that CUDA start-up,
 * library generation, upload, transport and teardown are all metered, like
 * the harness's elapsed time, which spans the whole process
 * (proj/src/harness.cpp:311-323). omcg_energy_since_mark_j() is the energy of
 * CUDA device `device` since the mark, in J. OMCG_EIO when NVML is
 * unavailable or no mark was taken. */
OMCG_API int omcg_energy_mark(void);
OMCG_API int omcg_energy_since_mark_j(int device, double* joules);

/* End of a process's GPU work: returns the pooled device memory and pinned
 * host words the library keeps between runs and destroys the CUDA contexts
 * of the devices it used, so that the `openmc` front end's teardown is metered
 * (it calls this before its final energy reading) instead of happening in the
 * process exit. No other omcg call may be in flight; problems stay valid and
 * later runs initialise the devices again. */
OMCG_API int omcg_release_devices(void);

/* NCCL unique id for a multi-process job (rank 0 creates, others receive). */
OMCG_API int omcg_nccl_unique_id(unsigned char out[128]);
OMCG_API int omcg_device_count(int* n);

/* Host-side fission-bank redistribution plan used between batches of a
 * multi-GPU run. S_all: canonical bank size of every rank;
 * off: the batch's resampling offset. plan (4*world+2 int64): send_first[w],
 * send_count[w], recv_first[w], recv_count[w], need_first, need_count. */
OMCG_API int omcg_bank_exchange_plan(const uint64_t* S_all, int world, int64_t n_batch, uint64_t off, int rank,
                                     int64_t* plan);

#ifdef __cplusplus
}
#endif
#endif /* OMCG_H */
