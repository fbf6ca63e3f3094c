/*
 * omc_oracle.h — CPU oracle for the event-based Monte Carlo transport hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in paper_2402_09222_b200/ links, loads or
 * calls this code; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may use it, and only as the checker or
 * the CPU baseline.
 *
 * PARITY STATUS: the transport arithmetic is "parity unpinned" against the
 * reference. arxiv/paper_2402_09222 (/root/reference) contains no transport
 * code: it launches an external OpenMC binary (proj/campaigns/openmc/
 * openmc.sh.in:5,7; SPEC.md:8 puts OpenMC out of scope). The semantics
 * restated here follow the paper's description of the tuned loop
 * (particles in flight, log hash grid, queued vs queueless,
 * sort threshold; FoM) and OpenMC's published design [ext].
 * What IS pinned against the reference: the seed-derivation stream
 * (derive_seed/splitmix64, proj/src/rng.hpp:10-25) that drives the synthetic
 * library generator, checked against the reference header compiled in
 * oracle/_ref, and the process boundary (FoM line, metrics.txt).
 *
 * This file is a plain-C, history-based restatement. The product is an
 * event-based CUDA implementation; because every history owns its own RNG
 * stream and tallies are int64 fixed point, both must agree bit-for-bit on
 * per-particle event counts, final states, tallies and k-eff.
 */
#ifndef OMC_ORACLE_H
#define OMC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_PINCELL = 0, ORC_ASSEMBLY = 1, ORC_CORE = 2, ORC_INFINITE = 3 };
/* ORC_INFINITE: analytic infinite medium, one energy-independent nuclide
 * (k_inf = ORC_INF_NU * ORC_INF_SIGMA_F / ORC_INF_SIGMA_A = 1.5625) */
#define ORC_INF_GRID 1001
#define ORC_INF_AWR 12.0
#define ORC_INF_SIGMA_T 1.0
#define ORC_INF_SIGMA_A 0.4
#define ORC_INF_SIGMA_F 0.25
#define ORC_INF_NU 2.5
enum { ORC_TERM_ABSORBED = 0, ORC_TERM_LEAKED = 1, ORC_TERM_LOST = 2 };
enum { ORC_N_SCORES = 4 }; /* flux, absorption, fission, nu-fission */
enum { ORC_MAX_BATCHES = 512 };

typedef struct orc_problem orc_problem;

typedef struct {
    int kind;
    int n_nuclides;      /* nuclides in this problem's library */
    int n_materials;
    int n_bins;          /* log hash-grid bins (P2) */
    int nx, ny;          /* global pin lattice */
    int n_tally_bins;    /* nx*ny pins (scores are ORC_N_SCORES per pin) */
    int fuel_material;   /* index of the (first) fissionable material */
    int fuel_nuclides;   /* nuclides in that material */
    int64_t n_grid_total;/* sum of grid points over nuclides */
    int64_t lib_bytes;   /* bytes of E + 4-channel rows */
    int64_t hash_bytes;  /* bytes of the hash index */
} orc_problem_info;

typedef struct {
    int64_t n_particles;   /* histories per batch */
    int n_batches;
    int n_inactive;
    uint64_t seed;         /* transport master seed */
    int n_threads;         /* <=0: all online cores */
    int record_batch;      /* batch (1-based) whose particles are recorded; 0 = none */
    int64_t record_n;      /* first record_n histories of that batch */
    int stop_after_batch;  /* >0: stop after this many batches (bounded sample) */
} orc_run_config;

typedef struct {
    int32_t n_xs, n_adv, n_cross, n_coll, n_sites, term;
    double e_final, x_final;
} orc_record;

typedef struct {
    int n_batches_run;
    double k_coll[ORC_MAX_BATCHES];
    double k_abs[ORC_MAX_BATCHES];
    double k_track[ORC_MAX_BATCHES];
    int64_t n_sites[ORC_MAX_BATCHES];     /* fission sites banked per batch */
    int64_t n_events[4];                  /* xs, advance, cross, collision over all batches */
    int64_t n_leaked, n_absorbed, n_lost;
    double k_mean, k_std;                 /* collision estimator over active batches */
    double t_active;                      /* seconds, active batches */
    double t_total;                       /* seconds, all batches */
    double fom;                           /* n_particles * n_active / t_active */
} orc_run_result;

/* ---- problem ---- */
int orc_problem_create(int kind, uint64_t xs_seed, int n_bins, orc_problem** out);
void orc_problem_free(orc_problem* p);
int orc_problem_get_info(const orc_problem* p, orc_problem_info* info);
/* FNV-1a over the bit patterns of every nuclide's energy grid and rows. */
uint64_t orc_library_checksum(const orc_problem* p);
/* FNV-1a over the hash index (int32). */
uint64_t orc_hash_checksum(const orc_problem* p);
int orc_nuclide_grid_size(const orc_problem* p, int nuc);
/* Copy one nuclide's grid: E[n], xs[4n] (total, absorption, fission, nu-fission). */
int orc_nuclide_copy(const orc_problem* p, int nuc, double* E, double* xs);
/* Copy the hash index of one nuclide: (n_bins+1) int32. */
int orc_hash_copy(const orc_problem* p, int nuc, int32_t* out);

/* ---- single lookups (golden vectors) ---- */
int orc_hash_bin(const orc_problem* p, double E);
int orc_micro_xs(const orc_problem* p, int nuc, double E, int32_t* idx, double xs[4]);
int orc_macro_xs(const orc_problem* p, int mat, double E, double xs[4]);
/* macro_xs + the folded total after each 16-nuclide segment but the last
 * (<= 16 values, count in *nck): what calculate_xs checkpoints for collision */
int orc_macro_xs_ckpt(const orc_problem* p, int mat, double E, double xs[4], double* ck, int* nck);
/* the same for n pairs: xs[4n], ck[16n], nck[n] */
int orc_macro_xs_ckpt_n(const orc_problem* p, int64_t n, const int32_t* mat, const double* E, double* xs,
                        double* ck, int32_t* nck);

/* ---- deterministic math + RNG (golden vectors) ---- */
double orc_log(double x);
double orc_exp(double x);
uint64_t orc_derive_seed(uint64_t base, uint64_t stream);
uint64_t orc_future_seed(uint64_t n, uint64_t seed);
double orc_prn(uint64_t* seed);
uint64_t orc_particle_seed(uint64_t master_seed, uint64_t particle_id);

/* ---- transport ---- */
/* tally_out: n_tally_bins*ORC_N_SCORES int64 fixed-point (2^-28) sums over
 * active batches (may be NULL). records: record_n entries (may be NULL). */
int orc_run(const orc_problem* p, const orc_run_config* cfg, orc_run_result* res,
            int64_t* tally_out, orc_record* records);

/* Queued-mode event-loop emulation of batch 1 (source = uniform fission
 * source): per iteration (queue id, length, sum of mix64(history+1)); queue 5
 * = tail (all live histories finished at once). Mirrors omcg_queue_trace. */
int orc_queue_trace(const orc_problem* p, int64_t n_particles, uint64_t seed, int64_t in_flight,
                    int64_t tail_threshold, int event_fusion, int move_cap, int64_t* out, int64_t max_entries,
                    int64_t* n_out);

const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
