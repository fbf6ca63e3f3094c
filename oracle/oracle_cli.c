/*
 * oracle_cli.c — `openmc-oracle`: the CPU oracle behind the same command line
 * as the product binary (`--event -i P1 -b P2 [-m P3]`, campaigns/openmc/
 * openmc.sh.in:5,7). TEST / BASELINE INFRASTRUCTURE ONLY: used by bench.py's
 * cpu_baseline and --impl reference legs, never by the product.
 *
 * History-based, so -i (particles in flight) and -m (sort threshold) cannot
 * change its results [P213]; they are accepted and reported only.
 * Problem selection uses the same environment variables as the product:
 *   OMCG_PROBLEM=pincell|assembly|core   OMCG_PARTICLES   OMCG_BATCHES
 *   OMCG_INACTIVE   OMCG_SEED   OMCG_XS_SEED   OMCG_THREADS
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "omc_oracle.h"

static long env_long(const char* k, long d) {
    const char* v = getenv(k);
    return (v && *v) ? strtol(v, NULL, 10) : d;
}

int main(int argc, char** argv) {
    long inflight = 1000000, bins = 4000, sort_thr = -1;
    for (int i = 1; i < argc; ++i) {
        if (!strcmp(argv[i], "--event")) continue;
        if (!strcmp(argv[i], "-i") && i + 1 < argc) inflight = strtol(argv[++i], NULL, 10);
        else if (!strcmp(argv[i], "-b") && i + 1 < argc) bins = strtol(argv[++i], NULL, 10);
        else if (!strcmp(argv[i], "-m") && i + 1 < argc) sort_thr = strtol(argv[++i], NULL, 10);
        else {
            fprintf(stderr, "openmc-oracle: unknown argument '%s'\n", argv[i]);
            return 2;
        }
    }
    const char* prob = getenv("OMCG_PROBLEM");
    int kind = ORC_ASSEMBLY;
    if (prob && !strcmp(prob, "pincell")) kind = ORC_PINCELL;
    else if (prob && !strcmp(prob, "core")) kind = ORC_CORE;
    else if (prob && !strcmp(prob, "infinite")) kind = ORC_INFINITE;
    orc_problem* p = NULL;
    if (orc_problem_create(kind, (uint64_t)env_long("OMCG_XS_SEED", 1234), (int)bins, &p) != 0) {
        fprintf(stderr, "openmc-oracle: %s\n", orc_last_error());
        return 1;
    }
    orc_run_config cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.n_particles = env_long("OMCG_PARTICLES", 1000000);
    cfg.n_batches = (int)env_long("OMCG_BATCHES", 15);
    cfg.n_inactive = (int)env_long("OMCG_INACTIVE", 5);
    cfg.seed = (uint64_t)env_long("OMCG_SEED", 1);
    cfg.n_threads = (int)env_long("OMCG_THREADS", 0);
    orc_run_result res;
    if (orc_run(p, &cfg, &res, NULL, NULL) != 0) {
        fprintf(stderr, "openmc-oracle: %s\n", orc_last_error());
        orc_problem_free(p);
        return 1;
    }
    int nth = cfg.n_threads > 0 ? cfg.n_threads : (int)sysconf(_SC_NPROCESSORS_ONLN);
    fprintf(stderr, "oracle: problem=%d in_flight=%ld bins=%ld sort=%ld threads=%d\n", kind, inflight,
            bins, sort_thr, nth);
    for (int b = 0; b < res.n_batches_run; ++b)
        fprintf(stderr, "batch %3d  k_coll %.6f  k_abs %.6f  k_track %.6f  sites %lld\n", b + 1,
                res.k_coll[b], res.k_abs[b], res.k_track[b], (long long)res.n_sites[b]);
    fprintf(stderr, "k_eff (collision) = %.6f +/- %.6f ; events xs %lld adv %lld cross %lld coll %lld\n",
            res.k_mean, res.k_std, (long long)res.n_events[0], (long long)res.n_events[1],
            (long long)res.n_events[2], (long long)res.n_events[3]);
    printf("FOM: %.6e particles/s\n", res.fom);
    orc_problem_free(p);
    return 0;
}
