/*
 * atune_run.c — drive the reference autotuner (its own C ABI, include/autotune/
 * autotune.h) over a campaign file, unchanged. Used to run
 * proj/campaigns/openmc/campaign.json against this repo's bin/openmc on PATH:
 * the reference's SubprocessEvaluator renders openmc.sh.in, spawns it, parses
 * "FOM: ... particles/s" and (metric edp) metrics.txt (src/harness.cpp).
 *
 * usage: atune_run <campaign.json> <out_dir> [max_evals] [workers] [seed] [edp]
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "autotune/autotune.h"

int main(int argc, char** argv) {
    if (argc < 3) {
        fprintf(stderr, "usage: %s <campaign.json> <out_dir> [max_evals] [workers] [seed] [edp]\n", argv[0]);
        return 2;
    }
    atune_campaign* c = NULL;
    if (atune_campaign_load(argv[1], &c) != ATUNE_OK) {
        fprintf(stderr, "load: %s\n", atune_last_error());
        return 1;
    }
    if (argc > 3 && atune_campaign_set_max_evals(c, atoi(argv[3])) != ATUNE_OK) goto fail;
    if (argc > 4 && atune_campaign_set_workers(c, atoi(argv[4])) != ATUNE_OK) goto fail;
    if (argc > 5 && atune_campaign_set_seed(c, strtoull(argv[5], NULL, 10)) != ATUNE_OK) goto fail;
    char* report = NULL;
    int rc = atune_campaign_run(c, argv[2], &report);
    if (report) {
        printf("%s\n", report);
        atune_string_free(report);
    }
    if (rc != ATUNE_OK) fprintf(stderr, "run: %s\n", atune_last_error());
    atune_campaign_free(c);
    return rc == ATUNE_OK ? 0 : 1;
fail:
    fprintf(stderr, "override: %s\n", atune_last_error());
    atune_campaign_free(c);
    return 1;
}
