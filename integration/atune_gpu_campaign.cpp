// atune_gpu_campaign — the reference tuner's campaign loop (proj/src/ensemble.cpp
// run_campaign, results.csv/trace.csv writers and report from proj/src/store.cpp,
// campaign file parsing from proj/src/campaign.cpp — all unchanged, linked from
// the reference's own sources) driving the in-process GPU evaluator
// (gpu_evaluator.hpp) instead of the subprocess one.
//
// usage: atune_gpu_campaign <campaign.json> <out_dir> [max_evals] [workers]
// The campaign file is the unchanged campaigns/openmc/campaign.json: its space,
// metric (fom | edp), seed and knobs are used; its mold/launcher are not
// (nothing is spawned). Problem size from OMCG_* (see bin/openmc).
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <filesystem>

#include "campaign.hpp"
#include "gpu_evaluator.hpp"
#include "store.hpp"

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s <campaign.json> <out_dir> [max_evals] [workers]\n", argv[0]);
        return 2;
    }
    try {
        autotune::CampaignDefinition def = autotune::load_campaign_file(argv[1]);
        autotune::CampaignOverrides ov;
        if (argc > 3) ov.max_evals = std::atoi(argv[3]);
        if (argc > 4) ov.workers = std::atoi(argv[4]);
        autotune::apply_overrides(def, ov);
        const std::filesystem::path out = argv[2];
        std::filesystem::create_directories(out);
        autotune::ResultsWriter writer(out / "results.csv", def.space);
        const autotune::Evaluator ev =
            omcg_integration::make_gpu_evaluator(def.space, def.metric, omcg_integration::options_from_env());
        const autotune::CampaignResult res = autotune::run_campaign(def.space, ev, def.config, &writer);
        autotune::write_trace_csv(out / "trace.csv", autotune::export_trace(res.records, def.baseline));
        std::printf("%s\n", autotune::render_report(def.space, res.records, def.config.direction, def.baseline).c_str());
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "atune_gpu_campaign: %s\n", e.what());
        return 1;
    }
}
