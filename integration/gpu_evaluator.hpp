// gpu_evaluator.hpp — an in-process GPU evaluator for the reference autotuner.
//
// The reference knows two evaluator kinds (proj/src/campaign.hpp:16:
// EvaluatorKind { synthetic, subprocess }); make_evaluator
// (proj/src/campaign.cpp:250-254) turns a campaign definition into an
// `Evaluator` = std::function<ExecutionOutcome(const EvalRequest&)>
// (proj/src/harness.hpp:92-102). This is the third kind the survey names
// (SURVEY.md §8b "tertiary boundary", §8f-4): the configuration goes straight
// into omcg_run() (include/omcg.h) inside the tuner's process — no shell, no
// per-evaluation process, CUDA context or library generation.
//
// Contract kept (proj/src/ensemble.cpp:163-197): called concurrently from
// n_workers threads; never throws; any failure (bad configuration, CUDA or NCCL
// error, non-finite objective) is status fail with req.penalty. Concurrent
// evaluations lease GPUs in-process (one evaluation per device at a time, the
// in-process form of bin/openmc's flock lease), and `elapsed` starts once the
// GPU is leased, so the EDP objective (energy x elapsed, harness.cpp:311-323)
// never includes queueing behind another worker. There is no in-process
// timeout (a thread cannot be killed); the subprocess boundary keeps that.
#pragma once
#include <cstdint>
#include <string>

#include "harness.hpp"
#include "space.hpp"

namespace omcg_integration {

struct GpuEvalOptions {
    int problem_kind = 1;          // OMCG_ASSEMBLY
    uint64_t xs_seed = 1234;
    int64_t n_particles = 1000000;  // histories per batch
    int n_batches = 6;
    int n_inactive = 2;
    uint64_t seed = 1;
    int n_gpus_per_eval = 1;
};

// Reads OMCG_PROBLEM / OMCG_PARTICLES / OMCG_BATCHES / OMCG_INACTIVE / OMCG_SEED
// / OMCG_XS_SEED / OMCG_GPUS like bin/openmc does.
GpuEvalOptions options_from_env();

autotune::Evaluator make_gpu_evaluator(const autotune::ParameterSpace& space, autotune::MetricSpec metric,
                                       GpuEvalOptions opt);

}  // namespace omcg_integration
