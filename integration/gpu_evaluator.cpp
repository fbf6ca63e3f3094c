// gpu_evaluator.cpp — see gpu_evaluator.hpp.
#include "gpu_evaluator.hpp"

#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <variant>
#include <vector>

#include "omcg.h"

namespace omcg_integration {
namespace {

long long env_ll(const char* k, long long d) {
    const char* v = std::getenv(k);
    return (v && *v) ? std::strtoll(v, nullptr, 10) : d;
}

// In-process GPU lease: every device runs one evaluation at a time.
struct Leases {
    std::mutex mu;
    std::condition_variable cv;
    std::vector<bool> busy;
    std::vector<int> take(int n, int hint) {
        std::unique_lock<std::mutex> lk(mu);
        for (;;) {
            std::vector<int> got;
            const int nd = (int)busy.size();
            for (int k = 0; k < nd && (int)got.size() < n; ++k) {
                const int d = (hint + k) % nd;
                if (!busy[d]) got.push_back(d);
            }
            if ((int)got.size() == n) {
                for (int d : got) busy[d] = true;
                return got;
            }
            cv.wait(lk);
        }
    }
    void give(const std::vector<int>& d) {
        {
            std::lock_guard<std::mutex> lk(mu);
            for (int x : d) busy[x] = false;
        }
        cv.notify_all();
    }
};

struct Shared {
    GpuEvalOptions opt;
    autotune::ParameterSpace space;
    autotune::MetricSpec metric;
    std::once_flag once;
    omcg_problem* problem = nullptr;
    std::string problem_error;
    Leases leases;
    Shared(GpuEvalOptions o, autotune::ParameterSpace s, autotune::MetricSpec m)
        : opt(o), space(std::move(s)), metric(std::move(m)) {}
    ~Shared() { omcg_problem_free(problem); }
};

const autotune::Value* get(const autotune::ParameterSpace& space, const autotune::Configuration& cfg,
                           const char* name) {
    const auto i = space.index_of(name);
    if (!i || *i >= cfg.size() || !cfg[*i]) return nullptr;  // absent or inactive (P3 under queueless)
    return &*cfg[*i];
}
int64_t as_int(const autotune::Value* v, int64_t d) {
    if (!v) return d;
    if (auto p = std::get_if<std::int64_t>(v)) return *p;
    if (auto p = std::get_if<double>(v)) return (int64_t)*p;
    return std::strtoll(std::get<std::string>(*v).c_str(), nullptr, 10);
}
std::string as_str(const autotune::Value* v, const char* d) {
    if (!v) return d;
    if (auto p = std::get_if<std::string>(v)) return *p;
    return std::to_string(as_int(v, 0));
}

// campaigns/openmc/space.json P0..P6 -> omcg_run_config (the mapping bin/openmc
// applies to `openmc --event -i P1 -b P2 -m P3` and AUTOTUNE_LAUNCHER_ARGS)
omcg_run_config to_run_config(const Shared& S, const autotune::Configuration& c) {
    omcg_run_config r;
    omcg_run_config_default(&r);
    const std::string p0 = as_str(get(S.space, c, "P0"), "openmc");
    if (p0 == "openmc") r.mode = OMCG_QUEUED;
    else if (p0 == "openmc-queueless") r.mode = OMCG_QUEUELESS;
    else throw std::invalid_argument("P0 must be openmc or openmc-queueless, got " + p0);
    r.particles_in_flight = as_int(get(S.space, c, "P1"), r.particles_in_flight);
    r.n_bins = (int)as_int(get(S.space, c, "P2"), r.n_bins);
    const autotune::Value* p3 = get(S.space, c, "P3");
    r.sort_threshold = r.mode == OMCG_QUEUED && p3 ? as_int(p3, r.sort_threshold) : -1;
    r.host_threads = (int)as_int(get(S.space, c, "P4"), r.host_threads);
    r.tasks_per_gpu = (int)as_int(get(S.space, c, "P5"), r.tasks_per_gpu);
    const std::string p6 = as_str(get(S.space, c, "P6"), "threads");
    r.cpu_bind = p6 == "cores" ? OMCG_BIND_CORES : p6 == "sockets" ? OMCG_BIND_SOCKETS : OMCG_BIND_THREADS;
    r.n_particles = S.opt.n_particles;
    r.n_batches = S.opt.n_batches;
    r.n_inactive = S.opt.n_inactive;
    r.seed = S.opt.seed;
    r.n_gpus = S.opt.n_gpus_per_eval;
    return r;
}

}  // namespace

GpuEvalOptions options_from_env() {
    GpuEvalOptions o;
    const char* prob = std::getenv("OMCG_PROBLEM");
    if (prob && !std::strcmp(prob, "pincell")) o.problem_kind = OMCG_PINCELL;
    else if (prob && !std::strcmp(prob, "core")) o.problem_kind = OMCG_CORE;
    else if (prob && !std::strcmp(prob, "infinite")) o.problem_kind = OMCG_INFINITE;
    o.n_particles = env_ll("OMCG_PARTICLES", o.n_particles);
    o.n_batches = (int)env_ll("OMCG_BATCHES", o.n_batches);
    o.n_inactive = (int)env_ll("OMCG_INACTIVE", o.n_inactive);
    o.seed = (uint64_t)env_ll("OMCG_SEED", 1);
    o.xs_seed = (uint64_t)env_ll("OMCG_XS_SEED", 1234);
    o.n_gpus_per_eval = (int)env_ll("OMCG_GPUS", 1);
    return o;
}

autotune::Evaluator make_gpu_evaluator(const autotune::ParameterSpace& space, autotune::MetricSpec metric,
                                       GpuEvalOptions opt) {
    auto S = std::make_shared<Shared>(opt, space, std::move(metric));
    return [S](const autotune::EvalRequest& req) -> autotune::ExecutionOutcome {
        autotune::ExecutionOutcome out;
        out.status = autotune::EvalStatus::fail;
        out.objective = req.penalty;
        const auto t_req = std::chrono::steady_clock::now();
        auto since = [](std::chrono::steady_clock::time_point t0) {
            return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        };
        try {
            std::call_once(S->once, [&] {  // the library is generated once per campaign, not per evaluation
                int nd = 0;
                if (omcg_device_count(&nd) != OMCG_OK || nd < 1) {
                    S->problem_error = std::string("no CUDA device: ") + omcg_last_error();
                    return;
                }
                S->leases.busy.assign((size_t)nd, false);
                if (omcg_problem_create(S->opt.problem_kind, S->opt.xs_seed, 8, &S->problem) != OMCG_OK)
                    S->problem_error = std::string("problem: ") + omcg_last_error();
            });
            if (!S->problem) throw std::runtime_error(S->problem_error);
            omcg_run_config cfg = to_run_config(*S, req.config);
            if (cfg.n_gpus < 1 || cfg.n_gpus > (int)S->leases.busy.size()) throw std::invalid_argument("OMCG_GPUS");
            const std::vector<int> devs = S->leases.take(cfg.n_gpus, req.worker_id);
            struct Give {
                Leases& L;
                const std::vector<int>& d;
                ~Give() { L.give(d); }
            } give{S->leases, devs};
            for (int i = 0; i < cfg.n_gpus; ++i) cfg.devices[i] = devs[(size_t)i];
            const auto t_run = std::chrono::steady_clock::now();  // elapsed: from the lease on
            omcg_run_result res;
            const int rc = omcg_run(S->problem, &cfg, &res, nullptr, nullptr);
            out.elapsed = since(t_run);
            if (rc != OMCG_OK) return out;
            double obj = res.fom;
            switch (S->metric.kind) {
            case autotune::MetricKind::fom: obj = res.fom; break;
            case autotune::MetricKind::runtime: obj = out.elapsed; break;
            case autotune::MetricKind::energy: obj = res.energy_j; break;
            case autotune::MetricKind::edp: obj = res.energy_j * out.elapsed; break;
            }
            if (!std::isfinite(obj)) return out;
            out.objective = obj;
            out.status = autotune::EvalStatus::ok;
        } catch (...) {  // the Evaluator contract: failures are outcomes, never exceptions
            out.status = autotune::EvalStatus::fail;
            out.objective = req.penalty;
            if (out.elapsed == 0) out.elapsed = since(t_req);
        }
        return out;
    };
}

}  // namespace omcg_integration
