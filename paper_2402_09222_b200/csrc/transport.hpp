// transport.hpp — host driver of the event-based loop (C++), called by the C ABI.
#pragma once
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/omcg.h"
#include "problem.hpp"

namespace omcg {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void run_transport(const Problem& p, const omcg_run_config& cfg, omcg_run_result* res, int64_t* tally_out,
                   omcg_record* records);

uint64_t device_hash_build(const Problem& p, int n_bins, int device, int32_t* hash_out);
void device_div_check(int device, int64_t n, const double* a, const double* b, double* q_fast, uint8_t* ok,
                      double* q_frac, double* q_ieee);
void device_xs_lookup(const Problem& p, int n_bins, int device, int64_t n, const int32_t* mat, const double* E,
                      double* out);
void device_xs_lookup_queue(const Problem& p, int n_bins, int device, int64_t n, const int32_t* mat, const double* E,
                            int64_t sort_threshold, double* out, double* ckpt_out);

std::vector<int64_t>& last_queue_trace();
void bank_exchange_plan(const uint64_t* S_all, int world, int64_t n_batch, uint64_t off, int rank, int64_t* plan);
void nccl_unique_id(unsigned char out[128]);
int device_count();

// NVML cumulative energy of one CUDA device, mJ (false when unavailable)
bool energy_counter_mj(int cuda_device, unsigned long long* mj);
// process-start marks of every NVML device (no CUDA init), and the energy of
// one CUDA device since them, J (false when unavailable / not marked)
bool energy_mark();
void release_devices();  // return pooled memory and destroy the contexts (no call in flight)
bool energy_since_mark_j(int cuda_device, double* joules);

// NVML energy counter (dlopen'ed; returns false when unavailable)
struct EnergyMeter {
    bool start(const std::vector<int>& cuda_devices);
    double stop_joules();  // energy since start, summed over devices
    std::vector<void*> handles;
    std::vector<unsigned long long> start_mj;
    double t0 = 0.0;  // steady-clock seconds at start
    bool ok = false;
};

}  // namespace omcg
