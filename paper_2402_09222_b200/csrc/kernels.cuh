// kernels.cuh — launch interface of the sm_100a event kernels (kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <atomic>

#include "device.cuh"

namespace omcg {

// Event queues of one sub-bank: N_QUEUES int32 lists of `cap` entries,
// contiguous (queue t at qbase + t*cap). Lengths of the live queues in
// count[0..4]; the dead queue is a ring whose tail lives on the device.
struct QueueSet {
    int32_t* qbase;
    int64_t cap;
    unsigned* count;
    unsigned long long* dead_tail;
    int adv_q;  // region receiving move-queue (EV_ADV) appends: EV_ADV or ADV_ALT (flips per capped move launch)
};
constexpr int ADV_ALT = 6;  // the second move-queue region (N_QUEUES + 1 regions are allocated)

// Device-driven queued loop (omcg_run_config.device_schedule): the kernel that
// completes an iteration applies the longest-queue rule itself (its last
// block, after every append) and writes the next iteration's choice here; the
// host enqueues candidate kernels ahead without reading counts back, and each
// candidate returns at once unless it is the recorded choice.
constexpr int SCHED_TAIL = 6;  // choice: few enough histories left for the tail kernel
constexpr int SCHED_DONE = 7;  // choice: every history of the sub-bank has finished
struct DevSched {
    int choice;      // EV_XS_FUEL / EV_ADV / EV_COLL, or SCHED_TAIL / SCHED_DONE
    int n;           // length of the chosen queue
    int n_front;     // collision queue: fuel entries at the front
    int sorted;      // fuel lookup: the queue is sorted first (n >= P3)
    int drain_q;     // move: region being drained
    int app_q;       // region receiving move-queue appends during this iteration
    int executed;    // iterations completed since the host handed over
    int cur;         // index of the current iteration (trace log)
    int sorts;       // sorted fuel lookups
    unsigned ticket; // last-block ticket of the running kernel
    unsigned long long chunk;  // work counter of the persistent fuel lookup
};

// Everything an event kernel needs, passed by value as the kernel parameter.
struct Ctx {
    QueueSet qs;
    unsigned long long* trace_chk;  // per-launch order-free checksum of processed histories
    DevLib lib;
    Geometry geo;  // geo.pin_map is a device pointer
    Bank b;
    Acc acc;
    int tally_on;
    int n_tally_bins;
    int tally_smem;       // 1: aggregate tallies in shared memory (few bins)
    unsigned long long* tally_priv;  // n_priv per-SM copies of the tally (folded per batch)
    int n_priv;
    double k_norm;
    int64_t rank_lo;      // batch-global index of this rank's first history
    int64_t n_batch;      // histories per batch, whole job
    int batch;            // 1-based
    uint64_t master;
    int64_t record_n;
    int recording;
    unsigned long long* ctrl;  // [0] refill ticket, [1] alive, [2] error flags, [3] tail list, [4] move chunks, [5] queueless lookup chunks
    int fused;                 // event fusion: non-fuel XS work goes to the move (advance) queue
    int move_cap;              // > 0: a history runs at most move_cap events per move launch, then rejoins the move queue
    // device-driven loop (nullptr: the host picks every iteration)
    DevSched* sched;
    int* sched_log;            // per iteration {choice, n} (max_iters entries)
    unsigned long long* sched_chk;  // trace mode: per-iteration id checksums
    int sched_max_iters;
    int sort_threshold;        // P3 (-1: never)
    int64_t tail_threshold;
};

constexpr int SMEM_TALLY_MAX = 64;  // tally bins*scores aggregated per block in smem (few-pin problems)

// bookkeeping: kernel launches are counted into the counter installed on the
// calling host thread (one per omcg_run), else into a process-wide counter
struct LaunchCounterScope {
    explicit LaunchCounterScope(std::atomic<long long>* c);
    ~LaunchCounterScope();
    LaunchCounterScope(const LaunchCounterScope&) = delete;
    LaunchCounterScope& operator=(const LaunchCounterScope&) = delete;
    std::atomic<long long>* prev;
};
long long launch_counter();

// library / hash
void launch_hash_build(const DevLib& lib, int32_t* hash, cudaStream_t s);
void launch_div_check(int64_t n, const double* a, const double* b, double* q_fast, uint8_t* ok, double* q_frac,
                      double* q_ieee, cudaStream_t s);
void launch_xs_pairs(const DevLib& lib, int64_t n, const int32_t* mat, const double* E, double* out,
                     cudaStream_t s);

// parity hook: slots 0..n-1 wait for calculate_xs at (mat[i], E[i]); q[i] = i
void launch_lookup_setup(const Ctx& c, int n, const int32_t* mat, const double* E, int32_t* q, cudaStream_t s);

// event kernels; q == nullptr selects the queueless variant over all cap slots
void launch_publish(const unsigned* count, unsigned* host, unsigned seq, cudaStream_t s);
void launch_init(const Ctx& c, uint64_t head, int n, int64_t first_local, const Site* src, cudaStream_t s);
// warp-per-history tail over the `live` remaining histories, listed into
// `list` first (ctrl[3] must be zero)
void launch_tail(const Ctx& c, bool queued, int64_t live, int32_t* list, cudaStream_t s);
void launch_refill_all(const Ctx& c, int64_t first_local, int64_t n_remaining, const Site* src,
                       cudaStream_t s);
void launch_xs(const Ctx& c, const int32_t* q, int n, cudaStream_t s);
// fuel-queue calculate_xs split by 16-nuclide segment in one launch: a block
// per 32 entries, segment partials in shared memory, in-order fold by warp 0
// (nseg <= 48); same arithmetic as launch_xs
void launch_xs_fuel_fused(const Ctx& c, const int32_t* q, int n, int nseg, cudaStream_t s);
void launch_advance(const Ctx& c, const int32_t* q, int n, cudaStream_t s);
void launch_cross(const Ctx& c, const int32_t* q, int n, cudaStream_t s);
// the collision queue is double-ended: n_front fuel entries at the front,
// n - n_front non-fuel entries at the back
void launch_collide(const Ctx& c, const int32_t* q, int n, int n_front, cudaStream_t s);

// fused transport: every history of the move queue runs advance / crossing /
// non-fuel calculate_xs / non-fuel collision in registers until it needs a
// fuel lookup, collides in fuel or dies
// (the queueless sweep, q == nullptr, runs the non-fuel collisions inside the
// loop too)
void launch_move(const Ctx& c, const int32_t* q, int n, cudaStream_t s);

// device-driven loop candidates (Ctx::sched set): each returns at once unless
// the recorded choice is its event; lengths come from the device
void launch_fuel_candidate(const Ctx& c, const int32_t* q_fuel, int32_t* q_sorted, int nseg, int n_fuel_mats,
                           unsigned int* hist, unsigned int* cursor, uint32_t* keys, unsigned int* bsum,
                           cudaStream_t s);
void launch_move_candidate(const Ctx& c, cudaStream_t s);
void launch_collide_candidate(const Ctx& c, cudaStream_t s);
// diagnostic build only (-DOMCG_MOVE_CYCLES): per-event-type cycle shares of k_move to stderr
void dump_move_cycles();
// diagnostic build only (-DOMCG_COOP_STATS): fuel-lookup blocks on the cooperative / per-lane path
void dump_coop_stats();
// diagnostic build only (-DOMCG_TAIL_CYCLES): per-event-type cycles of the tail's longest history to stderr
void dump_tail_cycles();

// material/energy sort of the fuel XS queue (16-bit energy radix per material)
void launch_sort(const Ctx& c, const int32_t* q_in, int32_t* q_out, int n, int n_fuel_mats,
                 unsigned int* hist, unsigned int* cursor, uint32_t* keys, unsigned int* bsum, cudaStream_t s);

// tally[i] += sum of the n_priv private copies; copies zeroed
void launch_tally_fold(unsigned long long* priv, int n_priv, int64_t n, unsigned long long* tally, cudaStream_t s);

// fission bank: canonical order + systematic resampling
void launch_scan_i32(const int32_t* in, int64_t* out, int64_t n, int64_t* tmp, cudaStream_t s);
void launch_bank_canon(const Site* bank, int64_t n_sites, const int64_t* offsets, int64_t rank_lo,
                       Site* canon, cudaStream_t s);
void launch_resample(const Site* src, int64_t src_first, uint64_t S, uint64_t off, int64_t n_batch,
                     int64_t rank_lo, int64_t n_local, Site* out, cudaStream_t s);

}  // namespace omcg
