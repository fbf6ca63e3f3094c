// transport.cu — host driver of the event-based transport loop on B200.
//
// One host thread per GPU (rank) and, inside it, P5 sub-banks ("tasks per
// GPU") each with its own CUDA stream, in-flight bank of P1
// slots, queues and host thread. Queued mode (P0 = "openmc") reads the queue
// lengths back after each compaction and launches the kernel of the longest
// queue, sorting the fuel XS queue first when its length >= P3; queueless
// mode (P0 = "openmc-queueless") sweeps all event kernels over every slot
// (PAPER.md:219-221). Between batches the rank reduces int64 tallies and
// k-eff accumulators with NCCL and redistributes the canonical fission bank.
#include <atomic>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <thread>

#include "kernels.cuh"
#include "nccl_api.hpp"
#include "transport.hpp"

namespace omcg {

// NVTX ranges (SURVEY.md §5 tracing): header-only NVTX3, one indirect call
// that returns at once unless a tool (nsys, ncu --nvtx) is attached. Every
// event-kernel launch of the queue loops is a range named by its kernel class
// (through Prof below); batches, init and the batch synchronisation are ranges too.
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};
const char* const kClassName[8] = {"calculate_xs fuel", "calculate_xs non-fuel", "advance / move",
                                   "surface_crossing", "collision", "sort fuel queue", "refill", "tail"};

inline NcclApi& nccl_checked() {
    NcclApi& a = nccl();
    if (!a.error.empty()) throw NcclError(a.error);
    return a;
}
}  // namespace omcg
// every NCCL call below goes through the dlopen'ed table
#define ncclGetUniqueId omcg::nccl_checked().GetUniqueId
#define ncclCommInitRank omcg::nccl_checked().CommInitRank
#define ncclCommInitAll omcg::nccl_checked().CommInitAll
#define ncclCommDestroy omcg::nccl_checked().CommDestroy
#define ncclCommAbort omcg::nccl_checked().CommAbort
#define ncclAllReduce omcg::nccl_checked().AllReduce
#define ncclAllGather omcg::nccl_checked().AllGather
#define ncclSend omcg::nccl_checked().Send
#define ncclRecv omcg::nccl_checked().Recv
#define ncclGroupStart omcg::nccl_checked().GroupStart
#define ncclGroupEnd omcg::nccl_checked().GroupEnd
#define ncclGetErrorString omcg::nccl_checked().GetErrorString

namespace omcg {

#define CK(x)                                                                                      \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess)                                                                     \
            throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_) + " (" __FILE__ ":" + \
                            std::to_string(__LINE__) + ")");                                       \
    } while (0)
#define NK(x)                                                                         \
    do {                                                                              \
        ncclResult_t r_ = (x);                                                        \
        if (r_ != ncclSuccess) throw NcclError(std::string(#x) + ": " + ncclGetErrorString(r_)); \
    } while (0)

using ull = unsigned long long;

namespace {

// queue trace of the calling thread's last omcg_run (trace_queues != 0)
thread_local std::vector<int64_t> t_trace;

// Device allocations owned by one object, freed on destruction. They come
// from the device's stream-ordered memory pool with the release threshold
// raised, so freeing returns the pages to the pool instead of unmapping them
// (a synchronous cudaFree of ~1 GB of bank buffers cost 0.04-0.7 s per run);
// a later run in the same process (the in-process evaluator, bench passes)
// reuses them. Allocated on the legacy stream and synchronised at once, so
// any stream may use the memory.
std::mutex g_pool_mu;
bool g_pool_done[64] = {};  // devices whose pool threshold is raised (= devices this process used)
void keep_pool_memory(int device) {
    std::mutex& mu = g_pool_mu;
    bool* done = g_pool_done;
    std::lock_guard<std::mutex> lk(mu);
    if (device < 0 || device >= 64 || done[device]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    done[device] = true;
}
// Pinned host words (queue lengths, control flags) read back every
// iteration. Kept for the life of the process and reused by later runs:
// cudaFreeHost synchronises the device and measured 0-0.5 s per call.
struct PinnedSlab {
    std::mutex mu;
    std::vector<void*> free_blocks;  // 64-byte blocks
    void* get() {
        std::lock_guard<std::mutex> lk(mu);
        if (!free_blocks.empty()) {
            void* p = free_blocks.back();
            free_blocks.pop_back();
            return p;
        }
        void* p = nullptr;
        CK(cudaMallocHost(&p, 64));
        return p;
    }
    void put(void* p) {
        if (!p) return;
        std::lock_guard<std::mutex> lk(mu);
        free_blocks.push_back(p);
    }
    void release() {  // (no run in flight) free every block
        std::lock_guard<std::mutex> lk(mu);
        for (void* p : free_blocks) cudaFreeHost(p);
        free_blocks.clear();
    }
};
PinnedSlab& pinned() {
    static PinnedSlab* s = new PinnedSlab();  // never destroyed (process lifetime)
    return *s;
}

struct DevArena {
    std::vector<void*> ptrs;
    int device = 0;
    template <typename T>
    T* alloc(int64_t n) {
        void* p = nullptr;
        if (n <= 0) n = 1;
        keep_pool_memory(device);
        CK(cudaMallocAsync(&p, sizeof(T) * (size_t)n, 0));
        CK(cudaStreamSynchronize(0));  // usable from any stream from here on
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    ~DevArena() {
        if (ptrs.empty()) return;
        cudaSetDevice(device);
        for (void* p : ptrs) cudaFreeAsync(p, 0);
    }
};

bool env_flag(const char* name);  // unset or nonzero -> true

// Library + hash grid + geometry resident in one GPU's HBM.
struct GpuProblem {
    DevArena arena;
    DevLib lib{};
    Geometry geo{};
    int n_fuel_mats = 0;
    int max_fuel_seg = 1;  // 16-nuclide segments of the largest fuel-queue material
    std::vector<double> host_dens;  // lib.host_dens points here (lifetime of the upload)
    int64_t h2d_bytes = 0;

    void upload(const Problem& p, int n_bins, int device, cudaStream_t s) {
        arena.device = device;
        if (n_bins < 1 || n_bins > 1000000) throw std::invalid_argument("n_bins (P2) out of range [1, 1e6]");
        const int nn = p.n_nuc, nm = (int)p.mat.size();
        std::vector<int32_t> goff(nn + 1);
        for (int i = 0; i <= nn; ++i) goff[i] = (int32_t)p.goff[i];
        std::vector<int32_t> moff(nm + 1), mnuc;
        std::vector<double> mdens;
        std::vector<uint8_t> mfis(nm), mfuel(nm), mrank(nm);
        int fuel_rank = 0;
        for (int m = 0; m < nm; ++m) {
            moff[m] = (int32_t)mnuc.size();
            for (size_t i = 0; i < p.mat[m].nuc.size(); ++i) {
                mnuc.push_back(p.mat[m].nuc[i]);
                mdens.push_back(p.mat[m].dens[i]);
            }
            mfis[m] = p.mat[m].fissionable;
            mfuel[m] = p.mat[m].fissionable;  // fissionable materials use the fuel XS queue
            mrank[m] = p.mat[m].fissionable ? (uint8_t)fuel_rank++ : 0;
        }
        moff[nm] = (int32_t)mnuc.size();
        n_fuel_mats = std::max(1, fuel_rank);
        for (int m = 0; m < nm; ++m)
            if (mfuel[m])
                max_fuel_seg = std::max(max_fuel_seg, (int)((p.mat[m].nuc.size() + CKPT_STRIDE - 1) / CKPT_STRIDE));
        std::vector<int4> mdesc(mnuc.size());
        for (size_t i = 0; i < mnuc.size(); ++i) {
            int n = mnuc[i];
            mdesc[i] = make_int4(goff[n], goff[n + 1] - goff[n], n * (n_bins + 1), n);
        }
        static const bool pin_lib = env_flag("OMCG_PIN_LIBRARY");
        if (pin_lib) {  // page-lock the two big host arrays once per problem (best effort)
            std::lock_guard<std::mutex> lk(p.pins.mu);
            auto pin = [](const void* ptr, size_t bytes, std::shared_ptr<void>& guard) {
                if (guard || bytes == 0) return;
                void* q = const_cast<void*>(ptr);
                if (cudaHostRegister(q, bytes, cudaHostRegisterDefault) == cudaSuccess)
                    guard.reset(q, [](void* r) { cudaHostUnregister(r); });
                else
                    cudaGetLastError();
            };
            pin(p.E.data(), sizeof(double) * p.E.size(), p.pins.E);
            pin(p.xs.data(), sizeof(XS4) * p.xs.size(), p.pins.xs);
        }
        auto up = [&](auto* dst, const auto* src, size_t n) {
            size_t bytes = sizeof(*src) * n;
            CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
            h2d_bytes += (int64_t)bytes;
        };
        int32_t* d_goff = arena.alloc<int32_t>(nn + 1);
        // rows, then grid energies, then the hash grid: one allocation
        const int64_t npts = p.grid_points();
        const int64_t hash_n = (int64_t)(n_bins + 1) * nn;
        char* d_lib = arena.alloc<char>(npts * (int64_t)(sizeof(double) + sizeof(XS4)) +
                                        hash_n * (int64_t)sizeof(int32_t) + 256);
        XS4* d_xs = reinterpret_cast<XS4*>(d_lib);
        double* d_E = reinterpret_cast<double*>(d_lib + npts * (int64_t)sizeof(XS4));
        double* d_awr = arena.alloc<double>(nn);
        int32_t* d_moff = arena.alloc<int32_t>(nm + 1);
        int32_t* d_mnuc = arena.alloc<int32_t>((int64_t)mnuc.size());
        int4* d_mdesc = arena.alloc<int4>((int64_t)mdesc.size());
        double* d_mdens = arena.alloc<double>((int64_t)mdens.size());
        uint8_t* d_mfis = arena.alloc<uint8_t>(nm);
        uint8_t* d_mfuel = arena.alloc<uint8_t>(nm);
        uint8_t* d_mrank = arena.alloc<uint8_t>(nm);
        uint8_t* d_pin = arena.alloc<uint8_t>((int64_t)p.pin_map_host.size());
        int32_t* d_hash = reinterpret_cast<int32_t*>(d_E + npts);  // right after the energies
        up(d_goff, goff.data(), goff.size());
        up(d_E, p.E.data(), p.E.size());
        up(d_xs, p.xs.data(), p.xs.size());
        up(d_awr, p.awr.data(), p.awr.size());
        up(d_moff, moff.data(), moff.size());
        up(d_mnuc, mnuc.data(), mnuc.size());
        up(d_mdesc, mdesc.data(), mdesc.size());
        up(d_mdens, mdens.data(), mdens.size());
        up(d_mfis, mfis.data(), mfis.size());
        up(d_mfuel, mfuel.data(), mfuel.size());
        up(d_mrank, mrank.data(), mrank.size());
        up(d_pin, p.pin_map_host.data(), p.pin_map_host.size());
        const double log_emin = det_log(E_MIN);
        const double ln_range = det_log(E_MAX) - log_emin;
        lib.n_nuc = nn;
        lib.n_bins = n_bins;
        lib.n_mat = nm;
        lib.inv_spacing = (double)n_bins / ln_range;
        lib.log_emin = log_emin;
        lib.goff = d_goff; lib.E = d_E; lib.xs = d_xs; lib.hash = d_hash; lib.awr = d_awr;
        lib.mat_off = d_moff; lib.mat_nuc = d_mnuc; lib.mat_desc = d_mdesc; lib.mat_dens = d_mdens;
        lib.mat_fissionable = d_mfis; lib.mat_fuel = d_mfuel; lib.mat_sort_rank = d_mrank;
        host_dens = mdens;  // launch-parameter copy of the densities (fuel lookup)
        lib.host_dens = host_dens.data();
        lib.n_dens = (int)host_dens.size();
        launch_hash_build(lib, d_hash, s);
        CK(cudaGetLastError());
        if ((int64_t)p.geo.nx * p.geo.ny > (1 << 20))  // cell_xy's exact range (kernels.cu)
            throw std::invalid_argument("more than 2^20 lattice cells");
        geo = p.geo;
        geo.pin_map = d_pin;
    }
};

constexpr int SCHED_RING = 8;       // read-backs of the schedule record in flight
constexpr int SCHED_LOG = 1 << 16;  // iterations per device-driven stretch

struct SubBank {
    cudaStream_t stream = nullptr;
    Bank b{};
    QueueSet qs{};
    int32_t* q_sorted = nullptr;
    int32_t* tail_list = nullptr;  // live slots for the warp-per-history tail
    uint32_t* keys = nullptr;
    unsigned* hist = nullptr;
    unsigned* cursor = nullptr;
    unsigned* bsum = nullptr;
    unsigned* h_counts = nullptr;  // pinned: live queue lengths [0..4], then dead tail (as 2 words)
    unsigned* d_h_counts = nullptr;  // its device alias (k_publish writes words 0-7, then the sequence word 8)
    unsigned pub_seq = 0;
    uint64_t dead_head = 0;        // ring head (host side; only the refill consumes)
    ull* ctrl = nullptr;           // [0] ticket [1] alive [2] errors
    ull* h_ctrl = nullptr;         // pinned
    ull* trace_chk = nullptr;
    ull* h_trace_chk = nullptr;
    int64_t lo = 0, hi = 0;        // rank-local history range
    int64_t tail_launches = 0;
    int prof_level = 0;
    std::vector<int64_t> trace;
    // profile
    struct EvPair {
        cudaEvent_t a = nullptr, b = nullptr;
        int cls = 0;
        int64_t items = 0;
    };
    std::vector<EvPair> evs;  // deferred per-kernel timing, read after each host sync
    int n_pending = 0;
    int n_done = 0;  // pending pairs known complete (recorded before the last host sync)
    double prof_ms[8] = {};
    int64_t prof_launches[8] = {};
    int64_t prof_items[8] = {};
    double xs_fuel_bytes = 0.0;
    int64_t iterations = 0, sorts = 0;
    // device-driven queued loop: schedule record, per-iteration log and
    // checksums, pinned read-back ring
    DevSched* sched = nullptr;
    int* sched_log = nullptr;
    ull* sched_chk = nullptr;
    DevSched* h_sched[SCHED_RING + 1] = {};
    cudaEvent_t sched_ev[SCHED_RING] = {};
};

struct BatchComm;

struct Rank {
    int device = 0, rank = 0, world = 1;
    ncclComm_t comm = nullptr;
    BatchComm* bc = nullptr;          // per-batch collectives (NCCL or in-process loopback)
    std::atomic<long long>* launches = nullptr;  // the call's kernel-launch counter
    std::vector<ull> sall;            // bank sizes of all ranks, this batch
    DevArena arena;
    GpuProblem gp;
    Acc acc{};
    int n_tally_bins = 0;
    int64_t N = 0, N_rank = 0, rank_lo = 0, bank_cap = 0;
    Site* source = nullptr;
    Site* canon = nullptr;
    Site* recv = nullptr;
    int64_t* scan_out = nullptr;
    int64_t* scan_tmp = nullptr;
    ull* d_sall = nullptr;  // allgathered bank counts
    ull* tally_priv = nullptr;  // per-SM private tally copies
    int n_priv = 0;
    double* d_time = nullptr;
    cudaStream_t main = nullptr;
    cudaEvent_t ev_a0 = nullptr, ev_a1 = nullptr;
    std::vector<SubBank> subs;
    std::vector<DevArena> sub_arenas;
    // host results
    std::vector<int64_t> tally_total;
    double k_coll[OMCG_MAX_BATCHES] = {}, k_abs[OMCG_MAX_BATCHES] = {}, k_track[OMCG_MAX_BATCHES] = {};
    int64_t n_sites[OMCG_MAX_BATCHES] = {};
    int64_t counts[7] = {};
    int batches_run = 0;
    double t_active = 0.0, t_init = 0.0;
    long long launches_active = 0;
    int64_t h2d = 0, d2h = 0;
    std::string error;
};

// ------------------------------------------------------------------ setup
void setup_rank(Rank& R, const Problem& p, const omcg_run_config& cfg) {
    auto t0 = std::chrono::steady_clock::now();
    static const bool trace_init = std::getenv("OMCG_TRACE_INIT") != nullptr;
    auto mark = [&](const char* what) {
        if (!trace_init) return;
        cudaDeviceSynchronize();
        std::fprintf(stderr, "[omcg init] %-28s %8.3f s\n", what,
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    };
    CK(cudaSetDevice(R.device));
    mark("set device");
    R.arena.device = R.device;
    CK(cudaStreamCreateWithFlags(&R.main, cudaStreamNonBlocking));
    CK(cudaEventCreate(&R.ev_a0));
    CK(cudaEventCreate(&R.ev_a1));
    mark("streams/events");
    {
        Nvtx r("init: library upload + hash build");
        R.gp.upload(p, cfg.n_bins, R.device, R.main);
    }
    mark("library upload + hash");
    R.h2d += R.gp.h2d_bytes;
    R.N = cfg.n_particles;
    R.rank_lo = R.N * R.rank / R.world;
    R.N_rank = R.N * (R.rank + 1) / R.world - R.rank_lo;
    R.n_tally_bins = p.geo.nx * p.geo.ny;
    R.bank_cap = 3 * R.N_rank + 4096;
    R.acc.tally = R.arena.alloc<ull>(4 * (int64_t)R.n_tally_bins);
    {   // per-SM private copies (bounded to 64 MB) unless tallies fit in shared memory
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, R.device);
        const int64_t per = 4 * (int64_t)R.n_tally_bins * (int64_t)sizeof(ull);
        R.n_priv = 4 * R.n_tally_bins <= SMEM_TALLY_MAX
                       ? 0
                       : (int)std::max<int64_t>(1, std::min<int64_t>(sms, (64LL << 20) / per));
        if (R.n_priv > 0) {
            R.tally_priv = R.arena.alloc<ull>((int64_t)R.n_priv * 4 * R.n_tally_bins);
            CK(cudaMemset(R.tally_priv, 0, (size_t)R.n_priv * (size_t)per));
        }
    }
    R.acc.k = R.arena.alloc<ull>(3);
    R.acc.counts = R.arena.alloc<ull>(8);
    R.acc.bank = R.arena.alloc<Site>(R.bank_cap);
    R.acc.bank_count = R.arena.alloc<ull>(1);
    R.acc.bank_cap = R.bank_cap;
    R.acc.sites_pp = R.arena.alloc<int32_t>(R.N_rank);
    R.acc.records = nullptr;
    if (cfg.record_batch > 0 && cfg.record_n > 0) R.acc.records = R.arena.alloc<omcg_record>(cfg.record_n);
    R.source = R.arena.alloc<Site>(R.N_rank);
    R.canon = R.arena.alloc<Site>(R.bank_cap);
    if (R.bc) R.recv = R.arena.alloc<Site>(R.bank_cap + R.N_rank);
    R.scan_out = R.arena.alloc<int64_t>(R.N_rank);
    R.scan_tmp = R.arena.alloc<int64_t>((R.N_rank + 1023) / 1024 + 1);
    R.d_sall = R.arena.alloc<ull>(R.world);
    R.d_time = R.arena.alloc<double>(1);
    R.tally_total.assign(4 * (size_t)R.n_tally_bins, 0);
    mark("rank buffers");

    const int tasks = std::max(1, cfg.tasks_per_gpu);
    R.subs.resize(tasks);
    R.sub_arenas.resize(tasks);
    for (int t = 0; t < tasks; ++t) {
        SubBank& S = R.subs[t];
        DevArena& A = R.sub_arenas[t];
        A.device = R.device;
        S.lo = R.N_rank * t / tasks;
        S.hi = R.N_rank * (t + 1) / tasks;
        int64_t cap = std::min<int64_t>(std::max<int64_t>(cfg.particles_in_flight, 1), std::max<int64_t>(S.hi - S.lo, 1));
        if (cap > (int64_t)1 << 30) throw std::invalid_argument("particles in flight too large");
        S.b.cap = cap;
        S.prof_level = cfg.profile;
        CK(cudaStreamCreateWithFlags(&S.stream, cudaStreamNonBlocking));
        Bank& B = S.b;
        B.p = A.alloc<PState>(cap);
        B.cnt = A.alloc<int4>(cap);
        B.xc = A.alloc<XsCache>(cap);
        B.event = A.alloc<int8_t>(cap);
        B.ckpt = A.alloc<double>((int64_t)NCKPT * cap);
        CK(cudaMemsetAsync(B.event, EV_DEAD, (size_t)cap, S.stream));
        S.qs.cap = cap;
        S.qs.qbase = A.alloc<int32_t>((int64_t)(N_QUEUES + 1) * cap);  // + the second move-queue region
        S.qs.adv_q = EV_ADV;
        S.qs.count = A.alloc<unsigned>(8);  // [0..4] live lengths, [6..7] dead tail (u64)
        S.qs.dead_tail = reinterpret_cast<ull*>(S.qs.count + 6);
        {   // every slot starts in the dead ring
            std::vector<int32_t> iota((size_t)cap);
            for (int64_t i = 0; i < cap; ++i) iota[(size_t)i] = (int32_t)i;
            CK(cudaMemcpy(S.qs.qbase + (int64_t)EV_DEAD * cap, iota.data(), sizeof(int32_t) * (size_t)cap,
                          cudaMemcpyHostToDevice));
            unsigned init_counts[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            ull tail = (ull)cap;
            std::memcpy(init_counts + 6, &tail, sizeof tail);
            CK(cudaMemcpy(S.qs.count, init_counts, sizeof init_counts, cudaMemcpyHostToDevice));
            S.dead_head = 0;
        }
        S.q_sorted = A.alloc<int32_t>(cap);
        S.tail_list = A.alloc<int32_t>(cap);
        S.keys = A.alloc<uint32_t>(cap);
        S.hist = A.alloc<unsigned>((int64_t)R.gp.n_fuel_mats * 65536);
        S.cursor = A.alloc<unsigned>((int64_t)R.gp.n_fuel_mats * 65536);
        S.bsum = A.alloc<unsigned>((int64_t)R.gp.n_fuel_mats * 64);
        CK(cudaMemsetAsync(S.hist, 0, sizeof(unsigned) * (size_t)R.gp.n_fuel_mats * 65536, S.stream));
        S.ctrl = A.alloc<ull>(8);
        S.trace_chk = A.alloc<ull>(1);
        CK(cudaMemsetAsync(S.ctrl, 0, sizeof(ull) * 8, S.stream));
        S.h_counts = static_cast<unsigned*>(pinned().get());  // 8 words
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&S.d_h_counts), S.h_counts, 0));
        S.h_counts[8] = S.pub_seq = 0;
        S.h_ctrl = static_cast<ull*>(pinned().get());         // 4 words
        S.h_trace_chk = static_cast<ull*>(pinned().get());
        S.sched = A.alloc<DevSched>(1);
        S.sched_log = A.alloc<int>(2 * (int64_t)SCHED_LOG);
        S.sched_chk = A.alloc<ull>(SCHED_LOG);
        static_assert(sizeof(DevSched) <= 64, "schedule record must fit a pinned block");
        for (auto& h : S.h_sched) h = static_cast<DevSched*>(pinned().get());
        for (auto& e : S.sched_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        S.evs.resize(64);
        for (auto& e : S.evs) {
            CK(cudaEventCreate(&e.a));
            CK(cudaEventCreate(&e.b));
        }
        CK(cudaStreamSynchronize(S.stream));
        mark("sub-bank");
    }
    CK(cudaStreamSynchronize(R.main));
    R.t_init = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void teardown_rank(Rank& R) {
    cudaSetDevice(R.device);
    static const bool trace_init = std::getenv("OMCG_TRACE_INIT") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (trace_init)
            std::fprintf(stderr, "[omcg teardown] %-22s %8.3f s\n", what,
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    };
    for (auto& S : R.subs) {
        if (S.stream) cudaStreamDestroy(S.stream);
        mark("stream");
        pinned().put(S.h_counts);
        pinned().put(S.h_ctrl);
        pinned().put(S.h_trace_chk);
        for (auto& h : S.h_sched) pinned().put(h);
        for (auto& e : S.sched_ev)
            if (e) cudaEventDestroy(e);
        mark("host buffers");
        for (auto& e : S.evs) {
            if (e.a) cudaEventDestroy(e.a);
            if (e.b) cudaEventDestroy(e.b);
        }
    }
    mark("events");
    if (R.main) cudaStreamDestroy(R.main);
    if (R.ev_a0) cudaEventDestroy(R.ev_a0);
    if (R.ev_a1) cudaEventDestroy(R.ev_a1);
    mark("main stream");
}

// ------------------------------------------------------------------ event loops
bool env_flag(const char* name) {  // unset or nonzero -> true
    const char* v = std::getenv(name);
    return !v || std::atoi(v) != 0;
}

// Per-kernel CUDA-event timing on the launching stream. Events are recorded
// around each launch and read back only after the loop's next host sync, so
// profiling adds two event records per launch and no extra synchronisation.
void drain_profile(SubBank& S) {
    if (S.n_pending == 0) return;
    CK(cudaEventSynchronize(S.evs[S.n_pending - 1].b));
    static const bool log = std::getenv("OMCG_PROF_LOG") != nullptr;  // per-launch lines to stderr
    for (int i = 0; i < S.n_pending; ++i) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, S.evs[i].a, S.evs[i].b));
        if (log) std::fprintf(stderr, "[launch] class %d items %lld ms %.4f\n", S.evs[i].cls, (long long)S.evs[i].items, ms);
        S.prof_ms[S.evs[i].cls] += ms;
        S.prof_launches[S.evs[i].cls] += 1;
        S.prof_items[S.evs[i].cls] += S.evs[i].items;
    }
    S.n_pending = 0;
    S.n_done = 0;
}

// The pairs recorded before the last host sync are complete: read them while
// the GPU runs the kernel just launched (no wait, off the host's critical
// path between a read-back and the next launch), keep the newer ones.
void drain_done(SubBank& S) {
    const int k = S.n_done;
    if (k == 0) return;
    static const bool log = std::getenv("OMCG_PROF_LOG") != nullptr;
    for (int i = 0; i < k; ++i) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, S.evs[i].a, S.evs[i].b));
        if (log) std::fprintf(stderr, "[launch] class %d items %lld ms %.4f\n", S.evs[i].cls, (long long)S.evs[i].items, ms);
        S.prof_ms[S.evs[i].cls] += ms;
        S.prof_launches[S.evs[i].cls] += 1;
        S.prof_items[S.evs[i].cls] += S.evs[i].items;
    }
    std::rotate(S.evs.begin(), S.evs.begin() + k, S.evs.begin() + S.n_pending);
    S.n_pending -= k;
    S.n_done = 0;
}

struct Prof {
    SubBank& S;
    bool on;
    Nvtx range;
    // profile level 1 times every kernel class; level 2 only the fuel calculate_xs
    Prof(SubBank& s, bool enabled, int cls, int64_t items)
        : S(s), on(enabled && (S.prof_level == 1 || cls == 0)), range(kClassName[cls]) {
        if (!on) return;
        if (S.n_pending == (int)S.evs.size()) drain_profile(S);
        auto& e = S.evs[S.n_pending];
        e.cls = cls;
        e.items = items;
        CK(cudaEventRecord(e.a, S.stream));
    }
    ~Prof() {
        if (!on) return;
        if (cudaEventRecord(S.evs[S.n_pending].b, S.stream) == cudaSuccess) S.n_pending++;
    }
};

// Device-driven stretch of the queued loop (cfg.device_schedule, event fusion,
// source exhausted): the host hands the current choice to the GPU, then keeps
// enqueueing candidates in the usual order of a history's cycle (fuel lookup,
// move, collision, move) without waiting; the kernel that ends an iteration
// records the next choice (the same longest-queue rule), candidates that are
// not the recorded choice return at once. The schedule record is read back
// asynchronously; the stretch ends when the GPU records "tail" or "done".
// Returns with the stream synchronised and c.qs.adv_q updated.
void run_device_loop(Rank& R, SubBank& S, Ctx& c, const omcg_run_config& cfg, bool prof, int fuel_nuc, int best,
                     int n, const int64_t* qlen) {
    const bool trace = cfg.trace_queues != 0;
    DevSched& h = *S.h_sched[SCHED_RING];
    h = DevSched{};
    h.choice = best;
    h.n = n;
    h.n_front = (int)S.h_counts[EV_COLL];
    h.sorted = best == EV_XS_FUEL && cfg.sort_threshold >= 0 && qlen[best] >= cfg.sort_threshold ? 1 : 0;
    h.sorts = h.sorted;
    h.app_q = h.drain_q = c.qs.adv_q;
    if (best == EV_ADV && c.move_cap) h.app_q = c.qs.adv_q == EV_ADV ? ADV_ALT : EV_ADV;
    CK(cudaMemcpyAsync(S.sched, &h, sizeof(DevSched), cudaMemcpyHostToDevice, S.stream));
    if (trace) CK(cudaMemsetAsync(S.sched_chk, 0, sizeof(ull) * SCHED_LOG, S.stream));
    Ctx cs = c;
    cs.sched = S.sched;
    cs.sched_log = S.sched_log;
    cs.sched_chk = trace ? S.sched_chk : nullptr;
    cs.sched_max_iters = SCHED_LOG;
    cs.sort_threshold = cfg.sort_threshold >= 0 && cfg.sort_threshold < (1LL << 31) ? (int)cfg.sort_threshold
                        : cfg.sort_threshold < 0 ? -1 : 0x7fffffff;
    cs.tail_threshold = cfg.tail_threshold;
    cs.trace_chk = nullptr;
    const int32_t* q_fuel = S.qs.qbase + (int64_t)EV_XS_FUEL * S.qs.cap;
    static const int pattern[4] = {EV_XS_FUEL, EV_ADV, EV_COLL, EV_ADV};
    int pos = best == EV_XS_FUEL ? 0 : best == EV_ADV ? 1 : 2;
    int64_t w = 0, r = 0, last_exec = -1, stale = 0;
    bool stop = false;
    while (!stop) {
        for (int j = 0; j < 4; ++j, ++pos) {
            const int k = pattern[pos & 3];
            Prof pf(S, prof, k == EV_XS_FUEL ? 0 : k == EV_ADV ? 2 : 4, 0);
            if (k == EV_XS_FUEL)
                launch_fuel_candidate(cs, q_fuel, S.q_sorted, R.gp.max_fuel_seg, R.gp.n_fuel_mats, S.hist, S.cursor,
                                      S.keys, S.bsum, S.stream);
            else if (k == EV_ADV)
                launch_move_candidate(cs, S.stream);
            else
                launch_collide_candidate(cs, S.stream);
        }
        const int slot = (int)(w % SCHED_RING);
        CK(cudaMemcpyAsync(S.h_sched[slot], S.sched, sizeof(DevSched), cudaMemcpyDeviceToHost, S.stream));
        CK(cudaEventRecord(S.sched_ev[slot], S.stream));
        ++w;
        while (r < w) {  // look at the read-backs that have landed (wait only when the ring is full)
            const int rs = (int)(r % SCHED_RING);
            if (w - r >= SCHED_RING) CK(cudaEventSynchronize(S.sched_ev[rs]));
            else if (cudaEventQuery(S.sched_ev[rs]) != cudaSuccess) {
                cudaGetLastError();
                break;
            }
            const DevSched& x = *S.h_sched[rs];
            ++r;
            if (x.choice < SCHED_TAIL && (x.n < 0 || x.n > S.qs.cap))
                throw std::logic_error("device-driven queue loop: queue " + std::to_string(x.choice) + " length " +
                                       std::to_string(x.n) + " at iteration " + std::to_string(x.executed));
            if (x.choice >= SCHED_TAIL) {
                stop = true;
                break;
            }
            if (x.executed == last_exec) {
                if (++stale > 64) throw CudaError("device-driven queue loop made no progress");
            } else {
                stale = 0;
                last_exec = x.executed;
            }
        }
    }
    CK(cudaStreamSynchronize(S.stream));
    DevSched fin;
    CK(cudaMemcpy(&fin, S.sched, sizeof(DevSched), cudaMemcpyDeviceToHost));
    if (fin.choice < SCHED_TAIL) throw CudaError("device-driven queue loop stopped early");
    if (prof) drain_profile(S);
    S.iterations += fin.executed;
    S.sorts += fin.sorts;
    c.qs.adv_q = fin.app_q;
    // the iterations' (queue, length): the host's own first entry, the rest from the device log
    std::vector<int> log(2 * (size_t)std::max(fin.executed, 1));
    if (fin.executed > 1)
        CK(cudaMemcpy(log.data() + 2, S.sched_log + 2, sizeof(int) * 2 * (size_t)(fin.executed - 1),
                      cudaMemcpyDeviceToHost));
    log[0] = best;
    log[1] = n;
    if (prof)
        for (int i = 0; i < fin.executed; ++i)
            if (log[2 * i] == EV_XS_FUEL) S.xs_fuel_bytes += (double)log[2 * i + 1] * (44.0 + 100.0 * (double)fuel_nuc);
    if (trace) {
        std::vector<ull> chk((size_t)fin.executed);
        if (fin.executed > 0)
            CK(cudaMemcpy(chk.data(), S.sched_chk, sizeof(ull) * (size_t)fin.executed, cudaMemcpyDeviceToHost));
        for (int i = 0; i < fin.executed; ++i) {
            S.trace.push_back(log[2 * i]);
            S.trace.push_back(log[2 * i + 1]);
            S.trace.push_back((int64_t)chk[(size_t)i]);
        }
    }
}

// Spin until k_publish's sequence word arrives; poll the stream now and then so
// a failed kernel (which never publishes) surfaces as an error instead of a hang.
void wait_published(SubBank& S) {
    volatile unsigned* h = S.h_counts;
    for (unsigned spins = 1;; ++spins) {
        if (h[8] == S.pub_seq) break;
        if ((spins & 1023u) == 0) {
            const cudaError_t e = cudaStreamQuery(S.stream);
            if (e != cudaSuccess && e != cudaErrorNotReady) CK(e);
            if (e == cudaSuccess && h[8] != S.pub_seq)
                throw std::logic_error("queue-length read-back: stream idle without the published counts");
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
}

void run_queued(Rank& R, SubBank& S, Ctx c, const Site* src, const omcg_run_config& cfg, bool prof,
                int fuel_nuc) {
    int64_t next = S.lo;
    const bool trace = cfg.trace_queues != 0;
    const int64_t tail = cfg.tail_threshold;
    bool pending_trace = false;
    // A fuel calculate_xs launch moves every one of its n entries to the move
    // queue (count[EV_ADV] += n, count[EV_XS_FUEL] = 0) and changes nothing
    // else, so after such an iteration (without a refill) the host knows the
    // next queue lengths exactly and skips the read-back and its sync.
    bool known = false, check_prediction = false;
    unsigned predicted[8];
    for (;;) {
        if (!known && !pending_trace) {
            // k_publish writes the counts to page-locked memory; spin on its sequence word
            launch_publish(S.qs.count, S.d_h_counts, ++S.pub_seq, S.stream);
            wait_published(S);
            S.n_done = S.n_pending;
            if (check_prediction && std::memcmp(predicted, S.h_counts, sizeof predicted) != 0)
                throw std::logic_error("queue-length prediction after a fuel calculate_xs launch was wrong");
            check_prediction = false;
        } else if (!known) {
            CK(cudaMemcpyAsync(S.h_counts, S.qs.count, sizeof(unsigned) * 8, cudaMemcpyDeviceToHost, S.stream));
            if (pending_trace)
                CK(cudaMemcpyAsync(S.h_trace_chk, S.trace_chk, sizeof(ull), cudaMemcpyDeviceToHost, S.stream));
            CK(cudaStreamSynchronize(S.stream));
            S.n_done = S.n_pending;  // read after the next launch (drain_done)
            if (check_prediction && std::memcmp(predicted, S.h_counts, sizeof predicted) != 0)
                throw std::logic_error("queue-length prediction after a fuel calculate_xs launch was wrong");
            check_prediction = false;
        }
        known = false;
        if (pending_trace) {
            S.trace.back() = (int64_t)S.h_trace_chk[0];
            pending_trace = false;
        }
        // queue lengths; the collision queue is double-ended (front count[4], back count[5])
        int64_t qlen[EV_DEAD];
        for (int k = 0; k < EV_DEAD; ++k) qlen[k] = S.h_counts[k];
        qlen[EV_COLL] += S.h_counts[5];
        int64_t live = 0;
        for (int k = 0; k < EV_DEAD; ++k) live += qlen[k];
        ull dead_tail;
        std::memcpy(&dead_tail, S.h_counts + 6, sizeof dead_tail);
        const int64_t dead = (int64_t)(dead_tail - S.dead_head);
        if (live == 0 && next >= S.hi) break;
        if (live > 0) {
            S.iterations++;
            if (trace) {
                CK(cudaMemsetAsync(S.trace_chk, 0, sizeof(ull), S.stream));
                c.trace_chk = S.trace_chk;
            }
            int best = 0;
            for (int k = 1; k < EV_DEAD; ++k)
                if (qlen[k] > qlen[best]) best = k;
            int n = (int)qlen[best];
            if (cfg.device_schedule && c.fused && next >= S.hi && live > tail &&
                (best == EV_XS_FUEL || best == EV_ADV || best == EV_COLL)) {
                S.iterations--;  // counted by the device-driven stretch
                c.trace_chk = nullptr;
                run_device_loop(R, S, c, cfg, prof, fuel_nuc, best, n, qlen);
                known = false;
                continue;
            }
            if (next >= S.hi && live <= tail) {
                // sparse end of the batch: one launch finishes every live history
                best = EV_DEAD;
                n = (int)live;
                CK(cudaMemsetAsync(S.ctrl + 3, 0, sizeof(ull), S.stream));
                Prof pf(S, prof, 7, live);
                launch_tail(c, true, live, S.tail_list, S.stream);
                S.tail_launches++;
            } else {
                const int32_t* qptr = S.qs.qbase + (int64_t)(best == EV_ADV ? c.qs.adv_q : best) * S.qs.cap;
                switch (best) {
                case EV_XS_FUEL:
                    if (cfg.sort_threshold >= 0 && n >= cfg.sort_threshold) {
                        Prof pf(S, prof, 5, n);
                        launch_sort(c, qptr, S.q_sorted, n, R.gp.n_fuel_mats, S.hist, S.cursor, S.keys, S.bsum,
                                    S.stream);
                        qptr = S.q_sorted;
                        S.sorts++;
                    }
                    {
                        Prof pf(S, prof, 0, n);
                        launch_xs_fuel_fused(c, qptr, n, R.gp.max_fuel_seg, S.stream);
                    }
                    if (prof) S.xs_fuel_bytes += (double)n * (44.0 + 100.0 * (double)fuel_nuc);
                    if (c.fused && !(dead > 0 && next < S.hi)) {
                        S.h_counts[EV_ADV] += (unsigned)n;  // the move queue receives every entry
                        S.h_counts[EV_XS_FUEL] = 0u;
                        if (trace) {  // trace mode reads back anyway and checks the prediction
                            std::memcpy(predicted, S.h_counts, sizeof predicted);
                            check_prediction = true;
                        } else {
                            known = true;
                        }
                    }
                    break;
                case EV_XS_NONFUEL: { Prof pf(S, prof, 1, n); launch_xs(c, qptr, n, S.stream); } break;
                case EV_ADV: {
                    Prof pf(S, prof, 2, n);
                    if (c.fused && c.move_cap)  // capped histories go to the other region
                        c.qs.adv_q = c.qs.adv_q == EV_ADV ? ADV_ALT : EV_ADV;
                    if (c.fused) launch_move(c, qptr, n, S.stream);
                    else launch_advance(c, qptr, n, S.stream);
                } break;
                case EV_CROSS: { Prof pf(S, prof, 3, n); launch_cross(c, qptr, n, S.stream); } break;
                default: {
                    Prof pf(S, prof, 4, n);
                    launch_collide(c, qptr, n, (int)S.h_counts[EV_COLL], S.stream);
                } break;
                }
            }
            c.trace_chk = nullptr;
            if (trace) {
                S.trace.push_back(best);
                S.trace.push_back(n);
                S.trace.push_back(0);
                pending_trace = true;
            }
        }
        // refill the in-flight bank from the dead ring
        if (dead > 0 && next < S.hi) {
            int n = (int)std::min<int64_t>(dead, S.hi - next);
            Prof pf(S, prof, 6, n);
            launch_init(c, S.dead_head, n, next, src, S.stream);
            S.dead_head += (uint64_t)n;
            next += n;
        }
        if (prof) drain_done(S);
    }
    if (prof) drain_profile(S);
}

void run_queueless(Rank& R, SubBank& S, Ctx c, const Site* src, bool prof, int64_t tail) {
    int64_t next = S.lo;
    for (;;) {
        int64_t remaining = S.hi - next;
        if (remaining > 0) {
            CK(cudaMemsetAsync(S.ctrl, 0, sizeof(ull), S.stream));
            Prof pf(S, prof, 6, S.b.cap);
            launch_refill_all(c, next, remaining, src, S.stream);
        }
        if (c.fused) {  // sweeps of the fused kernels: fuel lookups, move, fuel collisions
            const int cap = (int)S.b.cap;
            { Prof pf(S, prof, 0, cap); launch_xs_fuel_fused(c, nullptr, cap, R.gp.max_fuel_seg, S.stream); }
            { Prof pf(S, prof, 2, cap); launch_move(c, nullptr, cap, S.stream); }
            { Prof pf(S, prof, 4, cap); launch_collide(c, nullptr, 0, 0, S.stream); }
        } else {
            { Prof pf(S, prof, 0, S.b.cap); launch_xs(c, nullptr, 0, S.stream); }
            { Prof pf(S, prof, 2, S.b.cap); launch_advance(c, nullptr, 0, S.stream); }
            { Prof pf(S, prof, 3, S.b.cap); launch_cross(c, nullptr, 0, S.stream); }
            { Prof pf(S, prof, 4, S.b.cap); launch_collide(c, nullptr, 0, 0, S.stream); }
        }
        CK(cudaMemcpyAsync(S.h_ctrl, S.ctrl, sizeof(ull) * 3, cudaMemcpyDeviceToHost, S.stream));
        CK(cudaStreamSynchronize(S.stream));
        if (prof) drain_profile(S);
        S.iterations++;
        if (remaining > 0) next += std::min<int64_t>((int64_t)S.h_ctrl[0], remaining);
        const int64_t alive = (int64_t)S.h_ctrl[1];
        if (alive == 0 && next >= S.hi) break;
        if (next >= S.hi && alive <= tail) {
            CK(cudaMemsetAsync(S.ctrl + 3, 0, sizeof(ull), S.stream));
            Prof pf(S, prof, 7, alive);
            launch_tail(c, false, alive, S.tail_list, S.stream);
            S.tail_launches++;
            CK(cudaStreamSynchronize(S.stream));
            break;
        }
    }
}

// ------------------------------------------------------------------ collectives
// The three per-batch exchanges of the multi-rank path:
// exact int64 sums of k/counters/tallies + all-gather of bank sizes; the
// canonical fission-bank slices of bank_exchange_plan; max of the timed region.
struct BatchComm {
    virtual ~BatchComm() = default;
    virtual void reduce_batch(Rank& R, bool active) = 0;  // fills R.sall
    virtual void exchange(Rank& R, const int64_t* plan) = 0;
    virtual double max_over_ranks(Rank& R, double v) = 0;
};

// NCCL over NVLink between ranks on different GPUs.
struct NcclBatchComm : BatchComm {
    // self_p2p: a rank's own slice of the canonical bank also goes through
    // ncclSend/ncclRecv (to itself) instead of a device copy, so a one-rank
    // communicator (force_nccl) runs the point-to-point exchange on hardware
    explicit NcclBatchComm(bool self_p2p = false) : self_p2p(self_p2p) {}
    bool self_p2p;
    void reduce_batch(Rank& R, bool active) override {
        NK(ncclGroupStart());
        NK(ncclAllReduce(R.acc.k, R.acc.k, 3, ncclUint64, ncclSum, R.comm, R.main));
        NK(ncclAllReduce(R.acc.counts, R.acc.counts, 8, ncclUint64, ncclSum, R.comm, R.main));
        if (active)
            NK(ncclAllReduce(R.acc.tally, R.acc.tally, 4 * (size_t)R.n_tally_bins, ncclUint64, ncclSum, R.comm,
                             R.main));
        NK(ncclAllGather(R.acc.bank_count, R.d_sall, 1, ncclUint64, R.comm, R.main));
        NK(ncclGroupEnd());
        R.sall.resize(R.world);
        CK(cudaMemcpyAsync(R.sall.data(), R.d_sall, sizeof(ull) * R.world, cudaMemcpyDeviceToHost, R.main));
        CK(cudaStreamSynchronize(R.main));
    }
    void exchange(Rank& R, const int64_t* plan) override {
        const int W = R.world;
        NK(ncclGroupStart());
        for (int r = 0; r < W; ++r) {
            int64_t sf = plan[r], sc = plan[W + r], rf = plan[2 * W + r], rc = plan[3 * W + r];
            if (r == R.rank && !self_p2p) {
                if (sc > 0)
                    CK(cudaMemcpyAsync(R.recv + rf, R.canon + sf, sizeof(Site) * (size_t)sc, cudaMemcpyDeviceToDevice,
                                       R.main));
                continue;
            }
            if (sc > 0) NK(ncclSend(R.canon + sf, sizeof(Site) * (size_t)sc, ncclChar, r, R.comm, R.main));
            if (rc > 0) NK(ncclRecv(R.recv + rf, sizeof(Site) * (size_t)rc, ncclChar, r, R.comm, R.main));
        }
        NK(ncclGroupEnd());
    }
    double max_over_ranks(Rank& R, double v) override {
        CK(cudaMemcpyAsync(R.d_time, &v, sizeof(double), cudaMemcpyHostToDevice, R.main));
        NK(ncclAllReduce(R.d_time, R.d_time, 1, ncclFloat64, ncclMax, R.comm, R.main));
        CK(cudaMemcpyAsync(&v, R.d_time, sizeof(double), cudaMemcpyDeviceToHost, R.main));
        CK(cudaStreamSynchronize(R.main));
        return v;
    }
};

// In-process loopback for ranks that share one GPU (devices[] with repeats):
// the same exchanges through host staging and device-to-device pulls, so the
// multi-rank path (partition, reductions, bank redistribution) runs and is
// tested on a single B200.
struct LoopbackShared {
    int world = 1;
    std::mutex mu;
    std::condition_variable cv;
    int count = 0;
    uint64_t gen = 0;
    bool aborted = false;  // a rank failed: every barrier throws instead of waiting for it
    std::vector<std::vector<ull>> host;
    std::vector<Site*> canon;
    std::vector<double> vals;
    explicit LoopbackShared(int w) : world(w), host(w), canon(w), vals(w) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (aborted) throw std::runtime_error("another rank of this run failed");
        const uint64_t g = gen;
        if (++count == world) {
            count = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g || aborted; });
            if (gen == g) throw std::runtime_error("another rank of this run failed");
        }
    }
    void abort() {
        std::lock_guard<std::mutex> lk(mu);
        aborted = true;
        cv.notify_all();
    }
};

struct LoopbackBatchComm : BatchComm {
    LoopbackShared* sh;
    explicit LoopbackBatchComm(LoopbackShared* s) : sh(s) {}
    void reduce_batch(Rank& R, bool active) override {
        const size_t nt = active ? 4 * (size_t)R.n_tally_bins : 0;
        std::vector<ull>& h = sh->host[R.rank];
        h.assign(3 + 8 + nt + 1, 0);
        CK(cudaMemcpyAsync(h.data(), R.acc.k, sizeof(ull) * 3, cudaMemcpyDeviceToHost, R.main));
        CK(cudaMemcpyAsync(h.data() + 3, R.acc.counts, sizeof(ull) * 8, cudaMemcpyDeviceToHost, R.main));
        if (nt) CK(cudaMemcpyAsync(h.data() + 11, R.acc.tally, sizeof(ull) * nt, cudaMemcpyDeviceToHost, R.main));
        CK(cudaMemcpyAsync(h.data() + 11 + nt, R.acc.bank_count, sizeof(ull), cudaMemcpyDeviceToHost, R.main));
        CK(cudaStreamSynchronize(R.main));
        sh->barrier();
        std::vector<ull> sum(11 + nt, 0);
        R.sall.assign(R.world, 0);
        for (int r = 0; r < R.world; ++r) {
            for (size_t i = 0; i < sum.size(); ++i) sum[i] += sh->host[r][i];
            R.sall[r] = sh->host[r][11 + nt];
        }
        sh->barrier();  // every rank has read the staging before it is reused
        CK(cudaMemcpyAsync(R.acc.k, sum.data(), sizeof(ull) * 3, cudaMemcpyHostToDevice, R.main));
        CK(cudaMemcpyAsync(R.acc.counts, sum.data() + 3, sizeof(ull) * 8, cudaMemcpyHostToDevice, R.main));
        if (nt) CK(cudaMemcpyAsync(R.acc.tally, sum.data() + 11, sizeof(ull) * nt, cudaMemcpyHostToDevice, R.main));
        CK(cudaMemcpyAsync(R.d_sall, R.sall.data(), sizeof(ull) * R.world, cudaMemcpyHostToDevice, R.main));
        CK(cudaStreamSynchronize(R.main));
    }
    void exchange(Rank& R, const int64_t* plan) override {
        const int W = R.world;
        CK(cudaStreamSynchronize(R.main));  // canonical bank complete
        sh->canon[R.rank] = R.canon;
        sh->barrier();
        std::vector<uint64_t> G(W + 1, 0);
        for (int r = 0; r < W; ++r) G[r + 1] = G[r] + R.sall[r];
        const uint64_t my_a = (uint64_t)plan[4 * W];
        for (int r = 0; r < W; ++r) {
            const int64_t rf = plan[2 * W + r], rc = plan[3 * W + r];
            if (rc > 0)
                CK(cudaMemcpyAsync(R.recv + rf, sh->canon[r] + (my_a + (uint64_t)rf - G[r]), sizeof(Site) * (size_t)rc,
                                   cudaMemcpyDeviceToDevice, R.main));
        }
        CK(cudaStreamSynchronize(R.main));
        sh->barrier();  // all pulls done before any rank rewrites its canonical bank
    }
    double max_over_ranks(Rank& R, double v) override {
        sh->vals[R.rank] = v;
        sh->barrier();
        double m = v;
        for (double x : sh->vals) m = std::max(m, x);
        sh->barrier();
        return m;
    }
};

// NCCL communicators cost tens to hundreds of ms to create, so they are kept
// for the life of the process and reused by later omcg_run calls with the
// same placement (an in-process evaluator or bench pass calls omcg_run many
// times). A communicator is leased by one call at a time; a concurrent call
// with the same placement gets its own. One that saw a failure is aborted and
// dropped.
struct CommCache {
    struct Entry {
        std::string key;
        std::vector<ncclComm_t> comms;
        bool busy = false;
    };
    std::mutex mu;
    std::vector<std::unique_ptr<Entry>> entries;
};
CommCache& comm_cache() {
    static CommCache* c = new CommCache();  // process lifetime
    return *c;
}

struct CommLease {
    CommCache::Entry* e = nullptr;
    std::vector<ncclComm_t> comms;
    std::atomic<bool> aborted{false};

    CommCache::Entry* find_or_add(const std::string& key, bool& fresh) {
        CommCache& C = comm_cache();
        std::lock_guard<std::mutex> lk(C.mu);
        for (auto& x : C.entries)
            if (x->key == key && !x->busy) {
                x->busy = true;
                fresh = false;
                return x.get();
            }
        C.entries.emplace_back(new CommCache::Entry());
        CommCache::Entry* x = C.entries.back().get();
        x->key = key;
        x->busy = true;
        fresh = true;
        return x;
    }
    void drop_entry() {
        CommCache& C = comm_cache();
        std::lock_guard<std::mutex> lk(C.mu);
        for (size_t i = 0; i < C.entries.size(); ++i)
            if (C.entries[i].get() == e) {
                C.entries.erase(C.entries.begin() + (long)i);
                break;
            }
        e = nullptr;
    }
    // one rank of a multi-process job (ncclCommInitRank)
    void acquire_rank(const unsigned char id_bytes[128], int world, int rank, int device) {
        char hex[2 * 128 + 1];
        for (int i = 0; i < 128; ++i) std::snprintf(hex + 2 * i, 3, "%02x", id_bytes[i]);
        const std::string key = "rank " + std::to_string(world) + ":" + std::to_string(rank) + ":" +
                                std::to_string(device) + ":" + hex;
        bool fresh = false;
        e = find_or_add(key, fresh);
        if (fresh) {
            try {
                ncclUniqueId id;
                std::memcpy(id.internal, id_bytes, 128);
                ncclComm_t c = nullptr;
                CK(cudaSetDevice(device));
                NK(ncclCommInitRank(&c, world, id, rank));
                e->comms.assign(1, c);
            } catch (...) {
                drop_entry();
                throw;
            }
        }
        comms = e->comms;
    }
    // every rank in this process, one GPU each (ncclCommInitAll; also a
    // one-rank communicator when NCCL is forced on one GPU)
    void acquire_all(const std::vector<int>& devs) {
        std::string key = "all";
        for (int d : devs) key += " " + std::to_string(d);
        bool fresh = false;
        e = find_or_add(key, fresh);
        if (fresh) {
            try {
                std::vector<ncclComm_t> c(devs.size(), nullptr);
                NK(ncclCommInitAll(c.data(), (int)devs.size(), devs.data()));
                e->comms = c;
            } catch (...) {
                drop_entry();
                throw;
            }
        }
        comms = e->comms;
    }
    // called by a failing rank: unblocks the others' collectives
    void abort() {
        if (!e || aborted.exchange(true)) return;
        for (ncclComm_t c : comms)
            if (c) ncclCommAbort(c);
    }
    void release(bool failed) {
        if (!e) return;
        if (failed || aborted) {
            if (!aborted)
                for (ncclComm_t c : comms)
                    if (c) ncclCommAbort(c);
            drop_entry();
            return;
        }
        std::lock_guard<std::mutex> lk(comm_cache().mu);
        e->busy = false;
        e = nullptr;
    }
    ~CommLease() { release(true); }  // only reached with e set if release() was skipped (exception)
};

// ------------------------------------------------------------------ batches
void run_rank(Rank& R, const Problem& p, const omcg_run_config& cfg) {
    CK(cudaSetDevice(R.device));
    const int nb = cfg.n_batches;
    const double dN = (double)R.N;
    double k_norm = 1.0;
    bool have_source = false;
    const int fuel_nuc = (int)p.mat[MAT_FUEL].nuc.size();
    const int tally_smem = 4 * R.n_tally_bins <= SMEM_TALLY_MAX;
    long long launches0 = 0;
    char batch_name[32];
    for (int batch = 1; batch <= nb; ++batch) {
        const bool active = batch > cfg.n_inactive;
        std::snprintf(batch_name, sizeof batch_name, "batch %d%s", batch, active ? "" : " (inactive)");
        Nvtx batch_range(batch_name);
        if (batch == cfg.n_inactive + 1) {
            CK(cudaStreamSynchronize(R.main));
            CK(cudaEventRecord(R.ev_a0, R.main));
            launches0 = launch_counter();
        }
        CK(cudaMemsetAsync(R.acc.k, 0, sizeof(ull) * 3, R.main));
        CK(cudaMemsetAsync(R.acc.counts, 0, sizeof(ull) * 8, R.main));
        CK(cudaMemsetAsync(R.acc.bank_count, 0, sizeof(ull), R.main));
        if (active) CK(cudaMemsetAsync(R.acc.tally, 0, sizeof(ull) * 4 * (size_t)R.n_tally_bins, R.main));
        CK(cudaStreamSynchronize(R.main));

        Ctx base{};
        base.lib = R.gp.lib;
        base.geo = R.gp.geo;
        base.acc = R.acc;
        base.tally_on = active ? 1 : 0;
        base.n_tally_bins = R.n_tally_bins;
        base.tally_smem = tally_smem;
        base.tally_priv = R.tally_priv;
        base.n_priv = R.n_priv;
        base.k_norm = k_norm;
        base.rank_lo = R.rank_lo;
        base.n_batch = R.N;
        base.batch = batch;
        base.master = cfg.seed;
        base.record_n = cfg.record_n;
        base.recording = (R.acc.records && batch == cfg.record_batch) ? 1 : 0;
        base.fused = cfg.event_fusion ? 1 : 0;
        base.move_cap = cfg.event_fusion ? std::max(0, cfg.move_event_cap) : 0;
        const Site* src = have_source ? R.source : nullptr;
        const bool prof = cfg.profile != 0 && active;

        auto drive = [&](SubBank& S) {
            Nvtx r("event loop");
            Ctx c = base;
            c.b = S.b;
            c.qs = S.qs;
            c.ctrl = S.ctrl;
            c.trace_chk = nullptr;
            CK(cudaSetDevice(R.device));
            if (cfg.mode == OMCG_QUEUELESS) run_queueless(R, S, c, src, prof, cfg.tail_threshold);
            else run_queued(R, S, c, src, cfg, prof, fuel_nuc);
            CK(cudaStreamSynchronize(S.stream));
            drain_profile(S);
        };
        if (R.subs.size() == 1) {
            drive(R.subs[0]);
        } else {
            std::vector<std::thread> th;
            std::vector<std::exception_ptr> errs(R.subs.size());
            for (size_t t = 0; t < R.subs.size(); ++t)
                th.emplace_back([&, t] {
                    LaunchCounterScope count_task(R.launches);
                    try { drive(R.subs[t]); } catch (...) { errs[t] = std::current_exception(); }
                });
            for (auto& x : th) x.join();
            for (auto& e : errs)
                if (e) std::rethrow_exception(e);
        }
        for (auto& S : R.subs) {
            CK(cudaMemcpy(S.h_ctrl, S.ctrl, sizeof(ull) * 3, cudaMemcpyDeviceToHost));
            if (S.h_ctrl[2] & 1ULL) throw std::runtime_error("source rejection sampling failed");
            if (S.h_ctrl[2] & 2ULL) throw std::runtime_error("fission bank overflow");
        }

        Nvtx sync_range("batch sync: reduce + fission bank");
        if (active && R.n_priv > 0)
            launch_tally_fold(R.tally_priv, R.n_priv, 4 * (int64_t)R.n_tally_bins, R.acc.tally, R.main);
        // ---- batch reduction (NCCL across ranks: integer sums are exact)
        if (R.bc) {  // NCCL (or the loopback between ranks sharing a GPU)
            R.bc->reduce_batch(R, active);
        } else {
            R.sall.assign(1, 0);
            CK(cudaMemcpyAsync(R.sall.data(), R.acc.bank_count, sizeof(ull), cudaMemcpyDeviceToHost, R.main));
        }
        const std::vector<ull>& sall = R.sall;
        ull hk[3], hc[8];
        CK(cudaMemcpyAsync(hk, R.acc.k, sizeof hk, cudaMemcpyDeviceToHost, R.main));
        CK(cudaMemcpyAsync(hc, R.acc.counts, sizeof hc, cudaMemcpyDeviceToHost, R.main));
        std::vector<ull> tb;
        if (active) {
            tb.resize(4 * (size_t)R.n_tally_bins);
            CK(cudaMemcpyAsync(tb.data(), R.acc.tally, sizeof(ull) * tb.size(), cudaMemcpyDeviceToHost, R.main));
        }
        CK(cudaStreamSynchronize(R.main));
        R.d2h += (int64_t)(sizeof hk + sizeof hc + sizeof(ull) * (R.world + tb.size()));
        for (size_t i = 0; i < tb.size(); ++i) R.tally_total[i] += (int64_t)tb[i];
        for (int i = 0; i < 7; ++i) R.counts[i] += (int64_t)hc[i];
        R.k_coll[batch - 1] = (double)(int64_t)hk[0] / TALLY_SCALE / dN;
        R.k_abs[batch - 1] = (double)(int64_t)hk[1] / TALLY_SCALE / dN;
        R.k_track[batch - 1] = (double)(int64_t)hk[2] / TALLY_SCALE / dN;
        uint64_t S_total = 0, S_before = 0;
        for (int r = 0; r < R.world; ++r) {
            if (r < R.rank) S_before += sall[r];
            S_total += sall[r];
        }
        const uint64_t S_mine = sall[R.rank];
        R.n_sites[batch - 1] = (int64_t)S_total;
        k_norm = R.k_coll[batch - 1];
        R.batches_run = batch;
        if (S_total == 0) throw std::runtime_error("fission bank empty");
        if (batch == nb) break;

        // ---- canonical bank order (history, progeny) without a sort
        launch_scan_i32(R.acc.sites_pp, R.scan_out, R.N_rank, R.scan_tmp, R.main);
        launch_bank_canon(R.acc.bank, (int64_t)S_mine, R.scan_out, R.rank_lo, R.canon, R.main);
        // ---- systematic resampling to N for the next batch
        uint64_t bs = stream_seed(cfg.seed, (uint64_t)batch, STREAM_BANK);
        uint64_t off = (uint64_t)(prn(bs) * (double)S_total);
        if (off >= S_total) off = S_total - 1;
        if (!R.bc) {
            launch_resample(R.canon, 0, S_total, off, R.N, R.rank_lo, R.N_rank, R.source, R.main);
        } else {
            // each rank needs a contiguous slice of the global canonical bank
            std::vector<int64_t> plan(4 * (size_t)R.world + 2);
            bank_exchange_plan(reinterpret_cast<const uint64_t*>(sall.data()), R.world, R.N, off, R.rank, plan.data());
            const uint64_t my_a = (uint64_t)plan[4 * R.world];
            R.bc->exchange(R, plan.data());
            launch_resample(R.recv, (int64_t)my_a, S_total, off, R.N, R.rank_lo, R.N_rank, R.source, R.main);
        }
        CK(cudaGetLastError());
        have_source = true;
    }
    CK(cudaStreamSynchronize(R.main));
    for (auto& S : R.subs) CK(cudaStreamSynchronize(S.stream));
    CK(cudaEventRecord(R.ev_a1, R.main));
    CK(cudaEventSynchronize(R.ev_a1));
    R.launches_active = launch_counter() - launches0;
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, R.ev_a0, R.ev_a1));
    R.t_active = (double)ms * 1e-3;
    if (R.bc) R.t_active = R.bc->max_over_ranks(R, R.t_active);  // max over ranks
}

void validate(const omcg_run_config& cfg) {
    if (cfg.mode != OMCG_QUEUED && cfg.mode != OMCG_QUEUELESS) throw std::invalid_argument("mode (P0) must be 0 or 1");
    if (cfg.particles_in_flight < 1) throw std::invalid_argument("particles in flight (P1) must be >= 1");
    if (cfg.n_bins < 1) throw std::invalid_argument("hash bins (P2) must be >= 1");
    if (cfg.tasks_per_gpu < 1 || cfg.tasks_per_gpu > 8) throw std::invalid_argument("tasks per GPU (P5) must be 1..8");
    if (cfg.n_particles < 1 || cfg.n_particles > ((int64_t)1 << 31) - 1)
        throw std::invalid_argument("particles per batch out of range");
    if (cfg.n_batches < 1 || cfg.n_batches > OMCG_MAX_BATCHES) throw std::invalid_argument("batches out of range");
    if (cfg.n_inactive < 0 || cfg.n_inactive >= cfg.n_batches)
        throw std::invalid_argument("inactive batches must be in [0, batches)");
    if (cfg.world_size > 1 && (cfg.rank < 0 || cfg.rank >= cfg.world_size)) throw std::invalid_argument("bad rank");
    if (cfg.world_size > 1 && cfg.n_gpus > 1) throw std::invalid_argument("multi-process ranks use one GPU each");
    if (cfg.force_nccl < 0 || cfg.force_nccl > 1) throw std::invalid_argument("force_nccl must be 0 or 1");
    if (cfg.n_gpus < 1 || cfg.n_gpus > 8) throw std::invalid_argument("n_gpus must be 1..8");
}

}  // namespace

// Fission-bank redistribution plan. Global canonical order is
// rank 0's sites, then rank 1's, ... (ranks own contiguous history ranges).
// Rank r's next-batch histories [lo_r, hi_r) resample global sites
// [(lo_r*S+off)/N, ((hi_r-1)*S+off)/N], a contiguous range. plan layout
// (4W+2 int64): send_first[W] send_count[W] (offsets into my canonical bank),
// recv_first[W] recv_count[W] (offsets into my receive buffer),
// need_first (global index of recv[0]), need_count.
void bank_exchange_plan(const uint64_t* S_all, int W, int64_t N, uint64_t off, int me, int64_t* plan) {
    if (W < 1 || me < 0 || me >= W || N < 1) throw std::invalid_argument("bad exchange plan arguments");
    std::vector<uint64_t> G(W + 1, 0);
    for (int r = 0; r < W; ++r) G[r + 1] = G[r] + S_all[r];
    const uint64_t S = G[W];
    if (S == 0) throw std::invalid_argument("empty fission bank");
    auto need = [&](int r, uint64_t& a, uint64_t& b) {
        int64_t lo = N * r / W, hi = N * (r + 1) / W;
        if (hi <= lo) { a = b = 0; return; }
        a = ((uint64_t)lo * S + off) / (uint64_t)N;
        b = ((uint64_t)(hi - 1) * S + off) / (uint64_t)N + 1;  // exclusive
    };
    uint64_t my_a, my_b;
    need(me, my_a, my_b);
    for (int r = 0; r < W; ++r) {
        uint64_t a, b;
        need(r, a, b);
        uint64_t s0 = std::max(G[me], a), s1 = std::min(G[me + 1], b);
        uint64_t r0 = std::max(G[r], my_a), r1 = std::min(G[r + 1], my_b);
        plan[r] = s1 > s0 ? (int64_t)(s0 - G[me]) : 0;
        plan[W + r] = s1 > s0 ? (int64_t)(s1 - s0) : 0;
        plan[2 * W + r] = r1 > r0 ? (int64_t)(r0 - my_a) : 0;
        plan[3 * W + r] = r1 > r0 ? (int64_t)(r1 - r0) : 0;
    }
    plan[4 * W] = (int64_t)my_a;
    plan[4 * W + 1] = (int64_t)(my_b - my_a);
}

std::vector<int64_t>& last_queue_trace() { return t_trace; }

void nccl_unique_id(unsigned char out[128]) {
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    static_assert(sizeof(id.internal) == 128, "nccl id size");
    std::memcpy(out, id.internal, 128);
}

int device_count() {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    return n;
}

// ------------------------------------------------------------------ NVML (dlopen)
namespace {
typedef int (*nvml_init_t)(void);
typedef int (*nvml_by_pci_t)(const char*, void**);
typedef int (*nvml_energy_t)(void*, unsigned long long*);
typedef int (*nvml_power_t)(void*, unsigned int*);
typedef int (*nvml_count_t)(unsigned int*);
typedef int (*nvml_by_index_t)(unsigned int, void**);
struct Nvml {
    void* lib = nullptr;
    nvml_init_t init = nullptr;
    nvml_by_pci_t by_pci = nullptr;
    nvml_energy_t energy = nullptr;
    nvml_power_t power = nullptr;  // optional: mW, for runs shorter than the energy counter's update period
    nvml_count_t count = nullptr;
    nvml_by_index_t by_index = nullptr;
    bool ok = false;
    Nvml() {
        lib = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_LOCAL);
        if (!lib) return;
        init = (nvml_init_t)dlsym(lib, "nvmlInit_v2");
        by_pci = (nvml_by_pci_t)dlsym(lib, "nvmlDeviceGetHandleByPciBusId_v2");
        energy = (nvml_energy_t)dlsym(lib, "nvmlDeviceGetTotalEnergyConsumption");
        power = (nvml_power_t)dlsym(lib, "nvmlDeviceGetPowerUsage");
        count = (nvml_count_t)dlsym(lib, "nvmlDeviceGetCount_v2");
        by_index = (nvml_by_index_t)dlsym(lib, "nvmlDeviceGetHandleByIndex_v2");
        ok = init && by_pci && energy && init() == 0;
    }
};
Nvml& nvml() {
    static Nvml n;
    return n;
}
}  // namespace

bool energy_counter_mj(int cuda_device, unsigned long long* mj) {
    Nvml& N = nvml();
    if (!N.ok) return false;
    char bus[64];
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, cuda_device) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    void* h = nullptr;
    return N.by_pci(bus, &h) == 0 && N.energy(h, mj) == 0;
}

// Process-start energy marks: every NVML device's counter, read through NVML
// alone (no CUDA initialisation), matched to CUDA devices later by handle
// (NVML returns one handle per physical device, by index or by PCI bus id).
namespace {
std::mutex g_mark_mu;
std::vector<std::pair<void*, unsigned long long>> g_marks;
}  // namespace

// End of a process's GPU work (bin/openmc, before its last energy reading):
// return the pooled device memory and the pinned words, and destroy the
// device contexts, so that this teardown -- seconds' worth of unmapping at
// P1 = 8e6 -- happens inside the metered span instead of in the process
// exit after it. No omcg call may be in flight; later calls start afresh.
void release_devices() {
    {   // cached communicators live in the contexts about to be destroyed
        CommCache& cc = comm_cache();
        std::lock_guard<std::mutex> lk(cc.mu);
        for (auto& e : cc.entries)
            for (ncclComm_t cm : e->comms)
                if (cm) ncclCommDestroy(cm);
        cc.entries.clear();
    }
    pinned().release();
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (int d = 0; d < 64; ++d) {
        if (!g_pool_done[d]) continue;
        if (cudaSetDevice(d) == cudaSuccess) {
            cudaDeviceSynchronize();
            cudaDeviceReset();
        }
        g_pool_done[d] = false;
    }
    cudaGetLastError();
}

bool energy_mark() {
    Nvml& N = nvml();
    if (!N.ok || !N.count || !N.by_index) return false;
    unsigned int n = 0;
    if (N.count(&n) != 0) return false;
    std::vector<std::pair<void*, unsigned long long>> marks;
    for (unsigned int i = 0; i < n; ++i) {
        void* h = nullptr;
        unsigned long long mj = 0;
        if (N.by_index(i, &h) == 0 && N.energy(h, &mj) == 0) marks.emplace_back(h, mj);
    }
    std::lock_guard<std::mutex> lk(g_mark_mu);
    g_marks = std::move(marks);
    return !g_marks.empty();
}

bool energy_since_mark_j(int cuda_device, double* joules) {
    Nvml& N = nvml();
    if (!N.ok) return false;
    char bus[64];
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, cuda_device) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    void* h = nullptr;
    unsigned long long mj = 0;
    if (N.by_pci(bus, &h) != 0 || N.energy(h, &mj) != 0) return false;
    std::lock_guard<std::mutex> lk(g_mark_mu);
    for (const auto& m : g_marks)
        if (m.first == h) {
            *joules = (double)(mj - m.second) * 1e-3;
            return true;
        }
    return false;
}

bool EnergyMeter::start(const std::vector<int>& cuda_devices) {
    ok = false;
    handles.clear();
    start_mj.clear();
    Nvml& N = nvml();
    if (!N.ok) return false;
    for (int d : cuda_devices) {
        char bus[64];
        if (cudaDeviceGetPCIBusId(bus, sizeof bus, d) != cudaSuccess) return false;
        void* h = nullptr;
        if (N.by_pci(bus, &h) != 0) return false;
        unsigned long long mj = 0;
        if (N.energy(h, &mj) != 0) return false;
        handles.push_back(h);
        start_mj.push_back(mj);
    }
    t0 = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    ok = true;
    return true;
}
// The total-energy counter advances in steps (tens of ms on B200): a run
// shorter than one step can read 0 J, which would make its EDP 0 -- the best
// possible objective. Such a device is charged its current power draw over
// the run's wall time instead.
double EnergyMeter::stop_joules() {
    if (!ok) return 0.0;
    const double dt =
        std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count() - t0;
    Nvml& N = nvml();
    double j = 0.0;
    for (size_t i = 0; i < handles.size(); ++i) {
        unsigned long long mj = 0;
        if (N.energy(handles[i], &mj) != 0) continue;
        double dj = (double)(mj - start_mj[i]) * 1e-3;
        unsigned int mw = 0;
        if (dj <= 0.0 && N.power && N.power(handles[i], &mw) == 0) dj = 1e-3 * (double)mw * dt;
        j += dj;
    }
    return j;
}

// ------------------------------------------------------------------ entry
void run_transport(const Problem& p, const omcg_run_config& cfg_in, omcg_run_result* res, int64_t* tally_out,
                   omcg_record* records) {
    omcg_run_config cfg = cfg_in;
    if (cfg.world_size < 1) cfg.world_size = 1;
    validate(cfg);
    std::memset(res, 0, sizeof *res);
    auto t_call0 = std::chrono::steady_clock::now();
    const bool multiproc = cfg.world_size > 1;
    const int local_ranks = multiproc ? 1 : cfg.n_gpus;
    int ndev = device_count();
    std::vector<int> devs(local_ranks);
    bool shared_gpu = false;  // local ranks on one GPU: in-process loopback instead of NCCL
    for (int i = 0; i < local_ranks; ++i) {
        devs[i] = cfg.devices[i];
        if (devs[i] < 0 || devs[i] >= ndev) throw CudaError("CUDA device " + std::to_string(devs[i]) + " not available");
        for (int j = 0; j < i; ++j)
            if (devs[j] == devs[i]) shared_gpu = true;
    }
    std::vector<int> meter_devs = devs;
    std::sort(meter_devs.begin(), meter_devs.end());
    meter_devs.erase(std::unique(meter_devs.begin(), meter_devs.end()), meter_devs.end());
    static const bool trace_init = std::getenv("OMCG_TRACE_INIT") != nullptr;
    auto mark = [&](const char* what) {
        if (trace_init)
            std::fprintf(stderr, "[omcg run] %-28s %8.3f s\n", what,
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t_call0).count());
    };
    EnergyMeter meter;
    meter.start(meter_devs);
    mark("energy meter started");
    std::atomic<long long> launches{0};  // this call's kernel launches (all of its host threads)
    LaunchCounterScope count_here(&launches);
    std::vector<Rank> ranks(local_ranks);
    std::unique_ptr<LoopbackShared> loop_shared;
    std::vector<std::unique_ptr<BatchComm>> bcs(local_ranks);
    CommLease lease;  // NCCL communicators: created once per placement, reused by later calls
    if (multiproc) {
        lease.acquire_rank(cfg.nccl_id, cfg.world_size, cfg.rank, devs[0]);
        bcs[0].reset(new NcclBatchComm());
    } else if (local_ranks > 1 && shared_gpu) {
        loop_shared.reset(new LoopbackShared(local_ranks));
        for (int i = 0; i < local_ranks; ++i) bcs[i].reset(new LoopbackBatchComm(loop_shared.get()));
    } else if (local_ranks > 1 || cfg.force_nccl) {
        lease.acquire_all(devs);
        for (int i = 0; i < local_ranks; ++i) bcs[i].reset(new NcclBatchComm(local_ranks == 1));
    }
    mark("communicators");
    for (int i = 0; i < local_ranks; ++i) {
        ranks[i].device = devs[i];
        ranks[i].comm = lease.comms.empty() ? nullptr : lease.comms[i];
        ranks[i].bc = bcs[i].get();
        ranks[i].world = multiproc ? cfg.world_size : local_ranks;
        ranks[i].rank = multiproc ? cfg.rank : i;
        ranks[i].launches = &launches;
    }
    std::vector<std::exception_ptr> errs(local_ranks);
    auto body = [&](int i) {
        LaunchCounterScope count_rank(&launches);
        try {
            setup_rank(ranks[i], p, cfg);
            run_rank(ranks[i], p, cfg);
        } catch (...) {
            errs[i] = std::current_exception();
            // the other ranks of this call must not wait for this one forever:
            // loopback barriers throw, NCCL collectives are aborted
            if (loop_shared) loop_shared->abort();
            if (local_ranks > 1) lease.abort();
        }
    };
    if (local_ranks == 1) body(0);
    else {
        std::vector<std::thread> th;
        for (int i = 0; i < local_ranks; ++i) th.emplace_back(body, i);
        for (auto& t : th) t.join();
    }
    mark("ranks done");
    if (std::getenv("OMCG_MOVE_CYCLES")) dump_move_cycles();
    if (std::getenv("OMCG_COOP_STATS")) dump_coop_stats();
    if (std::getenv("OMCG_TAIL_CYCLES")) dump_tail_cycles();
    std::exception_ptr first;
    for (auto& e : errs)
        if (e && !first) first = e;
    if (!first) {
        Rank& R0 = ranks[0];
        res->n_batches_run = R0.batches_run;
        std::memcpy(res->k_coll, R0.k_coll, sizeof res->k_coll);
        std::memcpy(res->k_abs, R0.k_abs, sizeof res->k_abs);
        std::memcpy(res->k_track, R0.k_track, sizeof res->k_track);
        std::memcpy(res->n_sites, R0.n_sites, sizeof res->n_sites);
        for (int i = 0; i < 4; ++i) res->n_events[i] = R0.counts[i];
        res->n_absorbed = R0.counts[4 + TERM_ABSORBED];
        res->n_leaked = R0.counts[4 + TERM_LEAKED];
        res->n_lost = R0.counts[6];
        int n_active = 0;
        double ks = 0.0, kq = 0.0;
        for (int b = cfg.n_inactive; b < R0.batches_run; ++b) {
            ks += R0.k_coll[b];
            kq += R0.k_coll[b] * R0.k_coll[b];
            n_active++;
        }
        if (n_active > 0) {
            res->k_mean = ks / (double)n_active;
            double var = n_active > 1 ? (kq / (double)n_active - res->k_mean * res->k_mean) / (double)(n_active - 1) : 0.0;
            res->k_std = var > 0.0 ? std::sqrt(var) : 0.0;
        }
        double ta = 0.0, ti = 0.0;
        for (auto& R : ranks) {
            ta = std::max(ta, R.t_active);
            ti = std::max(ti, R.t_init);
            res->h2d_bytes += R.h2d;
            res->d2h_bytes += R.d2h;
            for (auto& S : R.subs) {
                for (int k = 0; k < 8; ++k) {
                    res->prof_ms[k] += S.prof_ms[k];
                    res->prof_launches[k] += S.prof_launches[k];
                    res->prof_items[k] += S.prof_items[k];
                }
                res->xs_fuel_bytes += S.xs_fuel_bytes;
                res->queue_iterations += S.iterations;
                res->sorts += S.sorts;
                res->tail_launches += S.tail_launches;
            }
        }
        res->t_active = ta;
        res->t_init = ti;
        res->fom = ta > 0.0 ? (double)cfg.n_particles * (double)n_active / ta : 0.0;
        res->kernel_launches = R0.launches_active;
        res->kernel_launches_total = launches.load();
        if (tally_out) {
            std::memcpy(tally_out, R0.tally_total.data(), sizeof(int64_t) * R0.tally_total.size());
            res->d2h_bytes += 0;
        }
        if (records && R0.acc.records && cfg.record_n > 0) {
            // records are indexed by batch-global history; each rank holds its own slice
            for (auto& R : ranks) {
                CK(cudaSetDevice(R.device));
                int64_t lo = std::max<int64_t>(R.rank_lo, 0), hi = std::min<int64_t>(R.rank_lo + R.N_rank, cfg.record_n);
                if (hi > lo)
                    CK(cudaMemcpy(records + lo, R.acc.records + lo, sizeof(omcg_record) * (size_t)(hi - lo),
                                  cudaMemcpyDeviceToHost));
            }
        }
        t_trace.clear();
        for (auto& S : R0.subs) t_trace.insert(t_trace.end(), S.trace.begin(), S.trace.end());
    }
    mark("results gathered");
    for (auto& R : ranks) teardown_rank(R);
    mark("streams/events destroyed");
    lease.release(first != nullptr);
    ranks.clear();  // device memory back before the call returns
    mark("teardown");
    res->energy_j = meter.stop_joules();
    mark("energy meter stopped");
    res->t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_call0).count();
    if (first) std::rethrow_exception(first);
}

// ------------------------------------------------------------------ parity hooks
uint64_t device_hash_build(const Problem& p, int n_bins, int device, int32_t* hash_out) {
    CK(cudaSetDevice(device));
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    uint64_t h;
    {
        GpuProblem gp;
        gp.upload(p, n_bins, device, s);
        size_t n = (size_t)(n_bins + 1) * (size_t)p.n_nuc;
        std::vector<int32_t> hh(n);
        CK(cudaMemcpyAsync(hh.data(), gp.lib.hash, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        h = fnv1a(1469598103934665603ULL, hh.data(), sizeof(int32_t) * n);
        if (hash_out) std::memcpy(hash_out, hh.data(), sizeof(int32_t) * n);
    }
    cudaStreamDestroy(s);
    return h;
}

void device_div_check(int device, int64_t n, const double* a, const double* b, double* q_fast, uint8_t* ok,
                      double* q_frac, double* q_ieee) {
    CK(cudaSetDevice(device));
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    {
        DevArena ar;
        ar.device = device;
        double* da = ar.alloc<double>(n);
        double* db = ar.alloc<double>(n);
        double* dq = ar.alloc<double>(5 * n);  // fast (div, sqrt), frac, ieee (div, sqrt)
        uint8_t* dok = ar.alloc<uint8_t>(2 * n);
        CK(cudaMemcpyAsync(da, a, sizeof(double) * n, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(db, b, sizeof(double) * n, cudaMemcpyHostToDevice, s));
        launch_div_check(n, da, db, dq, dok, dq + 2 * n, dq + 3 * n, s);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(q_fast, dq, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(q_frac, dq + 2 * n, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(q_ieee, dq + 3 * n, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(ok, dok, 2 * n, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    cudaStreamDestroy(s);
}

void device_xs_lookup(const Problem& p, int n_bins, int device, int64_t n, const int32_t* mat, const double* E,
                      double* out) {
    CK(cudaSetDevice(device));
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    {
        GpuProblem gp;
        gp.upload(p, n_bins, device, s);
        DevArena a;
        a.device = device;
        int32_t* dm = a.alloc<int32_t>(n);
        double* dE = a.alloc<double>(n);
        double* dout = a.alloc<double>(4 * n);
        for (int64_t i = 0; i < n; ++i)
            if (mat[i] < 0 || mat[i] >= (int)p.mat.size()) throw std::invalid_argument("material out of range");
        CK(cudaMemcpyAsync(dm, mat, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dE, E, sizeof(double) * n, cudaMemcpyHostToDevice, s));
        launch_xs_pairs(gp.lib, n, dm, dE, dout, s);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, dout, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    cudaStreamDestroy(s);
}

// The production fuel lookup on a queue: n histories waiting for
// calculate_xs at (mat[i], E[i]) in the fuel XS queue (entry i = slot i),
// sorted by (material, energy) when n >= sort_threshold >= 0 exactly as the
// queued loop sorts it, then one k_xs_fuel_fused launch. out: the four
// macroscopic XS per entry as stored in the record; ckpt_out (optional, n x 16):
// the segment checkpoints (entries past the material's count untouched, NaN).
// The launch must hand every entry on to the move queue: checked here.
void device_xs_lookup_queue(const Problem& p, int n_bins, int device, int64_t n, const int32_t* mat, const double* E,
                            int64_t sort_threshold, double* out, double* ckpt_out) {
    if (n > (int64_t)1 << 30) throw std::invalid_argument("n too large");
    for (int64_t i = 0; i < n; ++i)
        if (mat[i] < 0 || mat[i] >= (int)p.mat.size()) throw std::invalid_argument("material out of range");
    CK(cudaSetDevice(device));
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    try {
        GpuProblem gp;
        gp.upload(p, n_bins, device, s);
        int nseg = 1, n_sort_mats = 1;
        for (const auto& m : p.mat) {
            nseg = std::max(nseg, (int)((m.nuc.size() + CKPT_STRIDE - 1) / CKPT_STRIDE));
            n_sort_mats += m.fissionable ? 1 : 0;
        }
        DevArena a;
        a.device = device;
        Ctx c{};
        c.lib = gp.lib;
        c.geo = gp.geo;
        c.b.cap = n;
        c.b.p = a.alloc<PState>(n);
        c.b.xc = a.alloc<XsCache>(n);
        c.b.cnt = a.alloc<int4>(n);
        c.b.event = a.alloc<int8_t>(n);
        c.b.ckpt = a.alloc<double>(NCKPT * n);
        c.qs.cap = n;
        c.qs.qbase = a.alloc<int32_t>((int64_t)(N_QUEUES + 1) * n);
        c.qs.count = a.alloc<unsigned>(8);
        c.qs.dead_tail = reinterpret_cast<ull*>(c.qs.count + 6);
        c.qs.adv_q = EV_ADV;
        c.ctrl = a.alloc<ull>(8);
        int32_t* sorted = a.alloc<int32_t>(n);
        uint32_t* keys = a.alloc<uint32_t>(n);
        unsigned* hist = a.alloc<unsigned>((int64_t)n_sort_mats * 65536);
        unsigned* cursor = a.alloc<unsigned>((int64_t)n_sort_mats * 65536);
        unsigned* bsum = a.alloc<unsigned>((int64_t)n_sort_mats * 64);
        int32_t* dm = a.alloc<int32_t>(n);
        double* dE = a.alloc<double>(n);
        CK(cudaMemsetAsync(c.qs.count, 0, sizeof(unsigned) * 8, s));
        CK(cudaMemsetAsync(c.ctrl, 0, sizeof(ull) * 8, s));
        CK(cudaMemsetAsync(hist, 0, sizeof(unsigned) * (size_t)n_sort_mats * 65536, s));
        CK(cudaMemsetAsync(c.b.ckpt, 0xff, sizeof(double) * NCKPT * (size_t)n, s));
        CK(cudaMemcpyAsync(dm, mat, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dE, E, sizeof(double) * n, cudaMemcpyHostToDevice, s));
        int32_t* q = c.qs.qbase + (int64_t)EV_XS_FUEL * n;
        launch_lookup_setup(c, (int)n, dm, dE, q, s);
        const int32_t* qptr = q;
        if (sort_threshold >= 0 && n >= sort_threshold) {
            launch_sort(c, q, sorted, (int)n, n_sort_mats, hist, cursor, keys, bsum, s);
            qptr = sorted;
        }
        launch_xs_fuel_fused(c, qptr, (int)n, nseg, s);
        CK(cudaGetLastError());
        std::vector<PState> rec((size_t)n);
        std::vector<int32_t> moved((size_t)n);
        unsigned cnt[8];
        CK(cudaMemcpyAsync(rec.data(), c.b.p, sizeof(PState) * (size_t)n, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(moved.data(), c.qs.qbase + (int64_t)EV_ADV * n, sizeof(int32_t) * (size_t)n,
                           cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(cnt, c.qs.count, sizeof cnt, cudaMemcpyDeviceToHost, s));
        if (ckpt_out)
            CK(cudaMemcpyAsync(ckpt_out, c.b.ckpt, sizeof(double) * NCKPT * (size_t)n, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        // the launch appends every entry to the move queue once and empties its own queue
        if (cnt[EV_XS_FUEL] != 0u || cnt[EV_ADV] != (unsigned)n)
            throw std::logic_error("fuel lookup: queue lengths after the launch are wrong");
        std::vector<uint8_t> seen((size_t)n, 0);
        for (int64_t i = 0; i < n; ++i) {
            const int32_t sl = moved[(size_t)i];
            if (sl < 0 || sl >= n || seen[(size_t)sl]++) throw std::logic_error("fuel lookup: move queue is not a permutation");
        }
        for (int64_t i = 0; i < n; ++i) {
            out[4 * i] = rec[(size_t)i].st;
            out[4 * i + 1] = rec[(size_t)i].sa;
            out[4 * i + 2] = rec[(size_t)i].sf;
            out[4 * i + 3] = rec[(size_t)i].snf;
        }
    } catch (...) {
        cudaStreamDestroy(s);
        throw;
    }
    cudaStreamDestroy(s);
}

}  // namespace omcg
