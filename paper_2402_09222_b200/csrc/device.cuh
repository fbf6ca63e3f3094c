// device.cuh — device-side data layout of the transport hot path.
//
// HBM layout (per GPU):
//   library  : E[]  f64, all nuclide grids concatenated (goff[] offsets)
//              xs[] XS4 (32 B rows: total, absorption, fission, nu-fission)
//   hash     : int32 [n_nuc][n_bins+1], nuclide-major (P2 bins)
//   bank     : structure-of-arrays over P1 in-flight slots
//   queues   : int32 slot lists, one per event type, rebuilt in slot order
//   fission  : unordered append buffer of 40 B sites + per-history counts,
//              canonicalised to (history, progeny) order at batch end.
#pragma once
#include <cstdint>

#include "../../include/omcg.h"
#include "omcg_physics.cuh"
#include "problem.hpp"

namespace omcg {

struct DevLib {
    int n_nuc, n_bins, n_mat;
    double inv_spacing, log_emin;
    const int32_t* goff;     // n_nuc+1
    const double* E;
    const XS4* xs;
    const int32_t* hash;     // n_nuc*(n_bins+1)
    const double* awr;       // n_nuc
    const int32_t* mat_off;  // n_mat+1
    const int32_t* mat_nuc;
    const int4* mat_desc;    // per material entry: {E offset, grid size, hash-row offset, nuclide}
    const double* mat_dens;
    const uint8_t* mat_fissionable;
    const uint8_t* mat_fuel;  // material uses the fuel XS queue
    const uint8_t* mat_sort_rank;  // fuel material rank for the sort key
    const double* host_dens;       // host copy of mat_dens (launch parameters), nullptr if too large
    int n_dens;                    // entries in host_dens
};

struct Site {
    double x, y, z, E;
    uint64_t key;  // (batch-global history index << 24) | progeny
};

// Hot per-history state: one 128-byte record per in-flight slot. The event
// kernels reach a history through a queue entry (a gather), so what costs is
// the number of distinct 32 B sectors touched per event: a record keeps every
// field an event needs in one 128 B line (4 sectors, 16 B vector loads)
// instead of ~16 scattered SoA sectors.
struct alignas(128) PState {
    double x, y, z;         // position (cm)
    double u, v, w;         // direction
    double E, wgt;          // energy (eV), weight
    double st, sa, sf, snf; // macroscopic total / absorption / fission / nu-fission (1/cm)
    uint64_t seed;          // RNG state
    int32_t cell;           // global pin index gy*nx + gx
    int32_t gidx;           // batch-global history index
    int8_t ring, mat, surf, pad0;
    int32_t n_sites;        // fission sites banked so far
    int32_t bin;            // log hash-grid bin of E (set whenever E changes: one det_log per energy)
    int32_t pad1;
};
static_assert(sizeof(PState) == 128, "PState must be one 128-byte line");

// Last macroscopic cross sections of a history per material (materials
// 0..XS_CACHE_MATS-1). A history that crosses into a material it already
// looked up at an unchanged energy (no collision since) takes the cached
// values: same bits, lookup skipped (OpenMC skips unchanged lookups too).
// ck_mat: the material whose segment checkpoints are in Bank::ckpt, so a
// cached many-nuclide material is only reused when its checkpoints are current.
constexpr int XS_CACHE_MATS = 3;
struct alignas(128) XsCache {
    double E[XS_CACHE_MATS];
    int32_t ck_mat, pad;
    double m[XS_CACHE_MATS][4];  // total, absorption, fission, nu-fission
};
static_assert(sizeof(XsCache) == 128, "XsCache layout");

struct Bank {
    int64_t cap;
    PState* p;         // cap records
    XsCache* xc;       // cap cross-section caches
    int4* cnt;         // per-slot event counters: n_xs, n_adv, n_cross, n_coll
    int8_t* event;     // dense next-event array (queueless sweeps, tail, refill)
    // running macroscopic total after every CKPT_STRIDE nuclides of a large
    // material (written by calculate_xs, read by collision to jump straight
    // to the segment holding the sampled nuclide): cap x NCKPT, one 128-byte
    // line per slot (queue order is random in slots, so a slot-major layout
    // touches one line per lookup instead of NCKPT scattered sectors)
    double* ckpt;
};
constexpr int CKPT_STRIDE = 16;
constexpr int NCKPT = 16;

// Per-rank accumulators shared by the rank's sub-banks (tasks).
struct Acc {
    unsigned long long* tally;   // n_tally_bins * 4 (fixed point)
    unsigned long long* k;       // [0] collision, [1] absorption, [2] track length
    unsigned long long* counts;  // [0..3] events xs/adv/cross/coll, [4+term] absorbed/leaked/lost
    Site* bank;                  // unordered fission sites
    unsigned long long* bank_count;
    int64_t bank_cap;
    int32_t* sites_pp;           // per rank-local history: sites banked
    omcg_record* records;        // nullptr unless recording
};

}  // namespace omcg
