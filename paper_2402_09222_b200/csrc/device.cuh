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
    int32_t pad1[2];
};
static_assert(sizeof(PState) == 128, "PState must be one 128-byte line");

// Last fuel macroscopic cross sections of a history. A history that leaves a
// fuel pin and enters another without colliding has the same energy, so its
// fuel calculate_xs is this cache (OpenMC skips the lookup on unchanged
// material and energy too); the result is the same bits, the lookup is skipped.
struct alignas(16) FuelCache {
    double E, t, a, f, nf;
    int32_t mat, pad;
};
static_assert(sizeof(FuelCache) == 48, "FuelCache layout");

struct Bank {
    int64_t cap;
    PState* p;         // cap records
    FuelCache* fc;     // cap fuel caches
    int4* cnt;         // per-slot event counters: n_xs, n_adv, n_cross, n_coll
    int8_t* event;     // dense next-event array (queueless sweeps, tail, refill)
    // running macroscopic total after every CKPT_STRIDE nuclides of a large
    // material (written by calculate_xs, read by collision to jump straight
    // to the segment holding the sampled nuclide): NCKPT x cap
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
