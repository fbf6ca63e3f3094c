// problem.hpp — host-side synthetic problem: nuclide library (energy grids +
// 4-channel point cross sections), materials and lattice geometry.
//
// This plays the role of OpenMC's HDF5 library + geometry input that the
// reference's campaign never ships (HM-Large, 272 nuclides;
// library loading is initialisation, excluded from FoM but
// included in EDP via process wall time, proj/src/harness.cpp:320).
// Buffers live in host memory; omcg_run uploads them (the e2e path).
#pragma once
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "omcg_physics.cuh"

namespace omcg {

enum ProblemKind { PINCELL = 0, ASSEMBLY = 1, CORE = 2, INFINITE = 3 };
// the analytic infinite-medium problem (one energy-independent nuclide, density 1 atom/(b cm))
constexpr int INF_GRID = 1001;
constexpr double INF_AWR = 12.0;
constexpr double INF_SIGMA_T = 1.0, INF_SIGMA_A = 0.4, INF_SIGMA_F = 0.25, INF_NU = 2.5;
enum MaterialId { MAT_WATER = 0, MAT_CLAD = 1, MAT_FUEL = 2 };

struct alignas(32) XS4 {
    double t, a, f, nf;  // total, absorption, fission, nu-fission (barns)
};

struct Material {
    std::vector<int> nuc;      // local nuclide ids
    std::vector<double> dens;  // atoms / (barn cm)
    bool fissionable = false;
};

struct Problem {
    int kind = ASSEMBLY;
    uint64_t xs_seed = 1234;
    int n_nuc = 0;
    std::vector<int> global_id;     // local -> global nuclide id
    std::vector<double> awr;        // per local nuclide
    std::vector<int64_t> goff;      // n_nuc+1 offsets into E / xs
    std::vector<double> E;          // all grids, concatenated
    std::vector<XS4> xs;            // all rows, concatenated
    std::vector<Material> mat;
    Geometry geo{};                 // pin_map points into pin_map_host
    std::vector<uint8_t> pin_map_host;
    double gen_seconds = 0.0;       // library generation wall time
    // E / xs page-locked on first upload (cudaHostRegister), released with the
    // problem (or when it is reassigned): later uploads copy at full rate
    struct Pins {
        std::mutex mu;
        std::shared_ptr<void> E, xs;
        Pins() = default;
        Pins(const Pins&) {}
        Pins& operator=(const Pins&) {
            std::lock_guard<std::mutex> lk(mu);
            E.reset();
            xs.reset();
            return *this;
        }
    };
    mutable Pins pins;

    int64_t grid_points() const { return goff.empty() ? 0 : goff.back(); }
    int64_t library_bytes() const { return grid_points() * (int64_t)(sizeof(double) + sizeof(XS4)); }
};

// Build the synthetic problem; generation is threaded over nuclides with
// n_threads host threads (the launcher's -c P4), bit-identical for any count.
void build_problem(Problem& p, int kind, uint64_t xs_seed, int n_threads);

uint64_t fnv1a(uint64_t h, const void* data, size_t n);
uint64_t library_checksum(const Problem& p);  // same definition as the oracle's

}  // namespace omcg
