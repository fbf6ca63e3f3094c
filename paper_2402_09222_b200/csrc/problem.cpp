// problem.cpp — synthetic library / materials / geometry (host, threaded).
// Specification: DESIGN.md §2 (library) — restated independently by the CPU
// oracle (oracle/omc_oracle.c gen_nuclide); parity is checked by checksum.
#include "problem.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <thread>

namespace omcg {

namespace {

enum { CLS_LIGHT = 0, CLS_STRUCT = 1, CLS_ACTINIDE = 2, CLS_FP = 3 };

struct NucDef {
    int cls;
    double awr, s0, c0, f0, f_fast, ft, nu0, nu1;
    int nres;
    double res_lo, res_hi;
    int res_fis, h_rolloff;
};

constexpr int N_NAMED = 23;
constexpr int N_FP = 249;
constexpr int N_GLOBAL = N_NAMED + N_FP;  // 272

// H1 O16 B10 B11 Zr90 Zr91 Zr92 Zr94 Zr96 Fe56 Cr52 Sn118 U234 U235 U236 U238
// Np237 Pu238 Pu239 Pu240 Pu241 Pu242 Am241, then 249 fission products.
const NucDef NAMED[N_NAMED] = {
    {CLS_LIGHT, 0.99917, 20.0, 0.332, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1},
    {CLS_STRUCT, 15.858, 3.9, 1.9e-4, 0, 0, 0, 0, 0, 3, 4.0e5, 4.0e6, 0, 0},
    {CLS_LIGHT, 9.9269, 2.2, 3840.0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},
    {CLS_LIGHT, 10.9147, 5.0, 5.5e-3, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},
    {CLS_STRUCT, 89.132, 6.5, 0.011, 0, 0, 0, 0, 0, 6, 2.0e3, 1.0e5, 0, 0},
    {CLS_STRUCT, 90.122, 9.7, 1.2, 0, 0, 0, 0, 0, 8, 2.0e2, 5.0e4, 0, 0},
    {CLS_STRUCT, 91.112, 7.3, 0.22, 0, 0, 0, 0, 0, 6, 5.0e2, 5.0e4, 0, 0},
    {CLS_STRUCT, 93.096, 6.2, 0.05, 0, 0, 0, 0, 0, 5, 2.0e3, 5.0e4, 0, 0},
    {CLS_STRUCT, 95.081, 6.2, 0.023, 0, 0, 0, 0, 0, 4, 3.0e2, 5.0e4, 0, 0},
    {CLS_STRUCT, 55.454, 11.6, 2.6, 0, 0, 0, 0, 0, 6, 1.0e3, 5.0e5, 0, 0},
    {CLS_STRUCT, 51.549, 3.0, 0.86, 0, 0, 0, 0, 0, 5, 1.0e3, 5.0e5, 0, 0},
    {CLS_STRUCT, 116.92, 4.9, 0.22, 0, 0, 0, 0, 0, 6, 40.0, 1.0e4, 0, 0},
    {CLS_ACTINIDE, 232.03, 10.0, 100.0, 0, 0, 1.2, 2.4, 0.13, 15, 5.0, 2.0e3, 0, 0},
    {CLS_ACTINIDE, 233.02, 12.0, 99.0, 585.0, 1.3, 0, 2.43, 0.12, 40, 0.3, 2.0e3, 1, 0},
    {CLS_ACTINIDE, 234.02, 8.5, 5.1, 0, 0, 0.6, 2.35, 0.13, 15, 5.0, 2.0e3, 0, 0},
    {CLS_ACTINIDE, 236.01, 9.3, 2.68, 0, 0, 0.55, 2.6, 0.15, 40, 6.0, 1.0e4, 0, 0},
    {CLS_ACTINIDE, 235.01, 10.0, 175.0, 0, 0, 1.5, 2.7, 0.14, 20, 0.4, 2.0e3, 0, 0},
    {CLS_ACTINIDE, 236.0, 20.0, 540.0, 17.0, 2.0, 0, 2.9, 0.14, 12, 2.0, 2.0e3, 1, 0},
    {CLS_ACTINIDE, 236.99, 8.0, 270.0, 750.0, 1.7, 0, 2.87, 0.14, 35, 0.29, 2.0e3, 1, 0},
    {CLS_ACTINIDE, 237.99, 8.0, 290.0, 0, 0, 1.3, 2.8, 0.14, 20, 1.0, 2.0e3, 0, 0},
    {CLS_ACTINIDE, 238.98, 11.0, 360.0, 1010.0, 1.6, 0, 2.93, 0.14, 30, 0.26, 2.0e3, 1, 0},
    {CLS_ACTINIDE, 239.98, 8.0, 19.0, 0, 0, 1.2, 2.8, 0.14, 15, 2.6, 2.0e3, 0, 0},
    {CLS_ACTINIDE, 238.99, 11.0, 600.0, 3.1, 0, 1.0, 2.9, 0.14, 20, 0.57, 2.0e3, 0, 0},
};
enum {
    G_H1 = 0, G_O16, G_B10, G_B11, G_ZR90, G_ZR91, G_ZR92, G_ZR94, G_ZR96, G_FE56, G_CR52,
    G_SN118, G_U234, G_U235, G_U236, G_U238, G_NP237, G_PU238, G_PU239, G_PU240, G_PU241,
    G_PU242, G_AM241, G_FP0
};

constexpr int MAX_RES = 64;
struct Params {
    double awr = 0, s0 = 0, c0 = 0, f0 = 0, f_fast = 0, ft = 0, nu0 = 0, nu1 = 0;
    int h_rolloff = 0, nres = 0;
    double rE[MAX_RES], rH[MAX_RES], pe[MAX_RES], pc[MAX_RES], pf[MAX_RES];
};

XS4 point_xs(const Params& P, double E) {
    double inv_v = sqrt(0.0253 / E);
    double el = P.s0;
    if (P.h_rolloff) el = P.s0 / sqrt(1.0 + E / 1.0e5);
    double cap = P.c0 * inv_v;
    double fis = 0.0;
    if (P.f0 > 0.0) fis = P.f0 * inv_v + P.f_fast * E / (E + 1.0e3);
    if (P.ft > 0.0) fis = fis + P.ft / (1.0 + det_exp((1.0e6 - E) / 1.5e5));
    for (int r = 0; r < P.nres; ++r) {
        double dE = E - P.rE[r];
        double psi = P.rH[r] / (dE * dE + P.rH[r]);
        el = el + P.pe[r] * psi;
        cap = cap + P.pc[r] * psi;
        fis = fis + P.pf[r] * psi;
    }
    double nu = P.nu0 + P.nu1 * (E / 1.0e6);
    double a = cap + fis;
    XS4 out;
    out.t = el + a;
    out.a = a;
    out.f = fis;
    out.nf = nu * fis;
    return out;
}

struct GenOut {
    std::vector<double> E;
    std::vector<XS4> xs;
    double awr = 0;
    bool fissionable = false;
};

void generate(int g, uint64_t xs_seed, double ln_range, GenOut& out) {
    Params P;
    uint64_t s = derive_seed(xs_seed, (uint64_t)g);
    const int ng = 5000 + (int)(prn(s) * 12607.0);
    int cls, res_fis = 0;
    double lo = 0, hi = 0, plo, phi;
    if (g < N_NAMED) {
        const NucDef& d = NAMED[g];
        cls = d.cls;
        P.awr = d.awr; P.s0 = d.s0; P.c0 = d.c0; P.f0 = d.f0; P.f_fast = d.f_fast;
        P.ft = d.ft; P.nu0 = d.nu0; P.nu1 = d.nu1; P.nres = d.nres; P.h_rolloff = d.h_rolloff;
        lo = d.res_lo; hi = d.res_hi; res_fis = d.res_fis;
    } else {
        cls = CLS_FP;
        P.awr = 72.0 + 100.0 * prn(s);
        P.s0 = 3.0 + 9.0 * prn(s);
        P.c0 = det_exp10(-1.0 + 4.0 * prn(s));
        P.nres = 2 + (int)(16.0 * prn(s));
        if (g == G_FP0) P.c0 = 2.65e6;
        if (g == G_FP0 + 1) P.c0 = 4.1e4;
        lo = 1.0; hi = 1.0e4;
    }
    if (cls == CLS_STRUCT) { plo = 1.0; phi = 2.5; }
    else if (cls == CLS_ACTINIDE) { plo = 0.7; phi = 3.0; }
    else { plo = 1.0; phi = 3.5; }
    if (P.nres > MAX_RES) throw std::runtime_error("too many resonances");
    if (P.nres > 0) {
        double llo = det_log(lo), lhi = det_log(hi);
        for (int r = 0; r < P.nres; ++r) {
            double Er = det_exp(llo + (lhi - llo) * prn(s));
            double G = Er * det_exp10(-2.7 + 1.2 * prn(s));
            double pk = det_exp10(plo + (phi - plo) * prn(s));
            P.rE[r] = Er;
            P.rH[r] = 0.25 * G * G;
            if (cls == CLS_STRUCT) {
                P.pe[r] = 0.95 * pk; P.pc[r] = 0.05 * pk; P.pf[r] = 0.0;
            } else if (res_fis) {
                double ff = 0.3 + 0.5 * prn(s);
                P.pe[r] = 0.1 * pk; P.pc[r] = (1.0 - ff) * pk; P.pf[r] = ff * pk;
            } else {
                P.pe[r] = 0.1 * pk; P.pc[r] = pk; P.pf[r] = 0.0;
            }
        }
    }
    out.awr = P.awr;
    out.fissionable = (P.f0 > 0.0 || P.ft > 0.0);
    out.E.resize(ng);
    out.xs.resize(ng);
    out.E[0] = E_MIN;
    out.E[ng - 1] = E_MAX;
    for (int i = 1; i < ng - 1; ++i) {
        double t = ((double)i + 0.4 * (prn(s) - 0.5)) / (double)(ng - 1);
        out.E[i] = E_MIN * det_exp(t * ln_range);
    }
    for (int i = 0; i < ng; ++i) out.xs[i] = point_xs(P, out.E[i]);
}

// 17x17 guide-tube positions (row, col).
const int GT_POS[25][2] = {{2, 5}, {2, 8}, {2, 11}, {3, 3}, {3, 13}, {5, 2}, {5, 5}, {5, 8}, {5, 11},
                           {5, 14}, {8, 2}, {8, 5}, {8, 8}, {8, 11}, {8, 14}, {11, 2}, {11, 5},
                           {11, 8}, {11, 11}, {11, 14}, {13, 3}, {13, 13}, {14, 5}, {14, 8}, {14, 11}};

bool core_fuel_assembly(int ax, int ay) {
    static const int width[7] = {3, 5, 7, 7, 7, 5, 3};  // 37 assemblies (SMR-like core)
    int c0 = (7 - width[ay]) / 2;
    return ax >= c0 && ax < c0 + width[ay];
}

}  // namespace

uint64_t fnv1a(uint64_t h, const void* data, size_t n) {
    const unsigned char* c = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) {
        h ^= c[i];
        h *= 1099511628211ULL;
    }
    return h;
}

uint64_t library_checksum(const Problem& p) {
    uint64_t h = 1469598103934665603ULL;
    for (int n = 0; n < p.n_nuc; ++n) {
        int64_t o = p.goff[n], c = p.goff[n + 1] - p.goff[n];
        h = fnv1a(h, p.E.data() + o, sizeof(double) * (size_t)c);
        h = fnv1a(h, p.xs.data() + o, sizeof(XS4) * (size_t)c);
    }
    return h;
}

// Analytic check problem (kind INFINITE): an infinite homogeneous medium of
// one nuclide whose cross sections do not depend on energy (reflective box,
// every region the same material). Its expectations are exact and
// independent of this code base: k_inf = nu*Sigma_f / Sigma_a, every history
// is absorbed (the absorption estimator scores k_inf exactly), the mean number
// of collisions per history is Sigma_t / Sigma_a and the mean track length per
// history 1 / Sigma_a.
void build_infinite(Problem& p) {
    const double ln_range = det_log(E_MAX) - det_log(E_MIN);
    const int ng = INF_GRID;
    p.n_nuc = 1;
    p.global_id.assign(1, -1);
    p.awr.assign(1, INF_AWR);
    p.goff = {0, ng};
    p.E.resize(ng);
    p.xs.assign(ng, XS4{INF_SIGMA_T, INF_SIGMA_A, INF_SIGMA_F, INF_NU * INF_SIGMA_F});
    for (int i = 0; i < ng; ++i) p.E[i] = E_MIN * det_exp((double)i / (double)(ng - 1) * ln_range);
    p.E[0] = E_MIN;
    p.E[ng - 1] = E_MAX;
    p.mat.resize(3);
    for (auto& m : p.mat) {
        m.nuc = {0};
        m.dens = {1.0};
        m.fissionable = true;
    }
    Geometry& G = p.geo;
    for (auto& t : G.pt) t = PinType{0, {0.0, 0.0}, {MAT_FUEL, MAT_FUEL, MAT_FUEL}};
    G.pitch = 1.26;
    G.nx = G.ny = 1;
    G.bc_x = G.bc_y = G.bc_z = 1;
    G.x0 = G.y0 = -0.63;
    G.z_lo = -100.0;
    G.z_hi = 100.0;
    p.pin_map_host.assign(1, 0);
    G.pin_map = p.pin_map_host.data();
}

void build_problem(Problem& p, int kind, uint64_t xs_seed, int n_threads) {
    if (kind < PINCELL || kind > INFINITE) throw std::invalid_argument("unknown problem kind");
    auto t0 = std::chrono::steady_clock::now();
    p = Problem();
    p.kind = kind;
    p.xs_seed = xs_seed;
    if (kind == INFINITE) {
        build_infinite(p);
        p.gen_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return;
    }

    // material compositions in global ids (largest contributors first)
    std::vector<int> mg[3];
    std::vector<double> md[3];
    mg[MAT_WATER] = {G_H1, G_O16, G_B10, G_B11};
    md[MAT_WATER] = {4.94e-2, 2.47e-2, 8.0e-6, 3.2e-5};
    if (kind == PINCELL) {
        mg[MAT_CLAD] = {G_ZR90, G_ZR91, G_ZR92, G_ZR94};
        md[MAT_CLAD] = {2.18e-2, 4.75e-3, 7.26e-3, 7.36e-3};
        mg[MAT_FUEL] = {G_U238, G_O16, G_U235};
        md[MAT_FUEL] = {2.21e-2, 4.6e-2, 9.3e-4};
    } else {
        mg[MAT_CLAD] = {G_ZR90, G_ZR91, G_ZR92, G_ZR94, G_ZR96, G_FE56, G_CR52, G_SN118};
        md[MAT_CLAD] = {2.18e-2, 4.75e-3, 7.26e-3, 7.36e-3, 1.19e-3, 1.3e-4, 7.0e-5, 4.8e-4};
        mg[MAT_FUEL] = {G_U238, G_O16, G_U235, G_PU239, G_PU240, G_PU241,
                        G_U236, G_PU242, G_NP237, G_U234, G_PU238, G_AM241};
        md[MAT_FUEL] = {2.17e-2, 4.6e-2, 4.0e-4, 1.5e-4, 5.5e-5, 3.2e-5,
                        1.0e-4, 1.2e-5, 1.1e-5, 5.0e-6, 3.5e-6, 2.5e-6};
        uint64_t ms = derive_seed(xs_seed, 0xF00DULL);
        for (int k = 0; k < N_FP; ++k) {
            double d = det_exp10(-8.0 + 3.0 * prn(ms));
            if (k == 0) d = 1.0e-8;
            if (k == 1) d = 1.0e-7;
            mg[MAT_FUEL].push_back(G_FP0 + k);
            md[MAT_FUEL].push_back(d);
        }
    }

    std::vector<int> local(N_GLOBAL, -1);
    std::vector<char> used(N_GLOBAL, 0);
    for (int m = 0; m < 3; ++m)
        for (int g : mg[m]) used[g] = 1;
    for (int g = 0; g < N_GLOBAL; ++g)
        if (used[g]) {
            local[g] = p.n_nuc++;
            p.global_id.push_back(g);
        }

    // threaded generation (bit-identical for any thread count)
    const double ln_range = det_log(E_MAX) - det_log(E_MIN);
    std::vector<GenOut> gen(p.n_nuc);
    int nt = std::max(1, std::min(n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency(), p.n_nuc));
    std::atomic<int> next{0};
    std::vector<std::exception_ptr> errs(nt);
    auto work = [&](int t) {
        try {
            for (int i = next++; i < p.n_nuc; i = next++) generate(p.global_id[i], xs_seed, ln_range, gen[i]);
        } catch (...) {
            errs[t] = std::current_exception();
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);

    p.goff.resize(p.n_nuc + 1);
    p.goff[0] = 0;
    for (int n = 0; n < p.n_nuc; ++n) p.goff[n + 1] = p.goff[n] + (int64_t)gen[n].E.size();
    p.E.resize(p.goff.back());
    p.xs.resize(p.goff.back());
    p.awr.resize(p.n_nuc);
    std::vector<char> fiss(p.n_nuc);
    for (int n = 0; n < p.n_nuc; ++n) {
        std::copy(gen[n].E.begin(), gen[n].E.end(), p.E.begin() + p.goff[n]);
        std::copy(gen[n].xs.begin(), gen[n].xs.end(), p.xs.begin() + p.goff[n]);
        p.awr[n] = gen[n].awr;
        fiss[n] = gen[n].fissionable;
    }
    p.mat.resize(3);
    for (int m = 0; m < 3; ++m) {
        for (size_t i = 0; i < mg[m].size(); ++i) {
            int l = local[mg[m][i]];
            p.mat[m].nuc.push_back(l);
            p.mat[m].dens.push_back(md[m][i]);
            if (fiss[l]) p.mat[m].fissionable = true;
        }
    }

    // geometry
    Geometry& G = p.geo;
    G.pt[0] = PinType{2, {0.4096, 0.475}, {MAT_FUEL, MAT_CLAD, MAT_WATER}};
    G.pt[1] = PinType{2, {0.56, 0.602}, {MAT_WATER, MAT_CLAD, MAT_WATER}};
    G.pt[2] = PinType{0, {0.0, 0.0}, {MAT_WATER, MAT_WATER, MAT_WATER}};
    G.pitch = 1.26;
    if (kind == PINCELL) { G.nx = G.ny = 1; G.bc_x = G.bc_y = G.bc_z = 1; }
    else if (kind == ASSEMBLY) { G.nx = G.ny = 17; G.bc_x = G.bc_y = 1; G.bc_z = 0; }
    else { G.nx = G.ny = 7 * 17; G.bc_x = G.bc_y = G.bc_z = 0; }
    G.x0 = -0.5 * G.pitch * (double)G.nx;
    G.y0 = -0.5 * G.pitch * (double)G.ny;
    G.z_lo = -100.0;
    G.z_hi = 100.0;
    p.pin_map_host.assign((size_t)G.nx * G.ny, 0);
    for (int gy = 0; gy < G.ny; ++gy)
        for (int gx = 0; gx < G.nx; ++gx) {
            int t = 0;
            if (kind != PINCELL) {
                int ax = gx / 17, ay = gy / 17, lx = gx % 17, ly = gy % 17;
                if (kind == CORE && !core_fuel_assembly(ax, ay)) t = 2;
                else
                    for (auto& gt : GT_POS)
                        if (gt[0] == ly && gt[1] == lx) t = 1;
            }
            p.pin_map_host[(size_t)gy * G.nx + gx] = (uint8_t)t;
        }
    G.pin_map = p.pin_map_host.data();
    p.gen_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace omcg
