/*
 * omc_oracle.c — CPU oracle (history-based restatement) of the event-based
 * Monte Carlo transport loop tuned by arXiv 2402.09222.
 *
 * TEST INFRASTRUCTURE ONLY — see omc_oracle.h for the parity status
 * ("parity unpinned" for transport arithmetic; the reference ships none).
 *
 * Sources for every rule restated here:
 *   [P213]  PAPER.md:213  particles in flight never change the numerics
 *   [P217]  PAPER.md:217  log hash grid: bins narrow each nuclide's search
 *   [P219]  PAPER.md:219  event kernels: calculate_xs, advance, surface
 *                         crossing, collision (queued / queueless)
 *   [P221]  PAPER.md:221  sort by material and energy (affects time only)
 *   [P190]  PAPER.md:190  depleted fuel with 272 nuclides in total
 *   [P468]  PAPER.md:468  FoM = particles/s without initialisation
 *   [RNG]   proj/src/rng.hpp:10-25  splitmix64 / derive_seed (reference,
 *           pinned by tests/test_oracle_pins.py against oracle/_ref)
 *   [ext]   OpenMC public design: 64-bit LCG with PCG RXS-M-XS output and
 *           stride 152917, O(log n) skip-ahead (F. Brown 1994), log-hash
 *           grid search, elastic scattering in the CM frame, analog fission
 *           banking nu*sigma_f/sigma_t/k per collision.
 *
 * Determinism rules (shared with the CUDA product by specification, not by
 * code): compile with -ffp-contract=off; only + - * / sqrt, explicit fma()
 * where written (log/exp polynomials, XS interpolation and accumulation) and
 * the two polynomial transcendental functions below — all correctly rounded
 * IEEE operations; int64 fixed-point tallies.
 */
#define _GNU_SOURCE
#include "omc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

/* ------------------------------------------------------------------ */
/* errors                                                              */
/* ------------------------------------------------------------------ */
static __thread char g_err[512] = "";
static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return -1;
}
const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ */
/* constants                                                           */
/* ------------------------------------------------------------------ */
#define E_MIN 1.0e-5
#define E_MAX 2.0e7
#define KT 0.0253                  /* eV, 293.6 K */
#define FREE_GAS_CUTOFF (400.0 * KT)
#define TALLY_SCALE 268435456.0    /* 2^28 fixed point */
#define MAX_ADVANCE 100000
#define PRN_MULT 6364136223846793005ULL
#define PRN_ADD 1442695040888963407ULL
#define PRN_STRIDE 152917ULL
#define STREAM_TRACKING 0ULL
#define STREAM_BANK 1ULL
#define MATERIAL_STREAM 0xF00DULL
#define WATT_A 0.988e6
#define WATT_B 2.249e-6
#define SITE_PROGENY_BITS 24

enum { EV_XS = 0, EV_ADV = 1, EV_CROSS = 2, EV_COLL = 3, EV_DEAD = 4 };
enum { S_NONE = -1, S_XNEG = 0, S_XPOS, S_YNEG, S_YPOS, S_ZNEG, S_ZPOS, S_RING_OUT, S_RING_IN };
enum { MAT_WATER = 0, MAT_CLAD = 1, MAT_FUEL = 2 };

/* ------------------------------------------------------------------ */
/* deterministic math: log/exp from + - * / only                       */
/* ------------------------------------------------------------------ */
static inline uint64_t dbits(double x) { uint64_t b; memcpy(&b, &x, 8); return b; }
static inline double bitsd(uint64_t b) { double x; memcpy(&x, &b, 8); return x; }

#define LN2_HI 6.93147180369123816490e-01 /* 0x3fe62e42fee00000 */
#define LN2_LO 1.90821492927058770002e-10 /* 0x3dea39ef35793c76 */
#define SQRT2 1.41421356237309504880
#define INV_LN2 1.44269504088896338700e+00
#define LN10 2.30258509299404568402

/* log(x) for finite x > 0: x = m 2^e, m in (sqrt(1/2), sqrt(2)],
 * log m = 2 atanh(s), s = (m-1)/(m+1), odd series to s^23. */
double orc_log(double x) {
    uint64_t b = dbits(x);
    int e = (int)((b >> 52) & 0x7ff);
    if (e == 0) { /* subnormal: scale by 2^54 */
        x = x * 18014398509481984.0;
        b = dbits(x);
        e = (int)((b >> 52) & 0x7ff) - 54;
    }
    e -= 1023;
    double m = bitsd((b & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL);
    if (m > SQRT2) {
        m = m * 0.5;
        e = e + 1;
    }
    double s = (m - 1.0) / (m + 1.0);
    double s2 = s * s;
    double p = 1.0 / 23.0;
    p = fma(p, s2, 1.0 / 21.0);
    p = fma(p, s2, 1.0 / 19.0);
    p = fma(p, s2, 1.0 / 17.0);
    p = fma(p, s2, 1.0 / 15.0);
    p = fma(p, s2, 1.0 / 13.0);
    p = fma(p, s2, 1.0 / 11.0);
    p = fma(p, s2, 1.0 / 9.0);
    p = fma(p, s2, 1.0 / 7.0);
    p = fma(p, s2, 1.0 / 5.0);
    p = fma(p, s2, 1.0 / 3.0);
    double r = fma(2.0 * s, s2 * p, 2.0 * s);
    double de = (double)e;
    return fma(de, LN2_HI, fma(de, LN2_LO, r));
}

/* exp(x): x = k ln2 + r, |r| <= ln2/2, Taylor to r^14, scale by 2^k. */
double orc_exp(double x) {
    if (x > 709.0) return INFINITY;
    if (x < -708.0) return 0.0;
    double kd = floor(fma(x, INV_LN2, 0.5));
    int k = (int)kd;
    double r = fma(-kd, LN2_LO, fma(-kd, LN2_HI, x));
    double p = 1.0 / 87178291200.0; /* 1/14! */
    p = fma(p, r, 1.0 / 6227020800.0);
    p = fma(p, r, 1.0 / 479001600.0);
    p = fma(p, r, 1.0 / 39916800.0);
    p = fma(p, r, 1.0 / 3628800.0);
    p = fma(p, r, 1.0 / 362880.0);
    p = fma(p, r, 1.0 / 40320.0);
    p = fma(p, r, 1.0 / 5040.0);
    p = fma(p, r, 1.0 / 720.0);
    p = fma(p, r, 1.0 / 120.0);
    p = fma(p, r, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    /* multiply by 2^k in two steps so k in [-1022-52, 1023] stays exact */
    int k1 = k / 2, k2 = k - k / 2;
    double s1 = bitsd((uint64_t)(k1 + 1023) << 52);
    double s2 = bitsd((uint64_t)(k2 + 1023) << 52);
    return (p * s1) * s2;
}

static inline double exp10d(double x) { return orc_exp(x * LN10); }

/* ------------------------------------------------------------------ */
/* RNG                                                                 */
/* ------------------------------------------------------------------ */
/* [RNG] proj/src/rng.hpp:10-16 */
static inline uint64_t splitmix64(uint64_t* state) {
    *state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
/* [RNG] proj/src/rng.hpp:20-25 */
uint64_t orc_derive_seed(uint64_t base, uint64_t stream) {
    uint64_t state = base + stream * 0x9e3779b97f4a7c15ULL;
    uint64_t a = splitmix64(&state);
    uint64_t b = splitmix64(&state);
    return a ^ (b << 1);
}

/* [ext] LCG step + RXS-M-XS permutation; 53-bit uniform in [0,1). */
double orc_prn(uint64_t* seed) {
    *seed = PRN_MULT * *seed + PRN_ADD;
    uint64_t s = *seed;
    uint64_t word = ((s >> ((s >> 59u) + 5u)) ^ s) * 12605985483714917081ULL;
    uint64_t result = (word >> 43u) ^ word;
    return (double)(result >> 11) * 0x1.0p-53;
}

/* [ext] Brown 1994: x_n = G x_0 + C (mod 2^64) in O(log n). */
uint64_t orc_future_seed(uint64_t n, uint64_t seed) {
    uint64_t g = PRN_MULT, c = PRN_ADD, g_new = 1, c_new = 0;
    while (n > 0) {
        if (n & 1) {
            g_new *= g;
            c_new = c_new * g + c;
        }
        c = (g + 1) * c;
        g *= g;
        n >>= 1;
    }
    return g_new * seed + c_new;
}

static inline uint64_t stream_seed(uint64_t master, uint64_t id, uint64_t stream) {
    return orc_future_seed(id * PRN_STRIDE, master + stream);
}
uint64_t orc_particle_seed(uint64_t master_seed, uint64_t particle_id) {
    return stream_seed(master_seed, particle_id, STREAM_TRACKING);
}

/* ------------------------------------------------------------------ */
/* nuclide definitions (synthetic library; [P190] 272 nuclides)        */
/* ------------------------------------------------------------------ */
enum { CLS_LIGHT = 0, CLS_STRUCT = 1, CLS_ACTINIDE = 2, CLS_FP = 3 };

typedef struct {
    const char* name;
    int cls;
    double awr, s0, c0, f0, f_fast, ft, nu0, nu1;
    int nres;
    double res_lo, res_hi;
    int res_fis;   /* resonances carry a fission fraction */
    int h_rolloff; /* hydrogen-like elastic roll-off */
} nuc_def;

#define N_NAMED 23
#define N_FP 249
#define N_GLOBAL (N_NAMED + N_FP) /* 272 */

static const nuc_def NAMED[N_NAMED] = {
    /* name    cls          awr      s0    c0       f0     ffast ft    nu0   nu1  nres lo     hi    rf h */
    {"H1", CLS_LIGHT, 0.99917, 20.0, 0.332, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1},
    {"O16", CLS_STRUCT, 15.858, 3.9, 1.9e-4, 0, 0, 0, 0, 0, 3, 4.0e5, 4.0e6, 0, 0},
    {"B10", CLS_LIGHT, 9.9269, 2.2, 3840.0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},
    {"B11", CLS_LIGHT, 10.9147, 5.0, 5.5e-3, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},
    {"Zr90", CLS_STRUCT, 89.132, 6.5, 0.011, 0, 0, 0, 0, 0, 6, 2.0e3, 1.0e5, 0, 0},
    {"Zr91", CLS_STRUCT, 90.122, 9.7, 1.2, 0, 0, 0, 0, 0, 8, 2.0e2, 5.0e4, 0, 0},
    {"Zr92", CLS_STRUCT, 91.112, 7.3, 0.22, 0, 0, 0, 0, 0, 6, 5.0e2, 5.0e4, 0, 0},
    {"Zr94", CLS_STRUCT, 93.096, 6.2, 0.05, 0, 0, 0, 0, 0, 5, 2.0e3, 5.0e4, 0, 0},
    {"Zr96", CLS_STRUCT, 95.081, 6.2, 0.023, 0, 0, 0, 0, 0, 4, 3.0e2, 5.0e4, 0, 0},
    {"Fe56", CLS_STRUCT, 55.454, 11.6, 2.6, 0, 0, 0, 0, 0, 6, 1.0e3, 5.0e5, 0, 0},
    {"Cr52", CLS_STRUCT, 51.549, 3.0, 0.86, 0, 0, 0, 0, 0, 5, 1.0e3, 5.0e5, 0, 0},
    {"Sn118", CLS_STRUCT, 116.92, 4.9, 0.22, 0, 0, 0, 0, 0, 6, 40.0, 1.0e4, 0, 0},
    {"U234", CLS_ACTINIDE, 232.03, 10.0, 100.0, 0, 0, 1.2, 2.4, 0.13, 15, 5.0, 2.0e3, 0, 0},
    {"U235", CLS_ACTINIDE, 233.02, 12.0, 99.0, 585.0, 1.3, 0, 2.43, 0.12, 40, 0.3, 2.0e3, 1, 0},
    {"U236", CLS_ACTINIDE, 234.02, 8.5, 5.1, 0, 0, 0.6, 2.35, 0.13, 15, 5.0, 2.0e3, 0, 0},
    {"U238", CLS_ACTINIDE, 236.01, 9.3, 2.68, 0, 0, 0.55, 2.6, 0.15, 40, 6.0, 1.0e4, 0, 0},
    {"Np237", CLS_ACTINIDE, 235.01, 10.0, 175.0, 0, 0, 1.5, 2.7, 0.14, 20, 0.4, 2.0e3, 0, 0},
    {"Pu238", CLS_ACTINIDE, 236.0, 20.0, 540.0, 17.0, 2.0, 0, 2.9, 0.14, 12, 2.0, 2.0e3, 1, 0},
    {"Pu239", CLS_ACTINIDE, 236.99, 8.0, 270.0, 750.0, 1.7, 0, 2.87, 0.14, 35, 0.29, 2.0e3, 1, 0},
    {"Pu240", CLS_ACTINIDE, 237.99, 8.0, 290.0, 0, 0, 1.3, 2.8, 0.14, 20, 1.0, 2.0e3, 0, 0},
    {"Pu241", CLS_ACTINIDE, 238.98, 11.0, 360.0, 1010.0, 1.6, 0, 2.93, 0.14, 30, 0.26, 2.0e3, 1, 0},
    {"Pu242", CLS_ACTINIDE, 239.98, 8.0, 19.0, 0, 0, 1.2, 2.8, 0.14, 15, 2.6, 2.0e3, 0, 0},
    {"Am241", CLS_ACTINIDE, 238.99, 11.0, 600.0, 3.1, 0, 1.0, 2.9, 0.14, 20, 0.57, 2.0e3, 0, 0},
};
enum {
    G_H1 = 0, G_O16, G_B10, G_B11, G_ZR90, G_ZR91, G_ZR92, G_ZR94, G_ZR96, G_FE56, G_CR52,
    G_SN118, G_U234, G_U235, G_U236, G_U238, G_NP237, G_PU238, G_PU239, G_PU240, G_PU241,
    G_PU242, G_AM241, G_FP0
};

#define MAX_RES 64
typedef struct {
    double awr, s0, c0, f0, f_fast, ft, nu0, nu1;
    int h_rolloff, nres;
    double rE[MAX_RES], rH[MAX_RES], pe[MAX_RES], pc[MAX_RES], pf[MAX_RES];
} nuc_params;

/* point cross sections (barns): total, absorption, fission, nu-fission */
static void xs_point(const nuc_params* P, double E, double out[4]) {
    double inv_v = sqrt(0.0253 / E);
    double el = P->s0;
    if (P->h_rolloff) el = P->s0 / sqrt(1.0 + E / 1.0e5);
    double cap = P->c0 * inv_v;
    double fis = 0.0;
    if (P->f0 > 0.0) fis = P->f0 * inv_v + P->f_fast * E / (E + 1.0e3);
    if (P->ft > 0.0) fis = fis + P->ft / (1.0 + orc_exp((1.0e6 - E) / 1.5e5));
    for (int r = 0; r < P->nres; ++r) {
        double dE = E - P->rE[r];
        double psi = P->rH[r] / (dE * dE + P->rH[r]);
        el = el + P->pe[r] * psi;
        cap = cap + P->pc[r] * psi;
        fis = fis + P->pf[r] * psi;
    }
    double nu = P->nu0 + P->nu1 * (E / 1.0e6);
    double a = cap + fis;
    out[0] = el + a;
    out[1] = a;
    out[2] = fis;
    out[3] = nu * fis;
}

typedef struct {
    int n;       /* grid points */
    double* E;   /* n */
    double* xs;  /* 4n: total, absorption, fission, nu-fission */
    double awr;
    int fissionable;
} nuclide;

static double LN_RANGE, LOG_EMIN;
static pthread_once_t g_const_once = PTHREAD_ONCE_INIT;
static void init_consts(void) {
    LOG_EMIN = orc_log(E_MIN);
    LN_RANGE = orc_log(E_MAX) - LOG_EMIN;
}

/* Generate global nuclide g from stream derive_seed(xs_seed, g). */
static int gen_nuclide(int g, uint64_t xs_seed, nuclide* out) {
    nuc_params P;
    memset(&P, 0, sizeof P);
    uint64_t s = orc_derive_seed(xs_seed, (uint64_t)g);
    int ng = 5000 + (int)(orc_prn(&s) * 12607.0);
    int cls, res_fis = 0;
    double lo, hi, plo, phi;
    if (g < N_NAMED) {
        const nuc_def* d = &NAMED[g];
        cls = d->cls;
        P.awr = d->awr; P.s0 = d->s0; P.c0 = d->c0; P.f0 = d->f0; P.f_fast = d->f_fast;
        P.ft = d->ft; P.nu0 = d->nu0; P.nu1 = d->nu1; P.nres = d->nres; P.h_rolloff = d->h_rolloff;
        lo = d->res_lo; hi = d->res_hi; res_fis = d->res_fis;
    } else {
        cls = CLS_FP;
        P.awr = 72.0 + 100.0 * orc_prn(&s);
        P.s0 = 3.0 + 9.0 * orc_prn(&s);
        P.c0 = exp10d(-1.0 + 4.0 * orc_prn(&s));
        P.nres = 2 + (int)(16.0 * orc_prn(&s));
        if (g == G_FP0) P.c0 = 2.65e6;     /* Xe-135-like poison */
        if (g == G_FP0 + 1) P.c0 = 4.1e4;  /* Sm-149-like poison */
        lo = 1.0; hi = 1.0e4;
    }
    if (cls == CLS_STRUCT) { plo = 1.0; phi = 2.5; }
    else if (cls == CLS_ACTINIDE) { plo = 0.7; phi = 3.0; }
    else { plo = 1.0; phi = 3.5; }
    if (P.nres > MAX_RES) return fail("too many resonances");
    if (P.nres > 0) {
        double llo = orc_log(lo), lhi = orc_log(hi);
        for (int r = 0; r < P.nres; ++r) {
            double Er = orc_exp(llo + (lhi - llo) * orc_prn(&s));
            double G = Er * exp10d(-2.7 + 1.2 * orc_prn(&s));
            double pk = exp10d(plo + (phi - plo) * orc_prn(&s));
            P.rE[r] = Er;
            P.rH[r] = 0.25 * G * G;
            if (cls == CLS_STRUCT) {
                P.pe[r] = 0.95 * pk;
                P.pc[r] = 0.05 * pk;
                P.pf[r] = 0.0;
            } else if (res_fis) {
                double ff = 0.3 + 0.5 * orc_prn(&s);
                P.pe[r] = 0.1 * pk;
                P.pc[r] = (1.0 - ff) * pk;
                P.pf[r] = ff * pk;
            } else {
                P.pe[r] = 0.1 * pk;
                P.pc[r] = pk;
                P.pf[r] = 0.0;
            }
        }
    }
    out->n = ng;
    out->awr = P.awr;
    out->fissionable = (P.f0 > 0.0 || P.ft > 0.0);
    out->E = (double*)malloc(sizeof(double) * (size_t)ng);
    out->xs = (double*)malloc(sizeof(double) * 4 * (size_t)ng);
    if (!out->E || !out->xs) return fail("out of memory (library)");
    out->E[0] = E_MIN;
    out->E[ng - 1] = E_MAX;
    for (int i = 1; i < ng - 1; ++i) {
        double t = ((double)i + 0.4 * (orc_prn(&s) - 0.5)) / (double)(ng - 1);
        out->E[i] = E_MIN * orc_exp(t * LN_RANGE);
    }
    for (int i = 0; i < ng; ++i) xs_point(&P, out->E[i], out->xs + 4 * (size_t)i);
    return 0;
}

/* ------------------------------------------------------------------ */
/* materials and geometry                                              */
/* ------------------------------------------------------------------ */
typedef struct {
    int n;
    int* nuc;      /* local nuclide index */
    double* dens;  /* atoms / (barn cm) */
    int fissionable;
} material;

typedef struct {
    int nr;
    double r[4];
    int mat[5];
} pin_type;

typedef struct {
    int nx, ny;
    double pitch, x0, y0, z_lo, z_hi;
    int bc_x, bc_y, bc_z; /* 1 reflective, 0 vacuum */
    pin_type pt[3];
    unsigned char* pin_map; /* nx*ny pin type ids */
} geometry;

struct orc_problem {
    int kind, n_bins, n_nuc, n_mat;
    uint64_t xs_seed;
    nuclide* nuc;
    int* global_id;
    material mat[3];
    int32_t* hash; /* n_nuc * (n_bins+1), nuclide-major */
    double inv_spacing;
    geometry geo;
};

/* 17x17 guide-tube positions (row, col), standard PWR layout. */
static const int GT_POS[25][2] = {
    {2, 5}, {2, 8}, {2, 11}, {3, 3}, {3, 13}, {5, 2}, {5, 5}, {5, 8}, {5, 11}, {5, 14},
    {8, 2}, {8, 5}, {8, 8}, {8, 11}, {8, 14}, {11, 2}, {11, 5}, {11, 8}, {11, 11}, {11, 14},
    {13, 3}, {13, 13}, {14, 5}, {14, 8}, {14, 11}};

static int is_core_fuel_assembly(int ax, int ay) {
    static const int width[7] = {3, 5, 7, 7, 7, 5, 3};
    int w = width[ay];
    int c0 = (7 - w) / 2;
    return ax >= c0 && ax < c0 + w;
}

/* material nuclide lists in global ids (ordered: large contributors first) */
static const int WATER_G[4] = {G_H1, G_O16, G_B10, G_B11};
static const double WATER_D[4] = {4.94e-2, 2.47e-2, 8.0e-6, 3.2e-5};
static const int CLAD4_G[4] = {G_ZR90, G_ZR91, G_ZR92, G_ZR94};
static const double CLAD4_D[4] = {2.18e-2, 4.75e-3, 7.26e-3, 7.36e-3};
static const int CLAD8_G[8] = {G_ZR90, G_ZR91, G_ZR92, G_ZR94, G_ZR96, G_FE56, G_CR52, G_SN118};
static const double CLAD8_D[8] = {2.18e-2, 4.75e-3, 7.26e-3, 7.36e-3, 1.19e-3, 1.3e-4, 7.0e-5, 4.8e-4};
static const int FRESH_G[3] = {G_U238, G_O16, G_U235};
static const double FRESH_D[3] = {2.21e-2, 4.6e-2, 9.3e-4};
#define N_ACT_DEPLETED 12
static const int DEPL_G[N_ACT_DEPLETED] = {G_U238, G_O16, G_U235, G_PU239, G_PU240, G_PU241,
                                            G_U236, G_PU242, G_NP237, G_U234, G_PU238, G_AM241};
static const double DEPL_D[N_ACT_DEPLETED] = {2.17e-2, 4.6e-2, 4.0e-4, 1.5e-4, 5.5e-5, 3.2e-5,
                                               1.0e-4, 1.2e-5, 1.1e-5, 5.0e-6, 3.5e-6, 2.5e-6};

static void set_pin(pin_type* t, int nr, const double* r, const int* mats) {
    t->nr = nr;
    for (int i = 0; i < nr; ++i) t->r[i] = r[i];
    for (int i = 0; i <= nr; ++i) t->mat[i] = mats[i];
}

void orc_problem_free(orc_problem* p) {
    if (!p) return;
    if (p->nuc)
        for (int i = 0; i < p->n_nuc; ++i) {
            free(p->nuc[i].E);
            free(p->nuc[i].xs);
        }
    free(p->nuc);
    free(p->global_id);
    for (int m = 0; m < 3; ++m) {
        free(p->mat[m].nuc);
        free(p->mat[m].dens);
    }
    free(p->hash);
    free(p->geo.pin_map);
    free(p);
}

static int bin_of(const orc_problem* p, double E) {
    double t = (orc_log(E) - LOG_EMIN) * p->inv_spacing;
    if (!(t >= 0.0)) return 0;
    if (t >= (double)p->n_bins) return p->n_bins - 1;
    int b = (int)t;
    return b < p->n_bins ? b : p->n_bins - 1;
}

/* hash grid [P217]: hash[n][k] = last i with bin(E_i) < k (>= 0) */
static int build_hash(orc_problem* p) {
    const int n_bins = p->n_bins;
    p->inv_spacing = (double)n_bins / LN_RANGE;
    size_t hb = (size_t)(n_bins + 1);
    p->hash = (int32_t*)malloc(sizeof(int32_t) * hb * (size_t)p->n_nuc);
    if (!p->hash) return -1;
    for (int n = 0; n < p->n_nuc; ++n) {
        const nuclide* N = &p->nuc[n];
        for (int k = 0; k <= n_bins; ++k) {
            int lo = 0, hi = N->n - 1;
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                if (bin_of(p, N->E[mid]) < k) lo = mid + 1;
                else hi = mid;
            }
            p->hash[(size_t)n * hb + (size_t)k] = lo > 0 ? lo - 1 : 0;
        }
    }
    return 0;
}

/* Analytic check problem (ORC_INFINITE): infinite homogeneous medium of one
 * nuclide with energy-independent cross sections (1001-point log grid,
 * density 1 atom/(b cm)), every region fuel, reflective 1.26 x 1.26 x 200 cm
 * box. Exact expectations, independent of both code bases: k_inf =
 * nu*Sigma_f/Sigma_a, every history absorbed, Sigma_t/Sigma_a collisions and
 * 1/Sigma_a track length per history. */
static int build_infinite(orc_problem* p) {
    const int ng = ORC_INF_GRID;
    p->n_nuc = 1;
    p->nuc = (nuclide*)calloc(1, sizeof(nuclide));
    p->global_id = (int*)malloc(sizeof(int));
    if (!p->nuc || !p->global_id) return fail("out of memory");
    p->global_id[0] = -1;
    nuclide* N = &p->nuc[0];
    N->n = ng;
    N->awr = ORC_INF_AWR;
    N->fissionable = 1;
    N->E = (double*)malloc(sizeof(double) * (size_t)ng);
    N->xs = (double*)malloc(sizeof(double) * 4 * (size_t)ng);
    if (!N->E || !N->xs) return fail("out of memory");
    for (int i = 0; i < ng; ++i) {
        N->E[i] = E_MIN * orc_exp((double)i / (double)(ng - 1) * LN_RANGE);
        N->xs[4 * i] = ORC_INF_SIGMA_T;
        N->xs[4 * i + 1] = ORC_INF_SIGMA_A;
        N->xs[4 * i + 2] = ORC_INF_SIGMA_F;
        N->xs[4 * i + 3] = ORC_INF_NU * ORC_INF_SIGMA_F;
    }
    N->E[0] = E_MIN;
    N->E[ng - 1] = E_MAX;
    p->n_mat = 3;
    for (int m = 0; m < 3; ++m) {
        material* M = &p->mat[m];
        M->n = 1;
        M->nuc = (int*)malloc(sizeof(int));
        M->dens = (double*)malloc(sizeof(double));
        if (!M->nuc || !M->dens) return fail("out of memory");
        M->nuc[0] = 0;
        M->dens[0] = 1.0;
        M->fissionable = 1;
    }
    if (build_hash(p) != 0) return fail("out of memory (hash)");
    geometry* G = &p->geo;
    const int all_fuel[1] = {MAT_FUEL};
    for (int t = 0; t < 3; ++t) set_pin(&G->pt[t], 0, NULL, all_fuel);
    G->pitch = 1.26;
    G->nx = G->ny = 1;
    G->bc_x = G->bc_y = G->bc_z = 1;
    G->x0 = G->y0 = -0.63;
    G->z_lo = -100.0;
    G->z_hi = 100.0;
    G->pin_map = (unsigned char*)calloc(1, 1);
    if (!G->pin_map) return fail("out of memory");
    return 0;
}

int orc_problem_create(int kind, uint64_t xs_seed, int n_bins, orc_problem** out) {
    pthread_once(&g_const_once, init_consts);
    if (kind < ORC_PINCELL || kind > ORC_INFINITE) return fail("unknown problem kind");
    if (n_bins < 1 || n_bins > 10000000) return fail("n_bins out of range");
    orc_problem* p = (orc_problem*)calloc(1, sizeof *p);
    if (!p) return fail("out of memory");
    p->kind = kind;
    p->n_bins = n_bins;
    p->xs_seed = xs_seed;
    if (kind == ORC_INFINITE) {
        if (build_infinite(p) != 0) {
            orc_problem_free(p);
            return -1;
        }
        *out = p;
        return 0;
    }

    /* material composition in global ids */
    int mg_n[3];
    const int* mg_g[3];
    double* mg_d[3];
    int fp_g[N_FP];
    (void)fp_g;
    int fuel_n;
    int* fuel_g;
    double* fuel_d;
    if (kind == ORC_PINCELL) {
        fuel_n = 3;
        fuel_g = (int*)malloc(sizeof(int) * 3);
        fuel_d = (double*)malloc(sizeof(double) * 3);
        for (int i = 0; i < 3; ++i) { fuel_g[i] = FRESH_G[i]; fuel_d[i] = FRESH_D[i]; }
    } else {
        fuel_n = N_ACT_DEPLETED + N_FP;
        fuel_g = (int*)malloc(sizeof(int) * (size_t)fuel_n);
        fuel_d = (double*)malloc(sizeof(double) * (size_t)fuel_n);
        for (int i = 0; i < N_ACT_DEPLETED; ++i) { fuel_g[i] = DEPL_G[i]; fuel_d[i] = DEPL_D[i]; }
        uint64_t ms = orc_derive_seed(xs_seed, MATERIAL_STREAM);
        for (int k = 0; k < N_FP; ++k) {
            double d = exp10d(-8.0 + 3.0 * orc_prn(&ms));
            if (k == 0) d = 1.0e-8;
            if (k == 1) d = 1.0e-7;
            fuel_g[N_ACT_DEPLETED + k] = G_FP0 + k;
            fuel_d[N_ACT_DEPLETED + k] = d;
        }
    }
    mg_n[MAT_WATER] = 4; mg_g[MAT_WATER] = WATER_G;
    mg_d[MAT_WATER] = (double*)WATER_D;
    if (kind == ORC_PINCELL) { mg_n[MAT_CLAD] = 4; mg_g[MAT_CLAD] = CLAD4_G; mg_d[MAT_CLAD] = (double*)CLAD4_D; }
    else { mg_n[MAT_CLAD] = 8; mg_g[MAT_CLAD] = CLAD8_G; mg_d[MAT_CLAD] = (double*)CLAD8_D; }
    mg_n[MAT_FUEL] = fuel_n; mg_g[MAT_FUEL] = fuel_g; mg_d[MAT_FUEL] = fuel_d;

    /* library = used global ids, ascending */
    int used[N_GLOBAL];
    memset(used, 0, sizeof used);
    for (int m = 0; m < 3; ++m)
        for (int i = 0; i < mg_n[m]; ++i) used[mg_g[m][i]] = 1;
    int local[N_GLOBAL];
    p->n_nuc = 0;
    for (int g = 0; g < N_GLOBAL; ++g) local[g] = used[g] ? p->n_nuc++ : -1;
    p->nuc = (nuclide*)calloc((size_t)p->n_nuc, sizeof(nuclide));
    p->global_id = (int*)malloc(sizeof(int) * (size_t)p->n_nuc);
    for (int g = 0; g < N_GLOBAL; ++g)
        if (used[g]) {
            p->global_id[local[g]] = g;
            if (gen_nuclide(g, xs_seed, &p->nuc[local[g]]) != 0) {
                free(fuel_g); free(fuel_d);
                orc_problem_free(p);
                return -1;
            }
        }
    p->n_mat = 3;
    for (int m = 0; m < 3; ++m) {
        material* M = &p->mat[m];
        M->n = mg_n[m];
        M->nuc = (int*)malloc(sizeof(int) * (size_t)M->n);
        M->dens = (double*)malloc(sizeof(double) * (size_t)M->n);
        M->fissionable = 0;
        for (int i = 0; i < M->n; ++i) {
            M->nuc[i] = local[mg_g[m][i]];
            M->dens[i] = mg_d[m][i];
            if (p->nuc[M->nuc[i]].fissionable) M->fissionable = 1;
        }
    }
    free(fuel_g);
    free(fuel_d);

    if (build_hash(p) != 0) { orc_problem_free(p); return fail("out of memory (hash)"); }

    /* geometry */
    geometry* G = &p->geo;
    const double fuel_r[2] = {0.4096, 0.475};
    const int fuel_m[3] = {MAT_FUEL, MAT_CLAD, MAT_WATER};
    const double gt_r[2] = {0.56, 0.602};
    const int gt_m[3] = {MAT_WATER, MAT_CLAD, MAT_WATER};
    const int water_m[1] = {MAT_WATER};
    set_pin(&G->pt[0], 2, fuel_r, fuel_m);
    set_pin(&G->pt[1], 2, gt_r, gt_m);
    set_pin(&G->pt[2], 0, NULL, water_m);
    G->pitch = 1.26;
    if (kind == ORC_PINCELL) {
        G->nx = G->ny = 1;
        G->bc_x = G->bc_y = G->bc_z = 1;
    } else if (kind == ORC_ASSEMBLY) {
        G->nx = G->ny = 17;
        G->bc_x = G->bc_y = 1;
        G->bc_z = 0;
    } else {
        G->nx = G->ny = 7 * 17;
        G->bc_x = G->bc_y = G->bc_z = 0;
    }
    G->x0 = -0.5 * G->pitch * (double)G->nx;
    G->y0 = -0.5 * G->pitch * (double)G->ny;
    G->z_lo = -100.0;
    G->z_hi = 100.0;
    G->pin_map = (unsigned char*)calloc((size_t)G->nx * (size_t)G->ny, 1);
    for (int gy = 0; gy < G->ny; ++gy)
        for (int gx = 0; gx < G->nx; ++gx) {
            int t = 0;
            if (kind != ORC_PINCELL) {
                int ax = gx / 17, ay = gy / 17, lx = gx % 17, ly = gy % 17;
                if (kind == ORC_CORE && !is_core_fuel_assembly(ax, ay)) t = 2;
                else
                    for (int q = 0; q < 25; ++q)
                        if (GT_POS[q][0] == ly && GT_POS[q][1] == lx) t = 1;
            }
            G->pin_map[gy * G->nx + gx] = (unsigned char)t;
        }
    *out = p;
    return 0;
}

int orc_problem_get_info(const orc_problem* p, orc_problem_info* info) {
    if (!p || !info) return fail("null argument");
    memset(info, 0, sizeof *info);
    info->kind = p->kind;
    info->n_nuclides = p->n_nuc;
    info->n_materials = p->n_mat;
    info->n_bins = p->n_bins;
    info->nx = p->geo.nx;
    info->ny = p->geo.ny;
    info->n_tally_bins = p->geo.nx * p->geo.ny;
    info->fuel_material = MAT_FUEL;
    info->fuel_nuclides = p->mat[MAT_FUEL].n;
    for (int n = 0; n < p->n_nuc; ++n) info->n_grid_total += p->nuc[n].n;
    info->lib_bytes = info->n_grid_total * 40;
    info->hash_bytes = (int64_t)(p->n_bins + 1) * p->n_nuc * 4;
    return 0;
}

static uint64_t fnv(uint64_t h, const void* data, size_t n) {
    const unsigned char* c = (const unsigned char*)data;
    for (size_t i = 0; i < n; ++i) {
        h ^= c[i];
        h *= 1099511628211ULL;
    }
    return h;
}
uint64_t orc_library_checksum(const orc_problem* p) {
    uint64_t h = 1469598103934665603ULL;
    for (int n = 0; n < p->n_nuc; ++n) {
        h = fnv(h, p->nuc[n].E, sizeof(double) * (size_t)p->nuc[n].n);
        h = fnv(h, p->nuc[n].xs, sizeof(double) * 4 * (size_t)p->nuc[n].n);
    }
    return h;
}
uint64_t orc_hash_checksum(const orc_problem* p) {
    return fnv(1469598103934665603ULL, p->hash,
               sizeof(int32_t) * (size_t)(p->n_bins + 1) * (size_t)p->n_nuc);
}
int orc_nuclide_grid_size(const orc_problem* p, int nuc) {
    if (nuc < 0 || nuc >= p->n_nuc) return fail("nuclide out of range");
    return p->nuc[nuc].n;
}
int orc_nuclide_copy(const orc_problem* p, int nuc, double* E, double* xs) {
    if (nuc < 0 || nuc >= p->n_nuc) return fail("nuclide out of range");
    memcpy(E, p->nuc[nuc].E, sizeof(double) * (size_t)p->nuc[nuc].n);
    memcpy(xs, p->nuc[nuc].xs, sizeof(double) * 4 * (size_t)p->nuc[nuc].n);
    return 0;
}
int orc_hash_copy(const orc_problem* p, int nuc, int32_t* out) {
    if (nuc < 0 || nuc >= p->n_nuc) return fail("nuclide out of range");
    memcpy(out, p->hash + (size_t)nuc * (size_t)(p->n_bins + 1),
           sizeof(int32_t) * (size_t)(p->n_bins + 1));
    return 0;
}

/* ------------------------------------------------------------------ */
/* cross-section lookup [P217]                                         */
/* ------------------------------------------------------------------ */
/* Largest i with E_i <= E (clamped to [0, n-2]) using the hash bracket. */
static inline int grid_index(const orc_problem* p, int n, double E, int b, double* f) {
    const nuclide* N = &p->nuc[n];
    const double* Eg = N->E;
    int ng = N->n;
    if (E <= Eg[0]) { *f = 0.0; return 0; }
    if (E >= Eg[ng - 1]) { *f = 1.0; return ng - 2; }
    const int32_t* h = p->hash + (size_t)n * (size_t)(p->n_bins + 1);
    int lo = h[b], hi = h[b + 1] + 1;
    if (E < Eg[lo]) lo = 0;
    if (E >= Eg[hi]) hi = ng - 1;
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (Eg[mid] <= E) lo = mid;
        else hi = mid;
    }
    *f = (E - Eg[lo]) / (Eg[lo + 1] - Eg[lo]);
    return lo;
}

static inline double interp(const double* xs, int i, int c, double f) {
    double a = xs[4 * (size_t)i + c], b = xs[4 * (size_t)(i + 1) + c];
    return fma(f, b - a, a);
}

/* Macroscopic sums are segmented: the material's nuclides (in material order)
 * form segments of SEG_LEN; each segment is summed sequentially from 0 and the
 * segment sums are folded in order into the total. (Segments are independent
 * units of work for the GPU; for materials of <= SEG_LEN nuclides this is the
 * plain sequential sum.) */
#define SEG_LEN 16
static void macro_xs(const orc_problem* p, int m, double E, double out[4]) {
    const material* M = &p->mat[m];
    int b = bin_of(p, E);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int s0 = 0; s0 < M->n; s0 += SEG_LEN) {
        double seg[4] = {0.0, 0.0, 0.0, 0.0};
        int s1 = s0 + SEG_LEN < M->n ? s0 + SEG_LEN : M->n;
        for (int q = s0; q < s1; ++q) {
            int n = M->nuc[q];
            double f;
            int i = grid_index(p, n, E, b, &f);
            const double* xs = p->nuc[n].xs;
            double d = M->dens[q];
            for (int c = 0; c < 4; ++c) seg[c] = fma(d, interp(xs, i, c, f), seg[c]);
        }
        for (int c = 0; c < 4; ++c) acc[c] = acc[c] + seg[c];
    }
    for (int c = 0; c < 4; ++c) out[c] = acc[c];
}

/* macro_xs plus the folded running total after every segment but the last
 * (at most ORC_MAX_CKPT): the checkpoints the GPU's calculate_xs stores for the
 * collision's nuclide sampling (cum = folded earlier segments + running sum in
 * the segment, the order the collision below follows). */
#define ORC_MAX_CKPT 16
int orc_macro_xs_ckpt(const orc_problem* p, int mat, double E, double xs[4], double* ck, int* nck) {
    if (mat < 0 || mat >= p->n_mat) return fail("material out of range");
    const material* M = &p->mat[mat];
    int b = bin_of(p, E);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int k = 0;
    for (int s0 = 0; s0 < M->n; s0 += SEG_LEN) {
        double seg[4] = {0.0, 0.0, 0.0, 0.0};
        int s1 = s0 + SEG_LEN < M->n ? s0 + SEG_LEN : M->n;
        for (int q = s0; q < s1; ++q) {
            int n = M->nuc[q];
            double f;
            int i = grid_index(p, n, E, b, &f);
            const double* x = p->nuc[n].xs;
            double d = M->dens[q];
            for (int c = 0; c < 4; ++c) seg[c] = fma(d, interp(x, i, c, f), seg[c]);
        }
        for (int c = 0; c < 4; ++c) acc[c] = acc[c] + seg[c];
        if (s1 < M->n && k < ORC_MAX_CKPT) ck[k++] = acc[0];
    }
    for (int c = 0; c < 4; ++c) xs[c] = acc[c];
    *nck = k;
    return 0;
}

int orc_macro_xs_ckpt_n(const orc_problem* p, int64_t n, const int32_t* mat, const double* E, double* xs,
                        double* ck, int32_t* nck) {
    for (int64_t i = 0; i < n; ++i) {
        int k = 0;
        if (orc_macro_xs_ckpt(p, mat[i], E[i], xs + 4 * i, ck + ORC_MAX_CKPT * i, &k) != 0) return -1;
        nck[i] = k;
    }
    return 0;
}

int orc_hash_bin(const orc_problem* p, double E) { return bin_of(p, E); }
int orc_micro_xs(const orc_problem* p, int nuc, double E, int32_t* idx, double xs[4]) {
    if (nuc < 0 || nuc >= p->n_nuc) return fail("nuclide out of range");
    double f;
    int i = grid_index(p, nuc, E, bin_of(p, E), &f);
    if (idx) *idx = i;
    for (int c = 0; c < 4; ++c) xs[c] = interp(p->nuc[nuc].xs, i, c, f);
    return 0;
}
int orc_macro_xs(const orc_problem* p, int mat, double E, double xs[4]) {
    if (mat < 0 || mat >= p->n_mat) return fail("material out of range");
    macro_xs(p, mat, E, xs);
    return 0;
}

/* ------------------------------------------------------------------ */
/* particle physics                                                    */
/* ------------------------------------------------------------------ */
typedef struct {
    double x, y, z, u, v, w, E, wgt;
    double st, sa, sf, snf;
    uint64_t seed;
    int gx, gy, ring, mat, surf;
    int n_xs, n_adv, n_cross, n_coll, n_sites, term;
    int64_t gidx;
} particle;

typedef struct {
    double x, y, z, E;
    uint64_t key;
} site;

typedef struct {
    int64_t* tally;   /* n_tally_bins * 4 */
    int64_t k_coll, k_abs, k_track;
    int64_t n_events[4];
    int64_t n_leak, n_abs, n_lost;
    site* bank;
    int64_t n_bank, cap_bank;
    int error;
} accum;

static inline int64_t fx(double x) { return (int64_t)(x * TALLY_SCALE + 0.5); }

static inline int pin_type_at(const geometry* G, int gx, int gy) { return G->pin_map[gy * G->nx + gx]; }

/* polar-method pair of standard normals (rejection, no trig) */
static void gauss_pair(uint64_t* s, double* g1, double* g2) {
    double a, b, r2;
    do {
        a = 2.0 * orc_prn(s) - 1.0;
        b = 2.0 * orc_prn(s) - 1.0;
        r2 = a * a + b * b;
    } while (r2 >= 1.0 || r2 == 0.0);
    double f = sqrt(-2.0 * orc_log(r2) / r2);
    *g1 = a * f;
    *g2 = b * f;
}

/* azimuth cos/sin by rejection on the unit disk */
static void azimuth(uint64_t* s, double* c, double* sn) {
    double a, b, r2;
    do {
        a = 2.0 * orc_prn(s) - 1.0;
        b = 2.0 * orc_prn(s) - 1.0;
        r2 = a * a + b * b;
    } while (r2 > 1.0 || r2 == 0.0);
    *c = (a * a - b * b) / r2;
    *sn = 2.0 * a * b / r2;
}

static void isotropic(uint64_t* s, double* u, double* v, double* w) {
    double mu = 2.0 * orc_prn(s) - 1.0;
    double c, sn;
    azimuth(s, &c, &sn);
    double st = sqrt(1.0 - mu * mu);
    *u = mu;
    *v = st * c;
    *w = st * sn;
}

/* [ext] Maxwellian as Gamma(3/2): T*(Exp(1) + N(0,1)^2/2) */
static double maxwell(uint64_t* s, double T) {
    double e1 = -orc_log(1.0 - orc_prn(s));
    double g1, g2;
    gauss_pair(s, &g1, &g2);
    return T * (e1 + 0.5 * g1 * g1);
}
/* [ext] Watt fission spectrum via a Maxwellian; resample outside [E_MIN, E_MAX) */
static double watt(uint64_t* s) {
    double E;
    do {
        double w = maxwell(s, WATT_A);
        E = w + WATT_A * WATT_A * WATT_B / 4.0 + (2.0 * orc_prn(s) - 1.0) * sqrt(WATT_A * WATT_A * WATT_B * w);
    } while (E < E_MIN || E >= E_MAX);
    return E;
}

/* [ext] rotate direction by polar cosine mu with sampled azimuth */
static void rotate(uint64_t* s, double mu, double* u, double* v, double* w) {
    double c, sn;
    azimuth(s, &c, &sn);
    double a = sqrt(fmax(0.0, 1.0 - mu * mu));
    double u0 = *u, v0 = *v, w0 = *w;
    if (fabs(w0) < 0.9999) {
        double b = sqrt(1.0 - w0 * w0);
        *u = mu * u0 + a * (u0 * w0 * c - v0 * sn) / b;
        *v = mu * v0 + a * (v0 * w0 * c + u0 * sn) / b;
        *w = mu * w0 - a * b * c;
    } else {
        double b = sqrt(1.0 - v0 * v0);
        *u = mu * u0 + a * (u0 * v0 * c + w0 * sn) / b;
        *v = mu * v0 - a * b * c;
        *w = mu * w0 + a * (v0 * w0 * c - u0 * sn) / b;
    }
}

static void locate(const orc_problem* p, particle* q) {
    const geometry* G = &p->geo;
    int gx = (int)floor((q->x - G->x0) / G->pitch);
    int gy = (int)floor((q->y - G->y0) / G->pitch);
    if (gx < 0) gx = 0;
    if (gx >= G->nx) gx = G->nx - 1;
    if (gy < 0) gy = 0;
    if (gy >= G->ny) gy = G->ny - 1;
    const pin_type* T = &G->pt[pin_type_at(G, gx, gy)];
    double lx = q->x - (G->x0 + ((double)gx + 0.5) * G->pitch);
    double ly = q->y - (G->y0 + ((double)gy + 0.5) * G->pitch);
    double r2 = lx * lx + ly * ly;
    int ring = T->nr;
    for (int r = 0; r < T->nr; ++r)
        if (r2 < T->r[r] * T->r[r]) { ring = r; break; }
    q->gx = gx;
    q->gy = gy;
    q->ring = ring;
    q->mat = T->mat[ring];
}

/* Initialise history gidx of batch `batch` (1-based) from `src` or, for
 * batch 1 (src == NULL), from the uniform-in-fuel Watt source. */
static int init_particle(const orc_problem* p, particle* q, uint64_t master, int batch, int64_t N,
                         int64_t gidx, const site* src) {
    memset(q, 0, sizeof *q);
    uint64_t id = (uint64_t)(batch - 1) * (uint64_t)N + (uint64_t)gidx + 1;
    q->seed = stream_seed(master, id, STREAM_TRACKING);
    q->gidx = gidx;
    const geometry* G = &p->geo;
    if (!src) {
        int tries = 0;
        for (;;) {
            q->x = G->x0 + orc_prn(&q->seed) * (G->pitch * (double)G->nx);
            q->y = G->y0 + orc_prn(&q->seed) * (G->pitch * (double)G->ny);
            q->z = G->z_lo + orc_prn(&q->seed) * (G->z_hi - G->z_lo);
            locate(p, q);
            if (p->mat[q->mat].fissionable) break;
            if (++tries > 100000) return fail("source rejection sampling failed");
        }
        q->E = watt(&q->seed);
    } else {
        q->x = src->x; q->y = src->y; q->z = src->z; q->E = src->E;
        locate(p, q);
    }
    isotropic(&q->seed, &q->u, &q->v, &q->w);
    q->wgt = 1.0;
    q->surf = S_NONE;
    return 0;
}

static void distance_to_boundary(const orc_problem* p, const particle* q, double* dist, int* surf) {
    const geometry* G = &p->geo;
    const pin_type* T = &G->pt[pin_type_at(G, q->gx, q->gy)];
    double half = 0.5 * G->pitch;
    double lx = q->x - (G->x0 + ((double)q->gx + 0.5) * G->pitch);
    double ly = q->y - (G->y0 + ((double)q->gy + 0.5) * G->pitch);
    double d = INFINITY, dd;
    int s = S_NONE;
    if (q->u > 0.0) { dd = (half - lx) / q->u; if (dd < 0.0) dd = 0.0; if (dd < d) { d = dd; s = S_XPOS; } }
    else if (q->u < 0.0) { dd = (-half - lx) / q->u; if (dd < 0.0) dd = 0.0; if (dd < d) { d = dd; s = S_XNEG; } }
    if (q->v > 0.0) { dd = (half - ly) / q->v; if (dd < 0.0) dd = 0.0; if (dd < d) { d = dd; s = S_YPOS; } }
    else if (q->v < 0.0) { dd = (-half - ly) / q->v; if (dd < 0.0) dd = 0.0; if (dd < d) { d = dd; s = S_YNEG; } }
    if (q->w > 0.0) { dd = (G->z_hi - q->z) / q->w; if (dd < 0.0) dd = 0.0; if (dd < d) { d = dd; s = S_ZPOS; } }
    else if (q->w < 0.0) { dd = (G->z_lo - q->z) / q->w; if (dd < 0.0) dd = 0.0; if (dd < d) { d = dd; s = S_ZNEG; } }
    double a = q->u * q->u + q->v * q->v;
    if (a > 0.0) {
        double k = lx * q->u + ly * q->v;
        double c0 = lx * lx + ly * ly;
        if (q->ring < T->nr) {
            double R = T->r[q->ring];
            double disc = k * k - a * (c0 - R * R);
            if (disc < 0.0) disc = 0.0;
            dd = (-k + sqrt(disc)) / a;
            if (dd < 0.0) dd = 0.0;
            if (dd < d) { d = dd; s = S_RING_OUT; }
        }
        if (q->ring > 0 && k < 0.0) {
            double R = T->r[q->ring - 1];
            double disc = k * k - a * (c0 - R * R);
            if (disc >= 0.0) {
                dd = (-k - sqrt(disc)) / a;
                if (dd < 0.0) dd = 0.0;
                if (dd < d) { d = dd; s = S_RING_IN; }
            }
        }
    }
    *dist = d;
    *surf = s;
}

static int ev_xs(const orc_problem* p, particle* q) {
    double m[4];
    macro_xs(p, q->mat, q->E, m);
    q->st = m[0]; q->sa = m[1]; q->sf = m[2]; q->snf = m[3];
    q->n_xs++;
    return EV_ADV;
}

static int ev_advance(const orc_problem* p, particle* q, accum* A) {
    q->n_adv++;
    if (q->n_adv > MAX_ADVANCE) {
        q->term = ORC_TERM_LOST;
        return EV_DEAD;
    }
    double xi = orc_prn(&q->seed);
    double d_coll = -orc_log(1.0 - xi) / q->st;
    double d_surf;
    int surf;
    distance_to_boundary(p, q, &d_surf, &surf);
    double d;
    int next;
    if (d_coll < d_surf) { d = d_coll; next = EV_COLL; }
    else { d = d_surf; next = EV_CROSS; q->surf = surf; }
    q->x = q->x + d * q->u;
    q->y = q->y + d * q->v;
    q->z = q->z + d * q->w;
    double t = q->wgt * d;
    int64_t* tb = A->tally + 4 * (size_t)(q->gy * p->geo.nx + q->gx);
    tb[0] += fx(t);
    tb[1] += fx(t * q->sa);
    tb[2] += fx(t * q->sf);
    tb[3] += fx(t * q->snf);
    A->k_track += fx(t * q->snf);
    return next;
}

static int ev_cross(const orc_problem* p, particle* q) {
    const geometry* G = &p->geo;
    q->n_cross++;
    int old = q->mat;
    switch (q->surf) {
    case S_RING_OUT: q->ring++; break;
    case S_RING_IN: q->ring--; break;
    case S_XPOS:
    case S_XNEG: {
        int nx = q->gx + (q->surf == S_XPOS ? 1 : -1);
        if (nx >= 0 && nx < G->nx) { q->gx = nx; q->ring = G->pt[pin_type_at(G, q->gx, q->gy)].nr; }
        else if (G->bc_x) q->u = -q->u;
        else { q->term = ORC_TERM_LEAKED; return EV_DEAD; }
        break;
    }
    case S_YPOS:
    case S_YNEG: {
        int ny = q->gy + (q->surf == S_YPOS ? 1 : -1);
        if (ny >= 0 && ny < G->ny) { q->gy = ny; q->ring = G->pt[pin_type_at(G, q->gx, q->gy)].nr; }
        else if (G->bc_y) q->v = -q->v;
        else { q->term = ORC_TERM_LEAKED; return EV_DEAD; }
        break;
    }
    case S_ZPOS:
    case S_ZNEG:
        if (G->bc_z) q->w = -q->w;
        else { q->term = ORC_TERM_LEAKED; return EV_DEAD; }
        break;
    default: break;
    }
    q->mat = G->pt[pin_type_at(G, q->gx, q->gy)].mat[q->ring];
    return q->mat != old ? EV_XS : EV_ADV;
}

static int push_site(accum* A, const particle* q, double E) {
    if (A->n_bank == A->cap_bank) {
        int64_t nc = A->cap_bank ? 2 * A->cap_bank : 4096;
        site* nb = (site*)realloc(A->bank, sizeof(site) * (size_t)nc);
        if (!nb) return -1;
        A->bank = nb;
        A->cap_bank = nc;
    }
    site* s = &A->bank[A->n_bank++];
    s->x = q->x; s->y = q->y; s->z = q->z; s->E = E;
    s->key = ((uint64_t)q->gidx << SITE_PROGENY_BITS) | (uint64_t)q->n_sites;
    return 0;
}

static int ev_collide(const orc_problem* p, particle* q, accum* A, double k_norm) {
    q->n_coll++;
    const material* M = &p->mat[q->mat];
    int b = bin_of(p, q->E);
    /* sample the target nuclide from the cumulative rho_n sigma_t,n, accumulated
     * with the same segmented sums as macro_xs: cum = (folded earlier segments)
     * + (running sum inside the current segment) */
    double cutoff = orc_prn(&q->seed) * q->st;
    double acc = 0.0;
    int sel = M->n - 1, found = 0;
    for (int s0 = 0; s0 < M->n && !found; s0 += SEG_LEN) {
        int s1 = s0 + SEG_LEN < M->n ? s0 + SEG_LEN : M->n;
        double seg = 0.0;
        for (int j = s0; j < s1; ++j) {
            double f;
            int n = M->nuc[j];
            int i = grid_index(p, n, q->E, b, &f);
            seg = fma(M->dens[j], interp(p->nuc[n].xs, i, 0, f), seg);
            if (acc + seg > cutoff) { sel = j; found = 1; break; }
        }
        acc = acc + seg;
    }
    int n = M->nuc[sel];
    double f;
    int i = grid_index(p, n, q->E, b, &f);
    const double* xs = p->nuc[n].xs;
    double mt = interp(xs, i, 0, f), ma = interp(xs, i, 1, f), mnf = interp(xs, i, 3, f);
    A->k_coll += fx(q->wgt * q->snf / q->st);
    /* analog fission banking [ext] */
    if (mnf > 0.0) {
        double nu_t = q->wgt / k_norm * mnf / mt;
        int ns = (int)nu_t;
        if (orc_prn(&q->seed) < nu_t - (double)ns) ns++;
        for (int k = 0; k < ns; ++k) {
            double Es = watt(&q->seed);
            if (q->n_sites >= (1 << SITE_PROGENY_BITS) - 1) { A->error = 1; break; }
            if (push_site(A, q, Es) != 0) { A->error = 1; break; }
            q->n_sites++;
        }
    }
    /* absorption vs scattering */
    if (orc_prn(&q->seed) * mt < ma) {
        if (ma > 0.0) A->k_abs += fx(q->wgt * mnf / ma);
        q->term = ORC_TERM_ABSORBED;
        return EV_DEAD;
    }
    /* elastic scattering, isotropic in CM; free-gas target below 400 kT */
    double A_ = p->nuc[n].awr;
    double vel = sqrt(q->E);
    double vx = vel * q->u, vy = vel * q->v, vz = vel * q->w;
    double tx = 0.0, ty = 0.0, tz = 0.0;
    if (q->E < FREE_GAS_CUTOFF) {
        double sg = sqrt(KT / (2.0 * A_));
        double g1, g2, g3, g4;
        gauss_pair(&q->seed, &g1, &g2);
        gauss_pair(&q->seed, &g3, &g4);
        tx = sg * g1; ty = sg * g2; tz = sg * g3;
    }
    double cx = (vx + A_ * tx) / (A_ + 1.0);
    double cy = (vy + A_ * ty) / (A_ + 1.0);
    double cz = (vz + A_ * tz) / (A_ + 1.0);
    vx = vx - cx; vy = vy - cy; vz = vz - cz;
    double sp = sqrt(vx * vx + vy * vy + vz * vz);
    double mu = 2.0 * orc_prn(&q->seed) - 1.0;
    if (sp > 0.0) {
        double dx = vx / sp, dy = vy / sp, dz = vz / sp;
        rotate(&q->seed, mu, &dx, &dy, &dz);
        vx = sp * dx + cx; vy = sp * dy + cy; vz = sp * dz + cz;
    } else {
        vx = cx; vy = cy; vz = cz;
    }
    q->E = vx * vx + vy * vy + vz * vz;
    double nv = sqrt(q->E);
    q->u = vx / nv; q->v = vy / nv; q->w = vz / nv;
    return EV_XS;
}

/* One history, event by event [P219]: XS -> ADV -> (COLL | CROSS) -> ... */
static void transport(const orc_problem* p, particle* q, accum* A, double k_norm) {
    int ev = EV_XS;
    while (ev != EV_DEAD) {
        switch (ev) {
        case EV_XS: ev = ev_xs(p, q); break;
        case EV_ADV: ev = ev_advance(p, q, A); break;
        case EV_CROSS: ev = ev_cross(p, q); break;
        default: ev = ev_collide(p, q, A, k_norm); break;
        }
    }
    A->n_events[0] += q->n_xs;
    A->n_events[1] += q->n_adv;
    A->n_events[2] += q->n_cross;
    A->n_events[3] += q->n_coll;
    if (q->term == ORC_TERM_LEAKED) A->n_leak++;
    else if (q->term == ORC_TERM_ABSORBED) A->n_abs++;
    else A->n_lost++;
}

/* ------------------------------------------------------------------ */
/* queued event-loop emulation (queue contents)          */
/* ------------------------------------------------------------------ */
/* Restates the queued scheduling policy of the product's event loop so the
 * per-iteration queue contents can be compared: an in-flight bank of P1 slots;
 * each iteration reads the queue lengths, runs every particle of the longest
 * queue (ties: fuel XS, non-fuel XS, advance, crossing, collision) and then
 * refills the slots that were empty at the start of the iteration from the
 * source; once the source is exhausted and at most
 * tail_threshold histories are alive, all of them are finished at once
 * (recorded as queue 5). Trace entries: (queue, length, sum of mix64(id+1)).
 * event_fusion (the product's default, omcg_run_config.event_fusion): the
 * advance queue is the "move" queue — each of its histories runs flights,
 * surface crossings and non-fuel calculate_xs back to back until it needs a
 * calculate_xs in a fissionable (fuel) material, collides, or dies; every
 * non-fuel lookup (after a non-fuel collision, or of a new history) is done in
 * the move queue. move_cap > 0 (omcg_run_config.move_event_cap): a history
 * leaves a move iteration after at most move_cap events (the cross-section
 * cache hit that follows a crossing is part of the crossing) and stays in the
 * move queue, whatever its next event. */
enum { Q_XS_FUEL = 0, Q_XS_NONFUEL = 1, Q_ADV = 2, Q_CROSS = 3, Q_COLL = 4, Q_DEAD = 5 };

static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

int orc_queue_trace(const orc_problem* p, int64_t n_particles, uint64_t seed, int64_t in_flight,
                    int64_t tail_threshold, int event_fusion, int move_cap, int64_t* out, int64_t max_entries,
                    int64_t* n_out) {
    if (!p || !n_out || n_particles < 1 || in_flight < 1) return fail("invalid queue-trace arguments");
    int64_t cap = in_flight < n_particles ? in_flight : n_particles;
    particle* slots = (particle*)malloc(sizeof(particle) * (size_t)cap);
    int* ev = (int*)malloc(sizeof(int) * (size_t)cap);
    int* pend = (int*)malloc(sizeof(int) * (size_t)cap); /* pending event of each slot (the move
                                                              queue holds flights and non-fuel lookups) */
    /* per-slot cross-section cache: energy of the last lookup of each material,
     * and the last many-nuclide (> SEG_LEN) material looked up (whose segment
     * checkpoints the product keeps) */
    double* cache_E = (double*)malloc(sizeof(double) * 3 * (size_t)cap);
    int* cache_m = (int*)calloc((size_t)cap, sizeof(int));
    accum A;
    memset(&A, 0, sizeof A);
    A.tally = (int64_t*)calloc(4 * (size_t)p->geo.nx * (size_t)p->geo.ny, sizeof(int64_t));
    if (!slots || !ev || !pend || !A.tally || !cache_E || !cache_m) {
        free(slots); free(ev); free(pend); free(A.tally); free(cache_E); free(cache_m);
        return fail("out of memory");
    }
    for (int64_t s = 0; s < cap; ++s) ev[s] = Q_DEAD;
    int64_t next = 0, n = 0;
    int rc = 0;
    for (;;) {
        int64_t len[6] = {0, 0, 0, 0, 0, 0};
        for (int64_t s = 0; s < cap; ++s) len[ev[s]]++;
        int64_t live = len[0] + len[1] + len[2] + len[3] + len[4];
        int64_t dead = len[Q_DEAD];
        if (live == 0 && next >= n_particles) break;
        if (live > 0) {
            int best = 0;
            for (int k = 1; k < 5; ++k)
                if (len[k] > len[best]) best = k;
            int tail = next >= n_particles && live <= tail_threshold;
            int move = event_fusion && best == Q_ADV && !tail;
            uint64_t chk = 0;
            for (int64_t s = 0; s < cap; ++s) {
                if (ev[s] == Q_DEAD || (!tail && ev[s] != best)) continue;
                particle* q = &slots[s];
                chk += mix64((uint64_t)q->gidx + 1ULL);
                int e = pend[s], steps = 0;
                do {  /* one event, or the whole remainder in the tail */
                    const int prev = e;
                    steps++;
                    switch (e) {
                    case EV_XS: e = ev_xs(p, q); break;
                    case EV_ADV: e = ev_advance(p, q, &A); break;
                    case EV_CROSS: e = ev_cross(p, q); break;
                    default: e = ev_collide(p, q, &A, 1.0); break;
                    }
                    /* cross-section cache: a history re-entering a material at the energy
                     * of its last lookup of that material takes that lookup's (identical)
                     * values at once and goes straight to advance (OpenMC skips unchanged
                     * lookups too); a many-nuclide material only while it is still the
                     * last many-nuclide material looked up */
                    if (prev == EV_XS) {
                        cache_E[3 * s + q->mat] = q->E;
                        if (p->mat[q->mat].n > SEG_LEN) cache_m[s] = q->mat;
                    }
                    if (prev == EV_CROSS && e == EV_XS && cache_E[3 * s + q->mat] == q->E &&
                        (p->mat[q->mat].n <= SEG_LEN || cache_m[s] == q->mat))
                        e = ev_xs(p, q);
                } while (e != EV_DEAD &&
                         (tail || (move && !((e == EV_XS && p->mat[q->mat].fissionable) || e == EV_COLL) &&
                                   !(move_cap > 0 && steps >= move_cap))));
                pend[s] = e;
                ev[s] = e == EV_DEAD ? Q_DEAD
                        : e == EV_XS ? (p->mat[q->mat].fissionable ? Q_XS_FUEL : event_fusion ? Q_ADV : Q_XS_NONFUEL)
                        : e == EV_ADV ? Q_ADV : e == EV_CROSS ? (event_fusion ? Q_ADV : Q_CROSS) : Q_COLL;
            }
            if (out && n < max_entries) {
                out[3 * n] = tail ? Q_DEAD : best;
                out[3 * n + 1] = tail ? live : len[best];
                out[3 * n + 2] = (int64_t)chk;
            }
            n++;
        }
        /* refill slots that were empty when the iteration started */
        if (dead > 0 && next < n_particles) {
            int64_t k = dead < n_particles - next ? dead : n_particles - next;
            for (int64_t s = 0; s < cap && k > 0; ++s) {
                if (ev[s] != Q_DEAD) continue;
                if (init_particle(p, &slots[s], seed, 1, n_particles, next, NULL) != 0) { rc = -1; break; }
                cache_E[3 * s] = cache_E[3 * s + 1] = cache_E[3 * s + 2] = -1.0;
                cache_m[s] = -1;
                ev[s] = p->mat[slots[s].mat].fissionable ? Q_XS_FUEL : event_fusion ? Q_ADV : Q_XS_NONFUEL;
                pend[s] = EV_XS;
                next++;
                k--;
            }
            if (rc) break;
        }
    }
    *n_out = n;
    free(slots); free(ev); free(pend); free(A.tally); free(A.bank); free(cache_E); free(cache_m);
    return rc;
}

/* ------------------------------------------------------------------ */
/* batch driver (threaded over histories)                              */
/* ------------------------------------------------------------------ */
typedef struct {
    const orc_problem* p;
    uint64_t master;
    int batch;
    int64_t N;
    const site* source; /* NULL for batch 1 */
    double k_norm;
    _Atomic int64_t next;
    orc_record* records;
    int64_t record_n;
    int nbins;
} batch_job;

typedef struct {
    batch_job* job;
    accum acc;
} worker;

static void* worker_main(void* arg) {
    worker* W = (worker*)arg;
    batch_job* J = W->job;
    particle q;
    for (;;) {
        int64_t start = atomic_fetch_add(&J->next, 256);
        if (start >= J->N) break;
        int64_t end = start + 256 < J->N ? start + 256 : J->N;
        for (int64_t g = start; g < end; ++g) {
            if (init_particle(J->p, &q, J->master, J->batch, J->N, g, J->source ? &J->source[g] : NULL) != 0) {
                W->acc.error = 2;
                return NULL;
            }
            transport(J->p, &q, &W->acc, J->k_norm);
            if (J->records && g < J->record_n) {
                orc_record* r = &J->records[g];
                r->n_xs = q.n_xs; r->n_adv = q.n_adv; r->n_cross = q.n_cross; r->n_coll = q.n_coll;
                r->n_sites = q.n_sites; r->term = q.term; r->e_final = q.E; r->x_final = q.x;
            }
        }
    }
    return NULL;
}

static int cmp_site(const void* a, const void* b) {
    uint64_t ka = ((const site*)a)->key, kb = ((const site*)b)->key;
    return ka < kb ? -1 : ka > kb;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

int orc_run(const orc_problem* p, const orc_run_config* cfg, orc_run_result* res, int64_t* tally_out,
            orc_record* records) {
    if (!p || !cfg || !res) return fail("null argument");
    if (cfg->n_particles < 1 || cfg->n_batches < 1 || cfg->n_batches > ORC_MAX_BATCHES ||
        cfg->n_inactive < 0 || cfg->n_inactive >= cfg->n_batches)
        return fail("invalid run configuration");
    if (cfg->n_particles >= ((int64_t)1 << (63 - SITE_PROGENY_BITS))) return fail("too many particles");
    memset(res, 0, sizeof *res);
    int nth = cfg->n_threads > 0 ? cfg->n_threads : (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nth < 1) nth = 1;
    int nbins = p->geo.nx * p->geo.ny;
    int64_t N = cfg->n_particles;
    if (tally_out) memset(tally_out, 0, sizeof(int64_t) * 4 * (size_t)nbins);
    worker* W = (worker*)calloc((size_t)nth, sizeof(worker));
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nth);
    site* source = NULL;
    site* merged = NULL;
    double k_norm = 1.0;
    double ksum = 0.0, ksq = 0.0;
    int n_active = 0;
    double t0 = now_s(), t_act0 = 0.0;
    int nb = cfg->n_batches;
    if (cfg->stop_after_batch > 0 && cfg->stop_after_batch < nb) nb = cfg->stop_after_batch;
    int rc = 0;
    for (int batch = 1; batch <= nb; ++batch) {
        if (batch == cfg->n_inactive + 1) t_act0 = now_s();
        batch_job J;
        J.p = p; J.master = cfg->seed; J.batch = batch; J.N = N; J.source = source; J.k_norm = k_norm;
        atomic_store(&J.next, 0);
        J.records = (records && batch == cfg->record_batch) ? records : NULL;
        J.record_n = cfg->record_n;
        J.nbins = nbins;
        for (int t = 0; t < nth; ++t) {
            memset(&W[t].acc, 0, sizeof(accum));
            W[t].acc.tally = (int64_t*)calloc(4 * (size_t)nbins, sizeof(int64_t));
            W[t].job = &J;
            pthread_create(&th[t], NULL, worker_main, &W[t]);
        }
        for (int t = 0; t < nth; ++t) pthread_join(th[t], NULL);
        /* merge (integer sums: order independent) */
        int64_t kc = 0, ka = 0, kt = 0, nsites = 0;
        for (int t = 0; t < nth; ++t) {
            accum* A = &W[t].acc;
            if (A->error) rc = fail(A->error == 2 ? "source sampling failed" : "fission bank overflow");
            kc += A->k_coll; ka += A->k_abs; kt += A->k_track; nsites += A->n_bank;
            for (int e = 0; e < 4; ++e) res->n_events[e] += A->n_events[e];
            res->n_leaked += A->n_leak; res->n_absorbed += A->n_abs; res->n_lost += A->n_lost;
            if (tally_out && batch > cfg->n_inactive)
                for (int i = 0; i < 4 * nbins; ++i) tally_out[i] += A->tally[i];
        }
        free(merged);
        merged = (site*)malloc(sizeof(site) * (size_t)(nsites > 0 ? nsites : 1));
        int64_t off = 0;
        for (int t = 0; t < nth; ++t) {
            accum* A = &W[t].acc;
            if (A->n_bank) memcpy(merged + off, A->bank, sizeof(site) * (size_t)A->n_bank);
            off += A->n_bank;
            free(A->bank);
            free(A->tally);
        }
        if (rc) break;
        double dN = (double)N;
        res->k_coll[batch - 1] = (double)kc / TALLY_SCALE / dN;
        res->k_abs[batch - 1] = (double)ka / TALLY_SCALE / dN;
        res->k_track[batch - 1] = (double)kt / TALLY_SCALE / dN;
        res->n_sites[batch - 1] = nsites;
        if (batch > cfg->n_inactive) {
            ksum += res->k_coll[batch - 1];
            ksq += res->k_coll[batch - 1] * res->k_coll[batch - 1];
            n_active++;
        }
        k_norm = res->k_coll[batch - 1];
        res->n_batches_run = batch;
        if (nsites == 0) { rc = fail("fission bank empty"); break; }
        if (batch == nb) break;
        /* canonical order, then systematic resampling to N [ext] */
        qsort(merged, (size_t)nsites, sizeof(site), cmp_site);
        uint64_t bs = stream_seed(cfg->seed, (uint64_t)batch, STREAM_BANK);
        uint64_t S = (uint64_t)nsites;
        uint64_t o = (uint64_t)(orc_prn(&bs) * (double)S);
        if (o >= S) o = S - 1;
        free(source);
        source = (site*)malloc(sizeof(site) * (size_t)N);
        for (int64_t i = 0; i < N; ++i) source[i] = merged[((uint64_t)i * S + o) / (uint64_t)N];
    }
    double t1 = now_s();
    res->t_total = t1 - t0;
    res->t_active = n_active > 0 ? t1 - t_act0 : 0.0;
    if (n_active > 0) {
        res->k_mean = ksum / (double)n_active;
        double var = n_active > 1 ? (ksq / (double)n_active - res->k_mean * res->k_mean) / (double)(n_active - 1) : 0.0;
        res->k_std = var > 0.0 ? sqrt(var) : 0.0;
        res->fom = res->t_active > 0.0 ? (double)N * (double)n_active / res->t_active : 0.0;
    }
    free(source);
    free(merged);
    free(W);
    free(th);
    return rc;
}
