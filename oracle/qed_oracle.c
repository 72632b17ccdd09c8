/*
 * qed_oracle.c -- the PARITY ORACLE for tree-level n-photon Compton |M|^2.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2511_19456_b200/, libqed.so) never links, imports
 * or calls anything under oracle/, and this file shares no code, header,
 * table or constant with it.
 *
 * What it computes (the plain definition; §1.4 lines 62-68,
 * §3.1):
 *
 *   M(h) = e^N * sum over all N! orderings pi of the N photons on the single
 *          electron line of
 *            ubar(p',s') epsslash_{pi(N)} S(Q_{N-1}) ... S(Q_1) epsslash_{pi(1)} u(p,s)
 *   with Q_j = p + sum_{l<=j} q_{pi(l)},  q = +k (incoming photon), -k (outgoing),
 *   S(Q) = (Qslash + m) / (Q^2 - m^2)   (i and i*eps dropped: DESIGN.md readings R3/R4),
 *   one factor e per vertex (reading R2), overall phases (-i)^N i^(N-1) dropped
 *   (common to every diagram; |M|^2 unaffected).
 *
 *   |M|^2 is |M(h)|^2 for fixed h, or sum over the summed particles' states
 *   times 1/2 per summed INITIAL particle (average) -- SURVEY.md §8(c) item 7.
 *
 * Evaluation is deliberately naive: dense 4x4 complex Dirac matrices (Dirac
 * representation, "Dirac's gamma matrices"),
 * every diagram chained matrix-by-matrix, every helicity configuration
 * recomputed from scratch.  No sharing, no blocking.
 *
 * Precision: REAL is double by default; compiled a second time with
 * -DORACLE_REAL="long double" for the conditioning check.
 *
 * Parity pins (tests/test_oracle_pins.py): Klein-Nishina closed forms (n=1),
 * the spin-summed trace identity (independent algorithm, chiral basis),
 * the Feynman-gauge polarisation sum, Ward identity, Lorentz invariance,
 * Bose symmetry, the soft-photon limit and the (n+1)! diagram count.
 */
#include <complex.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef ORACLE_REAL
#define ORACLE_REAL double
#endif
typedef ORACLE_REAL real;
typedef ORACLE_REAL _Complex cplx;

#define MAX_PHOTONS 9
#define MAX_EXT (MAX_PHOTONS + 2)

/* electron mass and fine-structure constant (CODATA 2018). */
static const real MASS_E = 1;
static const real ALPHA = 1 / 137.035999084L;

/* ---------------------------------------------------------------- algebra */

/* gamma^mu in the Dirac representation:
   gamma^0 = diag(1,1,-1,-1), gamma^i = [[0, sigma^i], [-sigma^i, 0]]. */
static void dirac_gammas(cplx g[4][4][4]) {
    memset(g, 0, sizeof(cplx) * 64);
    cplx sig[3][2][2] = {
        {{0, 1}, {1, 0}},
        {{0, -I}, {I, 0}},
        {{1, 0}, {0, -1}},
    };
    g[0][0][0] = 1; g[0][1][1] = 1; g[0][2][2] = -1; g[0][3][3] = -1;
    for (int i = 0; i < 3; i++)
        for (int r = 0; r < 2; r++)
            for (int c = 0; c < 2; c++) {
                g[i + 1][r][c + 2] = sig[i][r][c];
                g[i + 1][r + 2][c] = -sig[i][r][c];
            }
}

/* aslash = gamma^mu a_mu = gamma^0 a^0 - gamma^i a^i (metric +,-,-,-). */
static void slash(const cplx a[4], cplx out[4][4]) {
    cplx g[4][4][4];
    dirac_gammas(g);
    for (int r = 0; r < 4; r++)
        for (int c = 0; c < 4; c++)
            out[r][c] = g[0][r][c] * a[0] - g[1][r][c] * a[1] - g[2][r][c] * a[2] - g[3][r][c] * a[3];
}

static void matvec(cplx m[4][4], const cplx v[4], cplx out[4]) {
    cplx t[4];
    for (int r = 0; r < 4; r++) {
        t[r] = 0;
        for (int c = 0; c < 4; c++) t[r] += m[r][c] * v[c];
    }
    memcpy(out, t, sizeof t);
}

static real minkowski_sq(const real a[4]) { return a[0] * a[0] - a[1] * a[1] - a[2] * a[2] - a[3] * a[3]; }

/* ------------------------------------------------------- external states */

/* u(p,s) = sqrt(E+m) (chi_s ; sigma.p chi_s / (E+m)), chi_up=(1,0), chi_down=(0,1)
   (normalisation ubar u = 2m). */
static void spinor_u(const real p[4], int s, cplx u[4]) {
    real E = p[0];
    real n = sqrtl(E + MASS_E);
    cplx chi[2] = {s == 0 ? 1 : 0, s == 0 ? 0 : 1};
    /* sigma.p = [[pz, px - i py], [px + i py, -pz]] */
    cplx sp[2][2] = {{p[3], p[1] - I * p[2]}, {p[1] + I * p[2], -p[3]}};
    u[0] = n * chi[0];
    u[1] = n * chi[1];
    u[2] = n * (sp[0][0] * chi[0] + sp[0][1] * chi[1]) / (E + MASS_E);
    u[3] = n * (sp[1][0] * chi[0] + sp[1][1] * chi[1]) / (E + MASS_E);
}

/* ubar = u^dagger gamma^0 */
static void spinor_ubar(const real p[4], int s, cplx ub[4]) {
    cplx u[4];
    spinor_u(p, s, u);
    ub[0] = conj(u[0]);
    ub[1] = conj(u[1]);
    ub[2] = -conj(u[2]);
    ub[3] = -conj(u[3]);
}

/* Linear polarisation basis (PAPER.md:402 PolX):
   theta = atan2(k_perp, k_z), phi = atan2(k_y, k_x) (phi := 0 if k_perp = 0),
   eps1 = (0, cos t cos f, cos t sin f, -sin t), eps2 = (0, -sin f, cos f, 0).
   Real, so eps* = eps for outgoing photons. */
static void polvec(const real k[4], int lam, real eps[4]) {
    real kperp = sqrtl(k[1] * k[1] + k[2] * k[2]);
    real th = atan2l(kperp, k[3]);
    real ph = kperp == 0 ? 0 : atan2l(k[2], k[1]);
    eps[0] = 0;
    if (lam == 0) {
        eps[1] = cosl(th) * cosl(ph);
        eps[2] = cosl(th) * sinl(ph);
        eps[3] = -sinl(th);
    } else {
        eps[1] = -sinl(ph);
        eps[2] = cosl(ph);
        eps[3] = 0;
    }
}

/* ------------------------------------------------------------ diagram sum */

/* next lexicographic permutation; returns 0 after the last one */
static int next_perm(int* a, int n) {
    int i = n - 2;
    while (i >= 0 && a[i] >= a[i + 1]) i--;
    if (i < 0) return 0;
    int j = n - 1;
    while (a[j] <= a[i]) j--;
    int t = a[i]; a[i] = a[j]; a[j] = t;
    for (int l = i + 1, r = n - 1; l < r; l++, r--) { t = a[l]; a[l] = a[r]; a[r] = t; }
    return 1;
}

/* Sum over all N! photon orderings of
     ubar epsslash_{pi(N)} S(Q_{N-1}) ... S(Q_1) epsslash_{pi(1)} u
   for explicit external wave functions (complex eps allowed, for the Ward
   identity and Feynman-gauge tests).  q: signed photon momenta.
   Returns the number of diagrams summed; *amp excludes the coupling. */
static long diagram_sum(int N, const real q[][4], const real p[4], const cplx u[4], const cplx ub[4],
                        const cplx eps[][4], cplx* amp) {
    cplx eslash[MAX_PHOTONS][4][4];
    for (int i = 0; i < N; i++) slash(eps[i], eslash[i]);
    int perm[MAX_PHOTONS];
    for (int i = 0; i < N; i++) perm[i] = i;
    long n_diagrams = 0;
    cplx total = 0;
    do {
        cplx v[4];
        memcpy(v, u, sizeof v);
        real Q[4] = {p[0], p[1], p[2], p[3]};
        for (int l = 0; l < N; l++) {
            matvec(eslash[perm[l]], v, v);              /* vertex: epsslash */
            if (l < N - 1) {                            /* propagator S(Q_l) */
                for (int mu = 0; mu < 4; mu++) Q[mu] += q[perm[l]][mu];
                cplx Qc[4] = {Q[0], Q[1], Q[2], Q[3]};
                cplx S[4][4];
                slash(Qc, S);
                for (int r = 0; r < 4; r++) S[r][r] += MASS_E;
                real den = minkowski_sq(Q) - MASS_E * MASS_E;
                matvec(S, v, v);
                for (int r = 0; r < 4; r++) v[r] /= den;
            }
        }
        cplx m = 0;
        for (int r = 0; r < 4; r++) m += ub[r] * v[r];
        total += m;
        n_diagrams++;
    } while (next_perm(perm, N));
    *amp = total;
    return n_diagrams;
}

/* ------------------------------------------------------------ process API */

/* Particle order: e-_in, gamma_in..., e-_out, gamma_out...
   momenta: mom[(point*n_ext + j)*4 + mu], mu = (E, px, py, pz), units of m_e.
   Helicity configuration index h: bit j = spin (0 up, 1 down) or
   polarisation (0 = eps1, 1 = eps2) of external particle j. */
typedef struct {
    int n_in_ph, n_out_ph, N, n_ext;
} proc_t;

static int proc_init(proc_t* P, int n_in_ph, int n_out_ph) {
    if (n_in_ph < 0 || n_out_ph < 0) return -1;
    P->n_in_ph = n_in_ph;
    P->n_out_ph = n_out_ph;
    P->N = n_in_ph + n_out_ph;
    P->n_ext = P->N + 2;
    if (P->N < 1 || P->N > MAX_PHOTONS) return -1;
    return 0;
}
static int idx_e_in(const proc_t* P) { (void)P; return 0; }
static int idx_e_out(const proc_t* P) { return P->n_in_ph + 1; }
/* particle index of photon i (photons numbered in particle order) */
static int idx_photon(const proc_t* P, int i) { return i < P->n_in_ph ? 1 + i : P->n_in_ph + 2 + (i - P->n_in_ph); }
static int photon_incoming(const proc_t* P, int i) { return i < P->n_in_ph; }

/* All 2^(N+2) helicity amplitudes at one point, including e^N. */
static long point_amps(const proc_t* P, const double* mom, cplx* amps) {
    real e = sqrtl(4 * (real)M_PI * ALPHA);
    real en = 1;
    for (int i = 0; i < P->N; i++) en *= e;
    real p[4], pp[4], k[MAX_PHOTONS][4], q[MAX_PHOTONS][4];
    for (int mu = 0; mu < 4; mu++) {
        p[mu] = mom[idx_e_in(P) * 4 + mu];
        pp[mu] = mom[idx_e_out(P) * 4 + mu];
    }
    for (int i = 0; i < P->N; i++)
        for (int mu = 0; mu < 4; mu++) {
            k[i][mu] = mom[idx_photon(P, i) * 4 + mu];
            q[i][mu] = photon_incoming(P, i) ? k[i][mu] : -k[i][mu];
        }
    long H = 1L << P->n_ext;
    long nd = 0;
    for (long h = 0; h < H; h++) {
        cplx u[4], ub[4], eps[MAX_PHOTONS][4];
        spinor_u(p, (h >> idx_e_in(P)) & 1, u);
        spinor_ubar(pp, (h >> idx_e_out(P)) & 1, ub);
        for (int i = 0; i < P->N; i++) {
            real ev[4];
            polvec(k[i], (h >> idx_photon(P, i)) & 1, ev);
            for (int mu = 0; mu < 4; mu++) eps[i][mu] = ev[mu];
        }
        cplx a;
        nd = diagram_sum(P->N, (const real(*)[4])q, p, u, ub, (const cplx(*)[4])eps, &a);
        amps[h] = en * a;
    }
    return nd;
}

/* |M|^2 at one point for the given spec: spec[j] = -1 summed over particle
   j's two states (averaged, x1/2, if j is initial), 0/1 = fixed state. */
static real point_msq(const proc_t* P, const double* mom, const int8_t* spec) {
    long H = 1L << P->n_ext;
    cplx amps[1L << MAX_EXT];
    point_amps(P, mom, amps);
    real s = 0;
    for (long h = 0; h < H; h++) {
        int ok = 1;
        for (int j = 0; j < P->n_ext; j++)
            if (spec[j] >= 0 && ((h >> j) & 1) != spec[j]) ok = 0;
        if (ok) s += creal(amps[h] * conj(amps[h]));
    }
    int n_initial = 1 + P->n_in_ph;
    for (int j = 0; j < n_initial; j++)
        if (spec[j] < 0) s *= 0.5L;
    return s;
}

/* ------------------------------------------------------------ threading */

typedef struct {
    const proc_t* P;
    const double* mom;
    const int8_t* spec;
    double* out;        /* msq or amps */
    long begin, end;
    int want_amps;
} job_t;

static void* worker(void* arg) {
    job_t* J = (job_t*)arg;
    long H = 1L << J->P->n_ext;
    for (long i = J->begin; i < J->end; i++) {
        const double* m = J->mom + i * J->P->n_ext * 4;
        if (J->want_amps) {
            cplx amps[1L << MAX_EXT];
            point_amps(J->P, m, amps);
            for (long h = 0; h < H; h++) {
                J->out[(i * H + h) * 2] = (double)creal(amps[h]);
                J->out[(i * H + h) * 2 + 1] = (double)cimag(amps[h]);
            }
        } else {
            J->out[i] = (double)point_msq(J->P, m, J->spec);
        }
    }
    return NULL;
}

static int run_parallel(const proc_t* P, const double* mom, long n_points, const int8_t* spec, double* out,
                        int want_amps, int n_threads) {
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    if (n_points < n_threads) n_threads = n_points > 0 ? (int)n_points : 1;
    pthread_t th[256];
    job_t jobs[256];
    for (int t = 0; t < n_threads; t++) {
        jobs[t] = (job_t){P, mom, spec, out, n_points * t / n_threads, n_points * (t + 1) / n_threads, want_amps};
        if (t > 0) pthread_create(&th[t], NULL, worker, &jobs[t]);
    }
    worker(&jobs[0]);
    for (int t = 1; t < n_threads; t++) pthread_join(th[t], NULL);
    return 0;
}

/* ------------------------------------------------------------ exported C API */

/* |M|^2 per point.  Returns 0 on success, -1 on bad arguments. */
int oracle_msq(int n_in_ph, int n_out_ph, const double* mom, long n_points, const int8_t* spec, double* out,
               int n_threads) {
    proc_t P;
    if (proc_init(&P, n_in_ph, n_out_ph)) return -1;
    int8_t all_summed[MAX_EXT];
    if (!spec) {
        for (int j = 0; j < P.n_ext; j++) all_summed[j] = -1;
        spec = all_summed;
    }
    return run_parallel(&P, mom, n_points, spec, out, 0, n_threads);
}

/* All helicity amplitudes per point (with e^N): amps[(point*H + h)*2 + {0,1}]. */
int oracle_amps(int n_in_ph, int n_out_ph, const double* mom, long n_points, double* amps, int n_threads) {
    proc_t P;
    if (proc_init(&P, n_in_ph, n_out_ph)) return -1;
    return run_parallel(&P, mom, n_points, NULL, amps, 1, n_threads);
}

/* Diagram sum for explicit external wave functions (no coupling factor):
   eps: N complex 4-vectors (contravariant) interleaved re/im [N][4][2];
   q: signed photon momenta [N][4]; u, ubar: [4][2].  Returns the number of
   diagrams (N!).  Used by the Ward-identity and Feynman-gauge pins. */
long oracle_diagram_sum_explicit(int N, const double* q, const double* p, const double* u, const double* ubar,
                                 const double* eps, double* amp) {
    if (N < 1 || N > MAX_PHOTONS) return -1;
    real qq[MAX_PHOTONS][4], pp[4];
    cplx uu[4], ub[4], ee[MAX_PHOTONS][4];
    for (int mu = 0; mu < 4; mu++) {
        pp[mu] = p[mu];
        uu[mu] = u[2 * mu] + I * u[2 * mu + 1];
        ub[mu] = ubar[2 * mu] + I * ubar[2 * mu + 1];
    }
    for (int i = 0; i < N; i++)
        for (int mu = 0; mu < 4; mu++) {
            qq[i][mu] = q[i * 4 + mu];
            ee[i][mu] = eps[(i * 4 + mu) * 2] + I * eps[(i * 4 + mu) * 2 + 1];
        }
    cplx a;
    long nd = diagram_sum(N, (const real(*)[4])qq, pp, uu, ub, (const cplx(*)[4])ee, &a);
    amp[0] = (double)creal(a);
    amp[1] = (double)cimag(a);
    return nd;
}

/* external states, exposed for the unit pins */
void oracle_spinor_u(const double* p, int s, double* out) {
    real pp[4] = {p[0], p[1], p[2], p[3]};
    cplx u[4];
    spinor_u(pp, s, u);
    for (int i = 0; i < 4; i++) { out[2 * i] = (double)creal(u[i]); out[2 * i + 1] = (double)cimag(u[i]); }
}
void oracle_spinor_ubar(const double* p, int s, double* out) {
    real pp[4] = {p[0], p[1], p[2], p[3]};
    cplx u[4];
    spinor_ubar(pp, s, u);
    for (int i = 0; i < 4; i++) { out[2 * i] = (double)creal(u[i]); out[2 * i + 1] = (double)cimag(u[i]); }
}
void oracle_polvec(const double* k, int lam, double* out) {
    real kk[4] = {k[0], k[1], k[2], k[3]};
    real e[4];
    polvec(kk, lam, e);
    for (int i = 0; i < 4; i++) out[i] = (double)e[i];
}
/* gamma^mu (Dirac rep) as [4][4][4][2] */
void oracle_gammas(double* out) {
    cplx g[4][4][4];
    dirac_gammas(g);
    for (int i = 0; i < 64; i++) {
        out[2 * i] = (double)creal(((cplx*)g)[i]);
        out[2 * i + 1] = (double)cimag(((cplx*)g)[i]);
    }
}
double oracle_coupling_e(void) { return (double)sqrtl(4 * (real)M_PI * ALPHA); }
int oracle_real_bytes(void) { return (int)sizeof(real); }

/* ======================================================================================
 * Monte-Carlo cross-section oracle (the paper gives no phase-space
 * algorithm, PAPER.md line 288 -- reading R9 in DESIGN.md).  Plain transcription of:
 *   - Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), key = seed, counter =
 *     (index_lo, index_hi, particle, draw); u = ((hi << 21 | lo >> 11) + 0.5) 2^-53;
 *   - massive RAMBO (Kleiss, Stirling, Ellis, CPC 40 (1986) 359, rambo.f conventions) for
 *     e- gamma -> e- + n gamma in the CM frame (photon along +z, electron along -z);
 *   - weight x cut (every outgoing photon E >= omega_min) x |M|^2 (point_msq above),
 *     summed per chunk of `chunk` consecutive global indices.
 * ====================================================================================== */

typedef struct { uint32_t v[4]; } u32x4;

static u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
    for (int r = 0; r < 10; r++) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c.v[0];
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c.v[2];
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        u32x4 n = {{hi1 ^ c.v[1] ^ k0, lo1, hi0 ^ c.v[3] ^ k1, lo0}};
        c = n;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

void oracle_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
    u32x4 c = {{ctr[0], ctr[1], ctr[2], ctr[3]}};
    u32x4 r = philox4x32_10(c, key[0], key[1]);
    for (int i = 0; i < 4; i++) out[i] = r.v[i];
}

static double u53(uint32_t hi, uint32_t lo) {
    uint64_t r = ((uint64_t)hi << 21) | (lo >> 11);
    return ((double)r + 0.5) * 0x1.0p-53;
}

/* One phase-space point: momenta [n+3][4] in particle order e_in, g_in, e_out, g_out...;
   returns the RAMBO weight. */
double oracle_rambo_point(int n_out_ph, double sqrt_s, uint64_t seed, uint64_t idx, double* mom) {
    int K = n_out_ph + 1;
    double s = sqrt_s * sqrt_s;
    double q[MAX_PHOTONS + 1][4], Q[4] = {0, 0, 0, 0};
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (int i = 0; i < K; i++) {
        u32x4 ca = {{(uint32_t)idx, (uint32_t)(idx >> 32), (uint32_t)i, 0u}};
        u32x4 cb = {{(uint32_t)idx, (uint32_t)(idx >> 32), (uint32_t)i, 1u}};
        u32x4 a = philox4x32_10(ca, k0, k1), b = philox4x32_10(cb, k0, k1);
        double r1 = u53(a.v[0], a.v[1]), r2 = u53(a.v[2], a.v[3]);
        double r3 = u53(b.v[0], b.v[1]), r4 = u53(b.v[2], b.v[3]);
        double c = 2 * r1 - 1, st = sqrt(1 - c * c), f = 2 * M_PI * r2;
        double q0 = -log(r3 * r4);
        q[i][0] = q0;
        q[i][1] = q0 * st * cos(f);
        q[i][2] = q0 * st * sin(f);
        q[i][3] = q0 * c;
        for (int mu = 0; mu < 4; mu++) Q[mu] += q[i][mu];
    }
    /* conformal transformation to total momentum (sqrt s, 0) */
    double M = sqrt(Q[0] * Q[0] - Q[1] * Q[1] - Q[2] * Q[2] - Q[3] * Q[3]);
    double b[3] = {-Q[1] / M, -Q[2] / M, -Q[3] / M};
    double x = sqrt_s / M, gam = Q[0] / M, a = 1 / (1 + gam);
    double p0[MAX_PHOTONS + 1], pv[MAX_PHOTONS + 1][3];
    for (int i = 0; i < K; i++) {
        double bq = b[0] * q[i][1] + b[1] * q[i][2] + b[2] * q[i][3];
        p0[i] = x * (gam * q[i][0] + bq);
        for (int l = 0; l < 3; l++) pv[i][l] = x * (q[i][1 + l] + b[l] * q[i][0] + a * bq * b[l]);
    }
    /* mass rescaling: sum_i sqrt(m_i^2 + xi^2 p0_i^2) = sqrt s, electron (i = 0) has m = 1 */
    double xi = sqrt(1 - 1 / s);
    for (int it = 0; it < 50; it++) {
        double f = -sqrt_s, df = 0;
        for (int i = 0; i < K; i++) {
            double m2 = i == 0 ? 1 : 0;
            double e = sqrt(m2 + xi * xi * p0[i] * p0[i]);
            f += e;
            df += xi * p0[i] * p0[i] / e;
        }
        double dxi = f / df;
        xi -= dxi;
        if (fabs(dxi) <= 1e-15 * xi) break;
    }
    double kin = (s - 1) / (2 * sqrt_s);
    mom[0] = (s + 1) / (2 * sqrt_s); mom[1] = 0; mom[2] = 0; mom[3] = -kin;
    mom[4] = kin; mom[5] = 0; mom[6] = 0; mom[7] = kin;
    double prod = 1, sum = 0;
    for (int i = 0; i < K; i++) {
        double m2 = i == 0 ? 1 : 0;
        double kx = xi * pv[i][0], ky = xi * pv[i][1], kz = xi * pv[i][2];
        double E = sqrt(m2 + xi * xi * p0[i] * p0[i]);
        double kk = sqrt(kx * kx + ky * ky + kz * kz);
        double* o = mom + 8 + 4 * i;
        o[0] = E; o[1] = kx; o[2] = ky; o[3] = kz;
        prod *= kk / E;
        sum += kk * kk / E;
    }
    /* massless volume (2pi)^(4-3K) (pi/2)^(K-1) s^(K-2) / ((K-1)! (K-2)!), times the massive factor */
    double vol = pow(2 * M_PI, 4 - 3 * K) * pow(M_PI / 2, K - 1) * pow(s, K - 2);
    for (int i = 2; i <= K - 1; i++) vol /= i;
    for (int i = 2; i <= K - 2; i++) vol /= i;
    return vol * pow(xi, 2 * K - 3) * sqrt_s * prod / sum;
}

typedef struct {
    int n;
    double sqrt_s, omega_min;
    uint64_t seed, first, count;
    int chunk;
    double* partials;    /* [n_chunks][3] local to this job */
    uint64_t c0;         /* first chunk index of this job */
} mc_job_t;

static void* mc_worker(void* arg) {
    mc_job_t* J = (mc_job_t*)arg;
    proc_t P;
    proc_init(&P, 1, J->n);
    int8_t spec[MAX_EXT];
    for (int j = 0; j < P.n_ext; j++) spec[j] = -1;
    double mom[MAX_EXT * 4];
    for (uint64_t i = J->first; i < J->first + J->count; i++) {
        double w = oracle_rambo_point(J->n, J->sqrt_s, J->seed, i, mom);
        int pass = 1;
        for (int k = 1; k <= J->n; k++)
            if (mom[8 + 4 * k] < J->omega_min) pass = 0;
        double m = (double)point_msq(&P, mom, spec);
        double v = pass ? w * m : 0;
        double* c = J->partials + 3 * (i / J->chunk - J->c0);
        c[0] += v;
        c[1] += v * v;
        c[2] += pass;
    }
    return NULL;
}

/* partials[3 * c + {0,1,2}] += (sum w|M|^2, sum (w|M|^2)^2, n_pass) for chunk c = index / chunk,
   indices first .. first + count - 1; partials must hold ceil((first + count) / chunk) chunks.
   Work is split over threads by whole chunks (each chunk summed in index order). */
int oracle_mc_sum(int n_out_ph, double sqrt_s, double omega_min, uint64_t seed, uint64_t first, uint64_t count,
                  int chunk, double* partials, int n_threads) {
    if (n_out_ph < 1 || n_out_ph + 1 > MAX_PHOTONS || chunk < 1 || !(sqrt_s > 1)) return -1;
    if (count == 0) return 0;
    uint64_t c0 = first / chunk, c1 = (first + count + chunk - 1) / chunk;
    uint64_t nch = c1 - c0;
    if (n_threads < 1) n_threads = 1;
    if ((uint64_t)n_threads > nch) n_threads = (int)nch;
    if (n_threads > 256) n_threads = 256;
    pthread_t th[256];
    mc_job_t jobs[256];
    for (int t = 0; t < n_threads; t++) {
        uint64_t ca = c0 + nch * t / n_threads, cb = c0 + nch * (t + 1) / n_threads;
        uint64_t lo = ca * chunk > first ? ca * chunk : first;
        uint64_t hi = cb * chunk < first + count ? cb * chunk : first + count;
        jobs[t] = (mc_job_t){n_out_ph, sqrt_s, omega_min, seed, lo, hi > lo ? hi - lo : 0, chunk,
                             partials + 3 * ca, ca};
        if (t > 0) pthread_create(&th[t], NULL, mc_worker, &jobs[t]);
    }
    mc_worker(&jobs[0]);
    for (int t = 1; t < n_threads; t++) pthread_join(th[t], NULL);
    return 0;
}
