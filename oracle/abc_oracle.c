/*
 * abc_oracle.c -- the PARITY ORACLE for tree-level |M|^2 in the ABC model.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2511_19456_b200/, libqed.so) never links, imports or calls anything under
 * oracle/, and this file shares no code, header, table or constant with it.
 *
 * What it computes (§1.3 line 56 and App. F; readings A1-A5):
 *   The ABC model has three scalar particles A, B, C and one vertex joining one of each
 *   (coupling g).  None is its own antiparticle, so in A + n_in B -> A + n_out B every tree
 *   diagram is one line from the incoming to the outgoing A with the N = n_in + n_out B-ons
 *   attached in some order, the line alternating A / C at every attachment (App. F):
 *   after l attachments it is a C-on for odd l and an A-on for even l (N must be even).
 *
 *   M = g^N * sum over all N! orderings pi of the B-ons of
 *         prod_{l=1}^{N-1} 1 / (Q_l^2 - m_{X_l}^2),   X_l = C (l odd), A (l even),
 *       Q_l = p_A + sum_{k<=l} q_{pi(k)},   q = +k (incoming B), -k (outgoing B),
 *   the factors i of the propagators and -i of the vertices dropped (common to every diagram),
 *   |M|^2 = |M|^2 (no spins).  Masses and g are arguments.
 *
 * Evaluation is deliberately naive: every diagram enumerated (next_permutation), every
 * denominator recomputed inside its diagram.  Parity pins: tests/test_abc_oracle.py.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <string.h>

#define ABC_MAX_B 10

static int abc_next_perm(int* a, int n) {
    int i = n - 2;
    while (i >= 0 && a[i] >= a[i + 1]) i--;
    if (i < 0) return 0;
    int j = n - 1;
    while (a[j] <= a[i]) j--;
    int t = a[i]; a[i] = a[j]; a[j] = t;
    for (int l = i + 1, r = n - 1; l < r; l++, r--) { t = a[l]; a[l] = a[r]; a[r] = t; }
    return 1;
}

/* sum over all N! orderings of prod_{l=1}^{N-1} 1/(Q_l^2 - m_{X_l}^2); returns the diagram count */
static long abc_diagram_sum(int N, const double q[][4], const double pA[4], double mA, double mC, double* amp) {
    int perm[ABC_MAX_B];
    for (int i = 0; i < N; i++) perm[i] = i;
    long nd = 0;
    double total = 0;
    do {
        double Q[4] = {pA[0], pA[1], pA[2], pA[3]};
        double term = 1;
        for (int l = 1; l <= N - 1; l++) {
            for (int mu = 0; mu < 4; mu++) Q[mu] += q[perm[l - 1]][mu];
            double m = (l % 2 == 1) ? mC : mA;
            double Q2 = Q[0] * Q[0] - Q[1] * Q[1] - Q[2] * Q[2] - Q[3] * Q[3];
            term /= Q2 - m * m;
        }
        total += term;
        nd++;
    } while (abc_next_perm(perm, N));
    *amp = total;
    return nd;
}

/* Particle order: A_in, B_in..., A_out, B_out...; mom[(point * n_ext + j) * 4 + mu]. */
typedef struct {
    int n_in, n_out, N, n_ext;
    double mA, mC, g;
    const double* mom;
    double* out;
    long begin, end;
} abc_job;

static double abc_point(const abc_job* J, const double* m) {
    double pA[4], q[ABC_MAX_B][4];
    for (int mu = 0; mu < 4; mu++) pA[mu] = m[mu];
    for (int i = 0; i < J->N; i++) {
        int j = i < J->n_in ? 1 + i : J->n_in + 2 + (i - J->n_in);     /* particle index of B-on i */
        for (int mu = 0; mu < 4; mu++) q[i][mu] = (i < J->n_in ? 1.0 : -1.0) * m[j * 4 + mu];
    }
    double a;
    abc_diagram_sum(J->N, (const double(*)[4])q, pA, J->mA, J->mC, &a);
    double gn = 1;
    for (int i = 0; i < J->N; i++) gn *= J->g;
    return (gn * a) * (gn * a);
}

static void* abc_worker(void* arg) {
    abc_job* J = (abc_job*)arg;
    for (long i = J->begin; i < J->end; i++) J->out[i] = abc_point(J, J->mom + i * J->n_ext * 4);
    return NULL;
}

/* |M|^2 per point of A + n_in B -> A + n_out B.  Returns 0, or -1 on bad arguments
   (N = n_in + n_out must be even and 2 <= N <= ABC_MAX_B). */
int oracle_abc_msq(int n_in, int n_out, double mA, double mC, double g, const double* mom, long n_points,
                   double* out, int n_threads) {
    int N = n_in + n_out;
    if (n_in < 0 || n_out < 0 || N < 2 || N > ABC_MAX_B || N % 2) return -1;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    if (n_points < n_threads) n_threads = n_points > 0 ? (int)n_points : 1;
    pthread_t th[256];
    abc_job jobs[256];
    for (int t = 0; t < n_threads; t++) {
        jobs[t] = (abc_job){n_in, n_out, N, N + 2, mA, mC, g, mom, out, n_points * t / n_threads,
                            n_points * (t + 1) / n_threads};
        if (t > 0) pthread_create(&th[t], NULL, abc_worker, &jobs[t]);
    }
    abc_worker(&jobs[0]);
    for (int t = 1; t < n_threads; t++) pthread_join(th[t], NULL);
    return 0;
}

/* Diagram sum for explicit signed B momenta q[N][4] (no coupling): for the count / closed-form pins. */
long oracle_abc_diagram_sum(int N, const double* q, const double* pA, double mA, double mC, double* amp) {
    if (N < 1 || N > ABC_MAX_B) return -1;
    return abc_diagram_sum(N, (const double(*)[4])q, pA, mA, mC, amp);
}
