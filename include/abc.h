/*
 * abc.h -- C ABI of the ABC-model |M|^2 kernels in libqed (sm_100a, FP64).
 *
 * What is computed (§1.3 line 56 and App. F):
 *   The ABC model has three scalar particles A, B, C and one vertex joining one of each.  For
 *   A + n_in B -> A + n_out B (N = n_in + n_out B-ons, N even) every tree diagram is one line from
 *   the incoming to the outgoing A with the B-ons attached in some order, the line a C-on after an
 *   odd and an A-on after an even number of attachments:
 *     |M|^2 = g^(2N) | sum over the N! orderings pi of prod_{l=1}^{N-1} 1/(Q_l^2 - m_{X_l}^2) |^2,
 *     Q_l = p_A + sum_{k<=l} q_pi(k),  q = +k (incoming B), -k (outgoing B),  X_l = C (l odd), A (l even),
 *   common factors i (propagators) and -i (vertices) dropped.  No spins: one value per point.
 *   Masses and coupling are the constants below (reading A2; the paper gives none).
 * Same structure as QED Compton scattering, scalar kernels: the paper's kernel-weight comparison
 * (PAPER.md line 530).  The same node-reduced CDAG (or the Berends-Giele rewrite) is emitted as
 * straight-line per-point code (paper_2511_19456_b200/gen/abc.py).
 *
 * Conventions: those of qed.h (SoA momenta in units of m_A, particle order A_in, B_in..., A_out,
 * B_out..., device pointers, asynchronous on `stream`, qed_status codes, qed_last_error(), device
 * binding).  The outgoing A-on's momentum is not read.
 */
#ifndef ABC_H
#define ABC_H

#include <stdint.h>

#include "qed.h"

#ifdef __cplusplus
extern "C" {
#endif

#define ABC_MASS_A 1.0
#define ABC_MASS_B 0.5
#define ABC_MASS_C 1.2
#define ABC_COUPLING 1.0

typedef struct abc_process abc_process; /* opaque, owned by libqed */

/* Handle for A + n_in B -> A + n_out B.  N = n_in + n_out must be even (tree diagrams exist only
   then).  algorithm: QED_ALGO_CDAG (the paper's node-reduced diagram DAG;
   N = 2, 4, 6) or QED_ALGO_BERENDS_GIELE (N = 2, 4, 6).  Other N: QED_ERR_UNSUPPORTED;
   odd N or negative counts: QED_ERR_INVALID_ARGUMENT. */
qed_status abc_process_create(int n_in, int n_out, int algorithm, abc_process** proc);
qed_status abc_process_destroy(abc_process* proc);

/* |M|^2 per point.  momenta: device SoA, 4 * (N + 2) * n_points doubles; out: device, n_points. */
qed_status abc_eval_msq(const abc_process* proc, const double* momenta, int64_t n_points, double* out,
                        void* stream);

typedef struct {
  int n_b;                   /* N */
  int n_diagrams;            /* N! */
  int algorithm;
  int grid_blocks;
  int threads_per_block;
  int64_t flops_per_point;   /* algorithmic FP64 flops (FMA = 2, add / mul / div = 1) */
  int64_t bytes_per_point;   /* algorithmic HBM bytes: A_in and the N B-ons in, |M|^2 out */
} abc_process_info;
qed_status abc_get_process_info(const abc_process* proc, abc_process_info* info);

#ifdef __cplusplus
}
#endif
#endif /* ABC_H */
