/*
 * qed.h -- C ABI of libqed: batched tree-level QED |M|^2 for n-photon Compton
 * scattering on NVIDIA B200 (sm_100a), FP64.
 *
 * What is computed (§1.4 lines 62-68, §3.1):
 *   |M|^2 = e^(2N) | sum over the (n+1)! orderings pi of the N = n+1 photons of
 *            ubar(p',s') epsslash_pi(N) S(Q_N-1) ... S(Q_1) epsslash_pi(1) u(p,s) |^2
 *   summed over the final and averaged over the initial spin/polarisation states
 *   that the process spec leaves free.  S(Q) = (Qslash + m)/(Q^2 - m^2), one factor
 *   e = sqrt(4 pi alpha) per vertex, alpha = 1/137.035999084, m_e = 1.  Linear photon
 *   polarisation basis and z-axis electron spin basis of DESIGN.md "Readings".
 * How: the paper's CDAG of all Feynman diagrams reduced to its node-reduction
 *   fixpoint (App. C) and lowered at build time to one CUDA
 *   kernel per photon count (paper_2511_19456_b200/gen/).
 *
 * Conventions shared by every entry point
 *   - Particle order: e-_in, gamma_in..., e-_out, gamma_out...  (n_ext = n + 3).
 *   - Momenta: FP64, units of m_e, (E, px, py, pz), structure-of-arrays
 *       momenta[(4*j + mu) * n_points + i]   (particle j, component mu, point i).
 *     They must be on shell and conserve 4-momentum; this is NOT checked (garbage in,
 *     garbage out).  Collinear/soft configurations with Q^2 = m^2 give inf/nan.
 *   - Pointers marked "device" must be CUDA device (or managed) memory, 8-byte aligned.
 *   - All calls that take a stream only ENQUEUE work on that stream (asynchronous);
 *     the caller owns every buffer and must keep it alive until the stream has run.
 *     libqed allocates no device memory per call.
 *   - Errors: every function returns a qed_status; qed_last_error() gives a
 *     thread-local message for the last non-OK status.  No exceptions cross the ABI.
 *     A handle is immutable after creation and may be used from several streams/threads.
 *   - Device binding: a handle belongs to the device that was current when it was
 *     created.  Every entry point that launches work checks the calling thread's current
 *     device against it and returns QED_ERR_INVALID_ARGUMENT on a mismatch (it never
 *     switches devices itself).
 */
#ifndef QED_H
#define QED_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  QED_OK = 0,
  QED_ERR_INVALID_ARGUMENT = 1, /* NULL handle/pointer, negative size, malformed spec */
  QED_ERR_UNSUPPORTED = 2,      /* photon count outside 1 <= n <= 5 (CDAG) / 1 <= n <= 8 (Berends-Giele) */
  QED_ERR_CUDA = 3,             /* a CUDA runtime call or kernel launch failed */
  QED_ERR_OUT_OF_MEMORY = 4,
  QED_ERR_INTERNAL = 5
} qed_status;

/* Spin / polarisation state of one external particle: QED_SUM = summed over both
   states (averaged with 1/2 if the particle is initial), 0 / 1 = fixed state:
   electrons 0 = spin up, 1 = spin down along z; photons 0 = eps_1, 1 = eps_2. */
enum { QED_SUM = -1 };

/* One side of the process: the electron plus n_photons photons.
   spins == NULL means every particle of this side is QED_SUM; otherwise
   spins[0] is the electron and spins[1..n_photons] the photons, in particle order. */
typedef struct {
  int n_photons;
  const int8_t* spins;
} qed_state_spec;

typedef struct qed_process qed_process; /* opaque, owned by libqed */

/* Create the handle for e- + in->n_photons gamma -> e- + out->n_photons gamma.
   n_photons is the paper's n: the total photon count minus one, i.e.
   in->n_photons + out->n_photons == n_photons + 1, 1 <= n_photons <= 5 (n <= 8 with
   qed_process_create_ex(..., QED_ALGO_BERENDS_GIELE)).
   North-star process e- gamma -> e- + n gamma: in = {1, ...}, out = {n, ...}.
   Paper process e- gamma^n -> e- gamma: in = {n, ...}, out = {1, ...}.
   No device work; selects the generated kernel for N = n+1 photons on the current device.
   *proc receives the handle (caller frees with qed_process_destroy). */
qed_status qed_process_create(const qed_state_spec* in, const qed_state_spec* out, int n_photons,
                              qed_process** proc);

/* Algorithm selection (extension).  QED_ALGO_CDAG (default) evaluates the paper's node-reduced
   diagram DAG: every one of the (n+1)! diagrams is joined separately (App. C).
   QED_ALGO_BERENDS_GIELE applies the distributive term rewriting the paper names as the route to
   exponential scaling: the sum over the
   orderings of each photon subset is taken inside the propagators (Berends-Giele currents), one join
   per subset.  Same |M|^2 (same oracle), fewer flops: 7.8 k vs 10.7 k (n = 2), 310 k vs 6.2 M (n = 5).
   At n = 1 the rewrite is the identity (one ordering per subset) and both algorithms run the same kernel;
   at n = 2 both run one-thread-per-point register kernels, at n >= 3 lane-group kernels.
   variant: launch-variant index (tuning), -1 = default / QED_VARIANT environment variable; an index
   >= qed_process_info.n_variants, or a QED_VARIANT that is not such an index, is
   QED_ERR_INVALID_ARGUMENT (no silent fallback).  With the default, qed_eval_msq* and qed_mc_sum each run
   their own best launch plan; an explicit variant applies to both (lane-group kernels).
   kernel_family: QED_FAMILY_DEFAULT picks the register kernels at n <= 2 and the lane-group kernels
   above; QED_FAMILY_LANE_GROUP forces the lane-group kernels at n <= 2 too (comparison runs).
   No other environment variable changes what the library does. */
typedef enum { QED_ALGO_CDAG = 0, QED_ALGO_BERENDS_GIELE = 1 } qed_algorithm;
typedef enum { QED_FAMILY_DEFAULT = 0, QED_FAMILY_LANE_GROUP = 1 } qed_kernel_family;
typedef struct {
  int algorithm;
  int variant;
  int kernel_family;
} qed_process_options;
qed_status qed_process_create_ex(const qed_state_spec* in, const qed_state_spec* out, int n_photons,
                                 const qed_process_options* options, qed_process** proc);

/* Free a handle (NULL is a no-op).  Work already enqueued with it is unaffected. */
qed_status qed_process_destroy(qed_process* proc);

/* |M|^2 per point.
   momenta: device, SoA as above, 4 * n_ext * n_points doubles.
   out:     device, n_points doubles (written, not accumulated).
   n_points >= 0 (0 is a no-op).  stream: cudaStream_t (NULL = legacy default stream). */
qed_status qed_eval_msq(const qed_process* proc, const double* momenta, int64_t n_points, double* out,
                        void* stream);

/* Per-configuration |M(h)|^2 = e^(2N) |M(h)|^2 for all 2^(n+3) spin/polarisation
   configurations h (bit j of h = state of external particle j), no averaging.
   out: device, n_points * 2^(n+3) doubles, out[i * 2^(n+3) + h].  (Extension for the
   "explicit helicity configurations" workload, BASELINE.json configs[4].) */
qed_status qed_eval_msq_configs(const qed_process* proc, const double* momenta, int64_t n_points,
                                double* out, void* stream);

/* Same as qed_eval_msq, but momenta and out are HOST buffers (same layouts; pin them with
   cudaHostAlloc / cudaHostRegister for full PCIe bandwidth): copies them through two chunk staging
   buffers owned by the handle, pipelined over chunks of >= 2^18 points on two streams owned by the
   handle (upload of chunk c+1 overlaps kernel and download of chunk c), and returns after the result
   is on the host (end-to-end path).  Synchronous; calls on one handle are serialised. */
qed_status qed_eval_msq_host(const qed_process* proc, const double* momenta_host, int64_t n_points,
                             double* out_host);

/* qed_eval_msq_host with upload flags (extension).  flags = 0 is qed_eval_msq_host.
   QED_HOST_ONSHELL: the energy rows momenta[4*j*n_points ...] are NOT read or uploaded.  Only the
   3-momenta cross PCIe (3/4 of the bytes), and a device kernel restores every energy from the
   mass shell the header's conventions already require, E_j = sqrt(|p_j|^2 + m_j^2) with m = m_e = 1
   for the electrons and 0 for the photons (§1.4 line 62: on-shell external states), before
   the |M|^2 kernel runs on the chunk.  Results then differ from flags = 0 by the rounding of the
   given energies (relative ~1e-15 for RAMBO inputs, up to ~1e-11 where propagator denominators cancel).
   QED_HOST_CONSERVE (only together with QED_HOST_ONSHELL): the outgoing electron's rows are not read or
   uploaded either; the device restores its 3-momentum from the 4-momentum conservation the header's
   conventions require, p' = p + sum(incoming k) - sum(outgoing k), then its energy from the shell
   (4/5 of the ONSHELL bytes at n = 2).  Unknown flag bits, or CONSERVE without ONSHELL:
   QED_ERR_INVALID_ARGUMENT. */
#define QED_HOST_ONSHELL 1u
#define QED_HOST_CONSERVE 2u
qed_status qed_eval_msq_host_ex(const qed_process* proc, const double* momenta_host, int64_t n_points,
                                double* out_host, uint32_t flags);

/* Monte-Carlo cross-section partial sums.
   Generates points first_index .. first_index + n_points - 1 of the phase-space
   sequence keyed by seed (Philox4x32-10, counter = global point index, so the
   sequence does not depend on how points are split over GPUs) with massive RAMBO
   in the CM frame at sqrt_s (incoming photon along +z, electron along -z), weights
   each point by the RAMBO weight times the cut (every outgoing photon with
   E >= omega_min, else weight 0), evaluates |M|^2 and accumulates per chunk of
   QED_MC_CHUNK consecutive global indices:
     partials[3*c + 0] += sum w |M|^2, partials[3*c + 1] += sum (w |M|^2)^2,
     partials[3*c + 2] += number of points passing the cut,
   for chunk c = global_index / QED_MC_CHUNK.  partials: device, 3 * n_chunks doubles with
   n_chunks >= ceil((first_index + n_points) / QED_MC_CHUNK); the caller zeroes it and
   all-reduces it across ranks (the only collective), then sums the
   chunks in index order -- bitwise identical for any split of the index range along
   chunk boundaries.  Only the north-star direction (in = 1 photon) is supported.
   QED_MC_CHUNK is small enough that a 2^24-point call has >= 10 chunks per resident block
   (load balance of the chunk-per-block kernel). */
#define QED_MC_CHUNK 1024
typedef struct {
  double sqrt_s;
  double omega_min;
  uint64_t seed;
  uint64_t first_index;
  uint64_t n_points;
} qed_mc_config;
qed_status qed_mc_sum(const qed_process* proc, const qed_mc_config* cfg, double* partials, void* stream);

/* Introspection (host only). */
typedef struct {
  int n_photons;             /* n */
  int n_ext;                 /* n + 3 */
  int n_configs;             /* 2^(n+3) */
  int n_diagrams;            /* (n+1)! */
  int lanes_per_point;       /* G */
  int warps_per_block;
  int64_t smem_per_block;    /* bytes */
  int grid_blocks;           /* persistent grid size used for large batches */
  int64_t flops_per_point;   /* algorithmic FP64 flops per point (FMA = 2) */
  int64_t bytes_per_point;   /* algorithmic HBM bytes per point (momenta in + |M|^2 out) */
  int algorithm;             /* qed_algorithm */
  int variant;               /* launch variant in use */
  int n_variants;            /* launch variants compiled for this size and algorithm (0 .. n_variants-1) */
} qed_process_info;
qed_status qed_get_process_info(const qed_process* proc, qed_process_info* info);

const char* qed_last_error(void);

/* Number of eval-kernel launches issued through this library since load (for the
   bench's gpu_launches claim). */
int64_t qed_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* QED_H */
