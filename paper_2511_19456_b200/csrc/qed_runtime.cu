// qed_runtime.cu -- libqed C-ABI (include/qed.h): handles, argument validation,
// launch configuration and error reporting around the generated kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "qed.h"
#include "qed_kernel_args.h"
#include "qed_mc_args.h"

extern "C" {
const void* qedgen_kernel_N2(int, int);
const void* qedgen_kernel_N3(int, int);
const void* qedgen_kernel_N4(int, int);
const void* qedgen_kernel_N5(int, int);
const void* qedgen_kernel_N6(int, int);
const void* qedgen_mc_kernel_N2(int);
int qedgen_num_variants_N2(void);
int qedgen_mc_variant_N2(void);
const void* qedgen_mc_kernel_N3(int);
int qedgen_num_variants_N3(void);
int qedgen_mc_variant_N3(void);
const void* qedgen_mc_kernel_N4(int);
int qedgen_num_variants_N4(void);
int qedgen_mc_variant_N4(void);
const void* qedgen_mc_kernel_N5(int);
int qedgen_num_variants_N5(void);
int qedgen_mc_variant_N5(void);
const void* qedgen_mc_kernel_N6(int);
int qedgen_num_variants_N6(void);
int qedgen_mc_variant_N6(void);
void qedgen_config_N2(int, int*, int*, long long*, long long*);
void qedgen_config_N3(int, int*, int*, long long*, long long*);
void qedgen_config_N4(int, int*, int*, long long*, long long*);
void qedgen_config_N5(int, int*, int*, long long*, long long*);
void qedgen_config_N6(int, int*, int*, long long*, long long*);
const void* qedbg_kernel_N2(int, int);
const void* qedbg_mc_kernel_N2(int);
int qedbg_num_variants_N2(void);
int qedbg_mc_variant_N2(void);
void qedbg_config_N2(int, int*, int*, long long*, long long*);
const void* qedbg_kernel_N3(int, int);
const void* qedbg_mc_kernel_N3(int);
int qedbg_num_variants_N3(void);
int qedbg_mc_variant_N3(void);
void qedbg_config_N3(int, int*, int*, long long*, long long*);
const void* qedbg_kernel_N4(int, int);
const void* qedbg_mc_kernel_N4(int);
int qedbg_num_variants_N4(void);
int qedbg_mc_variant_N4(void);
void qedbg_config_N4(int, int*, int*, long long*, long long*);
const void* qedbg_kernel_N5(int, int);
const void* qedbg_mc_kernel_N5(int);
int qedbg_num_variants_N5(void);
int qedbg_mc_variant_N5(void);
void qedbg_config_N5(int, int*, int*, long long*, long long*);
const void* qedbg_kernel_N6(int, int);
const void* qedbg_mc_kernel_N6(int);
int qedbg_num_variants_N6(void);
int qedbg_mc_variant_N6(void);
void qedbg_config_N6(int, int*, int*, long long*, long long*);
const void* qedbg_kernel_N7(int, int);
const void* qedbg_mc_kernel_N7(int);
int qedbg_num_variants_N7(void);
int qedbg_mc_variant_N7(void);
void qedbg_config_N7(int, int*, int*, long long*, long long*);
const void* qedbg_kernel_N8(int, int);
const void* qedbg_mc_kernel_N8(int);
int qedbg_num_variants_N8(void);
int qedbg_mc_variant_N8(void);
void qedbg_config_N8(int, int*, int*, long long*, long long*);
const void* qedbg_kernel_N9(int, int);
const void* qedbg_mc_kernel_N9(int);
int qedbg_num_variants_N9(void);
int qedbg_mc_variant_N9(void);
void qedbg_config_N9(int, int*, int*, long long*, long long*);
const void* qedregs_kernel_N2(int, int);
int qedregs_num_variants_N2(void);
const void* qedregs_kernel_N3(int, int);
int qedregs_num_variants_N3(void);
void qedregs_config_N2(int, int*, int*, long long*, long long*);
void qedregs_config_N3(int, int*, int*, long long*, long long*);
const void* qedregsbg_kernel_N3(int, int);
int qedregsbg_num_variants_N3(void);
void qedregsbg_config_N3(int, int*, int*, long long*, long long*);
}

namespace {

thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};

qed_status fail(qed_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

qed_status cuda_fail(cudaError_t e, const char* what) {
  return fail(QED_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct KernelEntry {
  const void* (*kernel)(int, int);
  const void* (*mc_kernel)(int);
  void (*config)(int, int*, int*, long long*, long long*);
  int (*num_variants)(void);
  int (*mc_variant)(void);   // launch variant of the fused MC kernel (nullptr: 0)
};

const KernelEntry kKernels[] = {
    {qedgen_kernel_N2, qedgen_mc_kernel_N2, qedgen_config_N2, qedgen_num_variants_N2, qedgen_mc_variant_N2},
    {qedgen_kernel_N3, qedgen_mc_kernel_N3, qedgen_config_N3, qedgen_num_variants_N3, qedgen_mc_variant_N3},
    {qedgen_kernel_N4, qedgen_mc_kernel_N4, qedgen_config_N4, qedgen_num_variants_N4, qedgen_mc_variant_N4},
    {qedgen_kernel_N5, qedgen_mc_kernel_N5, qedgen_config_N5, qedgen_num_variants_N5, qedgen_mc_variant_N5},
    {qedgen_kernel_N6, qedgen_mc_kernel_N6, qedgen_config_N6, qedgen_num_variants_N6, qedgen_mc_variant_N6},
};

const KernelEntry kBGKernels[] = {
    {qedbg_kernel_N2, qedbg_mc_kernel_N2, qedbg_config_N2, qedbg_num_variants_N2, qedbg_mc_variant_N2},
    {qedbg_kernel_N3, qedbg_mc_kernel_N3, qedbg_config_N3, qedbg_num_variants_N3, qedbg_mc_variant_N3},
    {qedbg_kernel_N4, qedbg_mc_kernel_N4, qedbg_config_N4, qedbg_num_variants_N4, qedbg_mc_variant_N4},
    {qedbg_kernel_N5, qedbg_mc_kernel_N5, qedbg_config_N5, qedbg_num_variants_N5, qedbg_mc_variant_N5},
    {qedbg_kernel_N6, qedbg_mc_kernel_N6, qedbg_config_N6, qedbg_num_variants_N6, qedbg_mc_variant_N6},
    {qedbg_kernel_N7, qedbg_mc_kernel_N7, qedbg_config_N7, qedbg_num_variants_N7, qedbg_mc_variant_N7},
    {qedbg_kernel_N8, qedbg_mc_kernel_N8, qedbg_config_N8, qedbg_num_variants_N8, qedbg_mc_variant_N8},
    {qedbg_kernel_N9, qedbg_mc_kernel_N9, qedbg_config_N9, qedbg_num_variants_N9, qedbg_mc_variant_N9},
};

// launch variant from QED_VARIANT (tuning experiments); unset = 0 (default); anything that is not an
// index in [0, n_variants) is an error (-1), never a silent fallback.
int variant_from_env(int n_variants) {
  const char* v = getenv("QED_VARIANT");
  if (!v || !*v) return 0;
  char* end = nullptr;
  long x = strtol(v, &end, 10);
  return (end && *end == '\0' && x >= 0 && x < n_variants) ? (int)x : -1;
}

// every entry point runs on the device the handle was created on (include/qed.h "Device binding")
qed_status check_device(int device) {
  int cur = -1;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (cur != device)
    return fail(QED_ERR_INVALID_ARGUMENT, "current device " + std::to_string(cur) + " differs from the handle's device " +
                                              std::to_string(device));
  return QED_OK;
}

}  // namespace

constexpr long long kHostChunkMin = 1LL << 18;   // points per pipelined chunk of qed_eval_msq_host (minimum)

// QED_HOST_ONSHELL / QED_HOST_CONSERVE (include/qed.h): complete one uploaded chunk.  One thread per point
// (consecutive threads on consecutive points: coalesced 8-byte rows).  CONSERVE: the outgoing electron's
// 3-momentum p' = p + sum_in k - sum_out k (rows of particle e_out were not uploaded); then every energy row
// E_j = sqrt(|p_j|^2 + m_j^2), m = 1 for the two electrons, 0 for the photons.
__global__ void __launch_bounds__(256) qed_onshell_energy_kernel(double* __restrict__ mom, long long cnt, int n_ext,
                                                                 int e_out, int conserve) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (long long)gridDim.x * blockDim.x) {
    double* r = mom + i;
    if (conserve) {
      double px = 0.0, py = 0.0, pz = 0.0;
      for (int j = 0; j < n_ext; ++j) {
        if (j == e_out) continue;
        const double sg = j < e_out ? 1.0 : -1.0;   // incoming: e- and photons before e_out
        px = fma(sg, r[(4 * j + 1) * cnt], px);
        py = fma(sg, r[(4 * j + 2) * cnt], py);
        pz = fma(sg, r[(4 * j + 3) * cnt], pz);
      }
      r[(4 * e_out + 1) * cnt] = px;
      r[(4 * e_out + 2) * cnt] = py;
      r[(4 * e_out + 3) * cnt] = pz;
    }
    for (int j = 0; j < n_ext; ++j) {
      const double px = r[(4 * j + 1) * cnt], py = r[(4 * j + 2) * cnt], pz = r[(4 * j + 3) * cnt];
      const double m2 = (j == 0 || j == e_out) ? 1.0 : 0.0;
      r[4 * j * cnt] = sqrt(fma(px, px, fma(py, py, fma(pz, pz, m2))));
    }
  }
}

struct qed_process {
  int n = 0, N = 0, n_in_ph = 0, n_out_ph = 0, n_ext = 0;
  qed::QedEvalArgs args{};
  const void* kern[2] = {nullptr, nullptr};
  const void* kern_mc = nullptr;
  int variant = 0, n_variants = 1, algorithm = 0;
  int wpb = 0, ppw = 0, grid_blocks = 0, mc_wpb = 0, mc_grid_blocks = 0, device = 0, num_sms = 0;
  long long smem = 0, smem_mc = 0, flops = 0;
  // staging for the host-buffer entry point
  std::mutex mu;
  // host entry point: two chunk staging buffers (momenta SoA of kHostChunk points, out), one stream each
  double* d_mom[2] = {nullptr, nullptr};
  double* d_out[2] = {nullptr, nullptr};
  long long cap = 0;
  cudaStream_t hstream[2] = {nullptr, nullptr};
};

extern "C" {

// shared with abc_runtime.cu (same library, same error slot and launch counter)
qed_status qed_internal_fail(qed_status st, const char* msg) { return fail(st, msg); }
void qed_internal_count_launch(void) { g_launches.fetch_add(1); }

const char* qed_last_error(void) { return g_last_error.c_str(); }

int64_t qed_launch_count(void) { return g_launches.load(); }

static qed_status check_spec(const qed_state_spec* s, const char* side) {
  if (!s) return fail(QED_ERR_INVALID_ARGUMENT, std::string(side) + " spec is NULL");
  if (s->n_photons < 0) return fail(QED_ERR_INVALID_ARGUMENT, std::string(side) + ".n_photons < 0");
  if (s->spins)
    for (int i = 0; i <= s->n_photons; ++i)
      if (s->spins[i] < -1 || s->spins[i] > 1)
        return fail(QED_ERR_INVALID_ARGUMENT, std::string(side) + ".spins entries must be -1, 0 or 1");
  return QED_OK;
}

qed_status qed_process_create(const qed_state_spec* in, const qed_state_spec* out, int n_photons,
                              qed_process** proc) {
  return qed_process_create_ex(in, out, n_photons, nullptr, proc);
}

qed_status qed_process_create_ex(const qed_state_spec* in, const qed_state_spec* out, int n_photons,
                                 const qed_process_options* options, qed_process** proc) {
  if (!proc) return fail(QED_ERR_INVALID_ARGUMENT, "proc is NULL");
  *proc = nullptr;
  qed_status st;
  if ((st = check_spec(in, "in")) != QED_OK) return st;
  if ((st = check_spec(out, "out")) != QED_OK) return st;
  const int N = in->n_photons + out->n_photons;
  if (N != n_photons + 1)
    return fail(QED_ERR_INVALID_ARGUMENT, "in.n_photons + out.n_photons must equal n_photons + 1");
  const int algorithm = options ? options->algorithm : QED_ALGO_CDAG;
  if (options && options->kernel_family != QED_FAMILY_DEFAULT && options->kernel_family != QED_FAMILY_LANE_GROUP)
    return fail(QED_ERR_INVALID_ARGUMENT, "unknown kernel_family");
  if (algorithm != QED_ALGO_CDAG && algorithm != QED_ALGO_BERENDS_GIELE)
    return fail(QED_ERR_INVALID_ARGUMENT, "unknown algorithm");
  const int n_max = algorithm == QED_ALGO_BERENDS_GIELE ? 8 : 5;
  if (n_photons < 1 || n_photons > n_max)
    return fail(QED_ERR_UNSUPPORTED, algorithm == QED_ALGO_BERENDS_GIELE
                                         ? "supported photon counts with QED_ALGO_BERENDS_GIELE: 1 <= n <= 8"
                                         : "supported photon counts with QED_ALGO_CDAG: 1 <= n <= 5 (n = 6..8: use "
                                           "QED_ALGO_BERENDS_GIELE)");

  qed_process* P = new (std::nothrow) qed_process;
  if (!P) return fail(QED_ERR_OUT_OF_MEMORY, "host allocation failed");
  P->n = n_photons;
  P->N = N;
  P->n_in_ph = in->n_photons;
  P->n_out_ph = out->n_photons;
  P->n_ext = N + 2;

  // particle indices: e-_in = 0, photons in 1..n_in, e-_out = n_in + 1, photons out after it
  const int e_out = P->n_in_ph + 1;
  auto photon_particle = [&](int i) { return i < P->n_in_ph ? 1 + i : P->n_in_ph + 2 + (i - P->n_in_ph); };
  auto spin_of = [&](int particle) -> int {
    if (particle <= P->n_in_ph) return in->spins ? in->spins[particle] : -1;
    int k = particle - e_out;
    return out->spins ? out->spins[k] : -1;
  };
  qed::QedEvalArgs& a = P->args;
  a.n_in_ph = P->n_in_ph;
  a.e_out_particle = e_out;
  a.photon_particle = 0;
  for (int i = 0; i < N; ++i) a.photon_particle |= (unsigned long long)photon_particle(i) << (4 * i);
  // internal configuration bits: 0 = e-_in spin, 1 + i = photon i, N + 1 = e-_out spin
  int ext_of_bit[12];
  ext_of_bit[0] = 0;
  for (int i = 0; i < N; ++i) ext_of_bit[1 + i] = photon_particle(i);
  ext_of_bit[N + 1] = e_out;
  a.ext_bit = 0;
  a.fixed_mask = a.fixed_val = 0;
  for (int b = 0; b < N + 2; ++b) {
    a.ext_bit |= (unsigned long long)ext_of_bit[b] << (4 * b);
    int sp = spin_of(ext_of_bit[b]);
    if (sp >= 0) {
      a.fixed_mask |= 1u << b;
      a.fixed_val |= (unsigned)sp << b;
    }
  }
  // e^(2N) and 1/2 per summed initial particle (averaging)
  const double alpha = 1.0 / 137.035999084;
  double norm = std::pow(4.0 * M_PI * alpha, N);
  a.coupling = norm;
  for (int j = 0; j <= P->n_in_ph; ++j)
    if (spin_of(j) < 0) norm *= 0.5;
  a.norm = norm;

  P->algorithm = algorithm;
  const KernelEntry& ke = algorithm == QED_ALGO_BERENDS_GIELE ? kBGKernels[N - 2] : kKernels[N - 2];
  // n = 1, 2: register-resident straight-line kernels (qed_eval_regs.cuh); n >= 3: lane-group
  // kernels with shared-memory trie staging (qed_eval_kernel.cuh).  QED_KERNEL=group forces the latter.
  // At n = 1 the Berends-Giele rewrite is the identity (every photon subset of one side has a single
  // ordering: J_in({a}) = S(Q_a) epsslash_a u, K_out({b}) = ubar epsslash_b), so it runs the same kernel.
  // At n = 2 the Berends-Giele currents have their own register body (qedregsbg_*).
  const bool use_regs = N <= 3 && !(options && options->kernel_family == QED_FAMILY_LANE_GROUP);
  const bool bg_regs = algorithm == QED_ALGO_BERENDS_GIELE && N == 3;
  if (use_regs) {
    const int nv = bg_regs ? qedregsbg_num_variants_N3() : N == 2 ? qedregs_num_variants_N2() : qedregs_num_variants_N3();
    if (options && options->variant >= nv) {
      delete P;
      return fail(QED_ERR_INVALID_ARGUMENT, "options.variant " + std::to_string(options->variant) + " >= " + std::to_string(nv));
    }
    const int v = (options && options->variant >= 0) ? options->variant : variant_from_env(nv);
    if (v < 0) {
      delete P;
      return fail(QED_ERR_INVALID_ARGUMENT, "QED_VARIANT must be an integer in [0, " + std::to_string(nv) + ")");
    }
    P->variant = v;
    P->n_variants = nv;
    P->kern[0] = bg_regs ? qedregsbg_kernel_N3(0, v) : N == 2 ? qedregs_kernel_N2(0, v) : qedregs_kernel_N3(0, v);
    P->kern[1] = bg_regs ? qedregsbg_kernel_N3(1, v) : N == 2 ? qedregs_kernel_N2(1, v) : qedregs_kernel_N3(1, v);
    (bg_regs ? qedregsbg_config_N3 : N == 2 ? qedregs_config_N2 : qedregs_config_N3)(v, &P->wpb, &P->ppw, &P->smem, &P->flops);
  } else {
    const int nv = ke.num_variants();
    if (options && options->variant >= nv) {
      delete P;
      return fail(QED_ERR_INVALID_ARGUMENT, "options.variant " + std::to_string(options->variant) + " >= " + std::to_string(nv));
    }
    const int v = (options && options->variant >= 0) ? options->variant : variant_from_env(nv);
    if (v < 0) {
      delete P;
      return fail(QED_ERR_INVALID_ARGUMENT, "QED_VARIANT must be an integer in [0, " + std::to_string(nv) + ")");
    }
    P->variant = v;
    P->n_variants = nv;
    P->kern[0] = ke.kernel(0, v);
    P->kern[1] = ke.kernel(1, v);
    ke.config(v, &P->wpb, &P->ppw, &P->smem, &P->flops);
  }
  int mc_wpb = 0, mc_ppw = 0;
  long long mc_smem = 0, mc_flops = 0;
  // the fused MC kernel: its own default launch variant, or the requested one for the lane-group kernels
  const char* env_v = getenv("QED_VARIANT");
  const bool explicit_v = !use_regs && ((options && options->variant >= 0) || (env_v && *env_v));
  const int mcv = explicit_v ? P->variant : (ke.mc_variant ? ke.mc_variant() : 0);
  ke.config(mcv, &mc_wpb, &mc_ppw, &mc_smem, &mc_flops);

  cudaError_t e = cudaGetDevice(&P->device);
  if (e != cudaSuccess) { delete P; return cuda_fail(e, "cudaGetDevice"); }
  e = cudaDeviceGetAttribute(&P->num_sms, cudaDevAttrMultiProcessorCount, P->device);
  if (e != cudaSuccess) { delete P; return cuda_fail(e, "cudaDeviceGetAttribute"); }
  int blocks_per_sm = 1 << 30;
  for (int v = 0; v < 2; ++v) {
    e = cudaFuncSetAttribute(P->kern[v], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smem);
    if (e != cudaSuccess) { delete P; return cuda_fail(e, "cudaFuncSetAttribute"); }
    int b = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, P->kern[v], P->wpb * 32, (size_t)P->smem);
    if (e != cudaSuccess) { delete P; return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor"); }
    blocks_per_sm = std::min(blocks_per_sm, std::max(b, 1));
  }
  P->grid_blocks = blocks_per_sm * P->num_sms;
  // fused MC kernel: same per-point layout plus WPB x 3 doubles of block reduction space
  P->kern_mc = ke.mc_kernel(mcv);
  P->mc_wpb = mc_wpb;
  // + the block reduction scratch (3 doubles per point of an eval pass) and the RAMBO staging (qed_mc_kernel.cuh:
  // min(wpb * 32 / SUB, 8 PB) points per round, SUB = 4 / 8 / 16 lanes for N <= 4 / 8 / more, 4 (N + 2) + 2
  // doubles each)
  const int mc_sub = N <= 4 ? 4 : N <= 8 ? 8 : 16, mc_pb = std::max(1, mc_wpb * 32 / (1 << N));
  const int mc_rb = std::min(mc_wpb * 32 / mc_sub, 8 * mc_pb);
  P->smem_mc = mc_smem + 8LL * (3LL * mc_pb + (long long)mc_rb * (4 * (N + 2) + 2));
  e = cudaFuncSetAttribute(P->kern_mc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smem_mc);
  if (e != cudaSuccess) { delete P; return cuda_fail(e, "cudaFuncSetAttribute(mc)"); }
  int bmc = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bmc, P->kern_mc, P->mc_wpb * 32, (size_t)P->smem_mc);
  if (e != cudaSuccess) { delete P; return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor(mc)"); }
  P->mc_grid_blocks = std::max(bmc, 1) * P->num_sms;
  *proc = P;
  return QED_OK;
}

qed_status qed_process_destroy(qed_process* proc) {
  if (!proc) return QED_OK;
  for (int b = 0; b < 2; ++b) {
    if (proc->d_mom[b]) cudaFree(proc->d_mom[b]);
    if (proc->d_out[b]) cudaFree(proc->d_out[b]);
    if (proc->hstream[b]) cudaStreamDestroy(proc->hstream[b]);
  }
  delete proc;
  return QED_OK;
}

static qed_status launch_eval(const qed_process* P, const double* mom, int64_t n_points, double* out,
                              cudaStream_t stream, int per_config) {
  if (!P) return fail(QED_ERR_INVALID_ARGUMENT, "proc is NULL");
  if (n_points < 0) return fail(QED_ERR_INVALID_ARGUMENT, "n_points < 0");
  if (n_points == 0) return QED_OK;
  if (!mom || !out) return fail(QED_ERR_INVALID_ARGUMENT, "momenta/out is NULL");
  qed_status dst = check_device(P->device);
  if (dst != QED_OK) return dst;
  if (((uintptr_t)mom & 7) || ((uintptr_t)out & 7)) return fail(QED_ERR_INVALID_ARGUMENT, "pointers must be 8-byte aligned");
  qed::QedEvalArgs a = P->args;
  a.mom = mom;
  a.out = out;
  a.n_points = n_points;
  const long long per_block = P->ppw > 0 ? (long long)P->wpb * P->ppw : (long long)P->wpb * 32 / (1 << P->N);
  const long long need = (n_points + per_block - 1) / per_block;
  const int grid = (int)std::min<long long>(need, P->grid_blocks);
  void* params[] = {&a};
  cudaError_t e = cudaLaunchKernel(P->kern[per_config], dim3(grid), dim3(P->wpb * 32), params, (size_t)P->smem, stream);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  g_launches.fetch_add(1);
  return QED_OK;
}

qed_status qed_eval_msq(const qed_process* proc, const double* momenta, int64_t n_points, double* out, void* stream) {
  return launch_eval(proc, momenta, n_points, out, (cudaStream_t)stream, 0);
}

qed_status qed_eval_msq_configs(const qed_process* proc, const double* momenta, int64_t n_points, double* out,
                                void* stream) {
  return launch_eval(proc, momenta, n_points, out, (cudaStream_t)stream, 1);
}

qed_status qed_eval_msq_host(const qed_process* cproc, const double* momenta_host, int64_t n_points,
                             double* out_host) {
  return qed_eval_msq_host_ex(cproc, momenta_host, n_points, out_host, 0u);
}

qed_status qed_eval_msq_host_ex(const qed_process* cproc, const double* momenta_host, int64_t n_points,
                                double* out_host, uint32_t flags) {
  qed_process* P = const_cast<qed_process*>(cproc);
  if (!P) return fail(QED_ERR_INVALID_ARGUMENT, "proc is NULL");
  if (flags & ~(QED_HOST_ONSHELL | QED_HOST_CONSERVE))
    return fail(QED_ERR_INVALID_ARGUMENT, "unknown flag bits in qed_eval_msq_host_ex");
  if ((flags & QED_HOST_CONSERVE) && !(flags & QED_HOST_ONSHELL))
    return fail(QED_ERR_INVALID_ARGUMENT, "QED_HOST_CONSERVE requires QED_HOST_ONSHELL");
  const bool onshell = (flags & QED_HOST_ONSHELL) != 0, conserve = (flags & QED_HOST_CONSERVE) != 0;
  const int e_out = P->args.e_out_particle;
  if (n_points < 0) return fail(QED_ERR_INVALID_ARGUMENT, "n_points < 0");
  if (n_points == 0) return QED_OK;
  if (!momenta_host || !out_host) return fail(QED_ERR_INVALID_ARGUMENT, "momenta/out is NULL");
  qed_status dst = check_device(P->device);
  if (dst != QED_OK) return dst;
  std::lock_guard<std::mutex> lock(P->mu);
  cudaError_t e;
  // On any error after the first enqueue, drain both streams before returning, so that no DMA still
  // targets the caller's host buffers when the call returns (the caller may free them).
  auto drain = [&](qed_status st) {
    for (int b = 0; b < 2; ++b)
      if (P->hstream[b]) cudaStreamSynchronize(P->hstream[b]);
    return st;
  };
  int max_pitch = 0;
  if (cudaDeviceGetAttribute(&max_pitch, cudaDevAttrMaxPitch, P->device) != cudaSuccess) max_pitch = 0;
  // Pipelined over chunks of points on two streams: chunk c's H2D (a 2D copy of its columns of the
  // SoA rows), kernel and D2H go to stream c % 2 and its staging buffer, so the upload of chunk c+1
  // overlaps the kernel and download of chunk c.  PCIe bound: ~160 B in per point at n = 2.
  const long long chunk = std::min<long long>(n_points, std::max<long long>(kHostChunkMin, (n_points + 7) / 8));
  for (int b = 0; b < 2; ++b)
    if (!P->hstream[b]) {
      e = cudaStreamCreateWithFlags(&P->hstream[b], cudaStreamNonBlocking);
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
    }
  if (P->cap < chunk) {
    for (int b = 0; b < 2; ++b) {
      if (P->d_mom[b]) cudaFree(P->d_mom[b]);
      if (P->d_out[b]) cudaFree(P->d_out[b]);
      P->d_mom[b] = P->d_out[b] = nullptr;
    }
    P->cap = 0;
    for (int b = 0; b < 2; ++b) {
      e = cudaMalloc(&P->d_mom[b], sizeof(double) * 4 * P->n_ext * (size_t)chunk);
      if (e != cudaSuccess) return fail(QED_ERR_OUT_OF_MEMORY, "cudaMalloc staging momenta");
      e = cudaMalloc(&P->d_out[b], sizeof(double) * (size_t)chunk);
      if (e != cudaSuccess) return fail(QED_ERR_OUT_OF_MEMORY, "cudaMalloc staging out");
    }
    P->cap = chunk;
  }
  const int rows = 4 * P->n_ext;
  int c = 0;
  for (long long i0 = 0; i0 < n_points; i0 += chunk, ++c) {
    const int b = c & 1;
    const long long cnt = std::min<long long>(chunk, n_points - i0);
    cudaStream_t st = P->hstream[b];
    const size_t spitch = sizeof(double) * (size_t)n_points;
    // row blocks to upload: all rows, or (ONSHELL) the 3 momentum rows 4j+1..4j+3 of every particle j
    const int nblk = onshell ? P->n_ext : 1, blk_rows = onshell ? 3 : rows;
    e = cudaSuccess;
    for (int k = 0; k < nblk && e == cudaSuccess; ++k) {
      if (conserve && k == e_out) continue;   // p' follows from momentum conservation on the device
      const int r0 = onshell ? 4 * k + 1 : 0;
      if (spitch <= (size_t)max_pitch) {
        e = cudaMemcpy2DAsync(P->d_mom[b] + (size_t)r0 * cnt, sizeof(double) * (size_t)cnt,
                              momenta_host + (size_t)r0 * n_points + i0, spitch, sizeof(double) * (size_t)cnt,
                              blk_rows, cudaMemcpyHostToDevice, st);
      } else {   // source pitch above the device limit (~2^28 points): one copy per SoA row
        for (int r = r0; r < r0 + blk_rows && e == cudaSuccess; ++r)
          e = cudaMemcpyAsync(P->d_mom[b] + (size_t)r * cnt, momenta_host + (size_t)r * n_points + i0,
                              sizeof(double) * (size_t)cnt, cudaMemcpyHostToDevice, st);
      }
    }
    if (e != cudaSuccess) return drain(cuda_fail(e, "H2D copy"));
    if (onshell) {
      const int grid = (int)std::min<long long>((cnt + 255) / 256, 8LL * P->num_sms);
      qed_onshell_energy_kernel<<<grid, 256, 0, st>>>(P->d_mom[b], cnt, P->n_ext, e_out, conserve ? 1 : 0);
      e = cudaGetLastError();
      if (e != cudaSuccess) return drain(cuda_fail(e, "on-shell energy kernel launch"));
      g_launches.fetch_add(1);
    }
    qed_status stt = launch_eval(P, P->d_mom[b], cnt, P->d_out[b], st, 0);
    if (stt != QED_OK) return drain(stt);
    e = cudaMemcpyAsync(out_host + i0, P->d_out[b], sizeof(double) * (size_t)cnt, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return drain(cuda_fail(e, "D2H copy"));
  }
  for (int b = 0; b < 2; ++b) {
    e = cudaStreamSynchronize(P->hstream[b]);
    if (e != cudaSuccess) return drain(cuda_fail(e, "stream synchronize"));
  }
  return QED_OK;
}

qed_status qed_mc_sum(const qed_process* proc, const qed_mc_config* cfg, double* partials, void* stream) {
  if (!proc || !cfg || !partials) return fail(QED_ERR_INVALID_ARGUMENT, "NULL argument");
  if (proc->n_in_ph != 1) return fail(QED_ERR_UNSUPPORTED, "qed_mc_sum supports e- gamma -> e- + n gamma only");
  if (!(cfg->sqrt_s > 1.0)) return fail(QED_ERR_INVALID_ARGUMENT, "sqrt_s must exceed m_e");
  if (!(cfg->omega_min >= 0.0)) return fail(QED_ERR_INVALID_ARGUMENT, "omega_min must be >= 0");
  if (cfg->n_points == 0) return QED_OK;
  if ((uintptr_t)partials & 7) return fail(QED_ERR_INVALID_ARGUMENT, "partials must be 8-byte aligned");
  qed_status dst = check_device(proc->device);
  if (dst != QED_OK) return dst;
  qed::QedEvalArgs a = proc->args;
  a.mom = nullptr;
  a.out = nullptr;
  a.n_points = 0;
  qed::QedMcArgs m;
  m.sqrt_s = cfg->sqrt_s;
  m.omega_min = cfg->omega_min;
  m.seed = cfg->seed;
  m.first_index = cfg->first_index;
  m.n_points = cfg->n_points;
  m.partials = partials;
  m.chunk = QED_MC_CHUNK;
  const unsigned long long c0 = cfg->first_index / QED_MC_CHUNK;
  const unsigned long long c1 = (cfg->first_index + cfg->n_points + QED_MC_CHUNK - 1) / QED_MC_CHUNK;
  const int grid = (int)std::min<unsigned long long>(c1 - c0, (unsigned long long)proc->mc_grid_blocks);
  void* params[] = {&a, &m};
  cudaError_t e = cudaLaunchKernel(proc->kern_mc, dim3(grid), dim3(proc->mc_wpb * 32), params, (size_t)proc->smem_mc,
                                   (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "mc kernel launch");
  g_launches.fetch_add(1);
  return QED_OK;
}

qed_status qed_get_process_info(const qed_process* P, qed_process_info* info) {
  if (!P || !info) return fail(QED_ERR_INVALID_ARGUMENT, "NULL argument");
  info->n_photons = P->n;
  info->n_ext = P->n_ext;
  info->n_configs = 1 << P->n_ext;   // up to 2^11
  long long f = 1;
  for (int i = 2; i <= P->N; ++i) f *= i;
  info->n_diagrams = (int)f;
  info->lanes_per_point = P->ppw > 0 ? 32 / P->ppw : 1 << P->N;
  info->warps_per_block = P->wpb;
  info->smem_per_block = P->smem;
  info->grid_blocks = P->grid_blocks;
  info->flops_per_point = P->flops;
  info->bytes_per_point = 8LL * (4 * P->n_ext + 1);
  info->algorithm = P->algorithm;
  info->variant = P->variant;
  info->n_variants = P->n_variants;
  return QED_OK;
}

}  // extern "C"
