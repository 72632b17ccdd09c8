// abc_runtime.cu -- libqed C-ABI of the ABC-model kernels (include/abc.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <new>
#include <string>

#include "abc.h"
#include "abc_kernel.cuh"

extern "C" {
const void* abcgen_kernel_cdag_N2(void);
const void* abcgen_kernel_cdag_N4(void);
const void* abcgen_kernel_cdag_N6(void);
const void* abcgen_kernel_bg_N2(void);
const void* abcgen_kernel_bg_N4(void);
const void* abcgen_kernel_bg_N6(void);
long long abcgen_flops_cdag_N2(void);
long long abcgen_flops_cdag_N4(void);
long long abcgen_flops_cdag_N6(void);
long long abcgen_flops_bg_N2(void);
long long abcgen_flops_bg_N4(void);
long long abcgen_flops_bg_N6(void);
// shared with qed_runtime.cu: error message and launch counter of the library
qed_status qed_internal_fail(qed_status st, const char* msg);
void qed_internal_count_launch(void);
}

namespace {
struct Entry {
  const void* (*kernel)(void);
  long long (*flops)(void);
};
const Entry kCdag[] = {{abcgen_kernel_cdag_N2, abcgen_flops_cdag_N2}, {abcgen_kernel_cdag_N4, abcgen_flops_cdag_N4},
                       {abcgen_kernel_cdag_N6, abcgen_flops_cdag_N6}};
const Entry kBg[] = {{abcgen_kernel_bg_N2, abcgen_flops_bg_N2}, {abcgen_kernel_bg_N4, abcgen_flops_bg_N4},
                     {abcgen_kernel_bg_N6, abcgen_flops_bg_N6}};
constexpr int kThreads = 256;

qed_status cuda_fail(cudaError_t e, const char* what) {
  return qed_internal_fail(QED_ERR_CUDA, (std::string(what) + ": " + cudaGetErrorString(e)).c_str());
}
}  // namespace

struct abc_process {
  int N = 0, n_in = 0, algorithm = 0, device = 0, grid = 0;
  const void* kern = nullptr;
  long long flops = 0;
  qed::AbcArgs args{};
};

extern "C" {

qed_status abc_process_create(int n_in, int n_out, int algorithm, abc_process** proc) {
  if (!proc) return qed_internal_fail(QED_ERR_INVALID_ARGUMENT, "proc is NULL");
  *proc = nullptr;
  if (n_in < 0 || n_out < 0) return qed_internal_fail(QED_ERR_INVALID_ARGUMENT, "negative B-on count");
  const int N = n_in + n_out;
  if (N % 2) return qed_internal_fail(QED_ERR_INVALID_ARGUMENT, "the number of B-ons must be even (PAPER.md:523)");
  if (algorithm != QED_ALGO_CDAG && algorithm != QED_ALGO_BERENDS_GIELE)
    return qed_internal_fail(QED_ERR_INVALID_ARGUMENT, "unknown algorithm");
  const Entry* tab = algorithm == QED_ALGO_CDAG ? kCdag : kBg;
  const void* kern = (N >= 2 && N <= 6) ? tab[N / 2 - 1].kernel() : nullptr;
  if (!kern)
    return qed_internal_fail(QED_ERR_UNSUPPORTED, algorithm == QED_ALGO_CDAG ? "ABC CDAG kernels: N = 2, 4, 6 B-ons"
                                                                             : "ABC Berends-Giele kernels: N = 2, 4, 6 B-ons");
  abc_process* P = new (std::nothrow) abc_process;
  if (!P) return qed_internal_fail(QED_ERR_OUT_OF_MEMORY, "host allocation failed");
  P->N = N;
  P->n_in = n_in;
  P->algorithm = algorithm;
  P->kern = kern;
  P->flops = tab[N / 2 - 1].flops();
  for (int b = 0; b < N; ++b) {
    P->args.part[b] = b < n_in ? 1 + b : n_in + 2 + (b - n_in);
    P->args.sg[b] = b < n_in ? 1.0 : -1.0;
  }
  P->args.g2n = std::pow(ABC_COUPLING, 2 * N);
  cudaError_t e = cudaGetDevice(&P->device);
  int sms = 0, bps = 0;
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P->device);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kThreads, 0);
  if (e != cudaSuccess) {
    delete P;
    return cuda_fail(e, "abc_process_create");
  }
  P->grid = std::max(bps, 1) * sms;
  *proc = P;
  return QED_OK;
}

qed_status abc_process_destroy(abc_process* proc) {
  delete proc;
  return QED_OK;
}

qed_status abc_eval_msq(const abc_process* P, const double* mom, int64_t n_points, double* out, void* stream) {
  if (!P) return qed_internal_fail(QED_ERR_INVALID_ARGUMENT, "proc is NULL");
  if (n_points < 0) return qed_internal_fail(QED_ERR_INVALID_ARGUMENT, "n_points < 0");
  if (n_points == 0) return QED_OK;
  if (!mom || !out) return qed_internal_fail(QED_ERR_INVALID_ARGUMENT, "momenta/out is NULL");
  if (((uintptr_t)mom & 7) || ((uintptr_t)out & 7))
    return qed_internal_fail(QED_ERR_INVALID_ARGUMENT, "pointers must be 8-byte aligned");
  int cur = -1;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (cur != P->device) return qed_internal_fail(QED_ERR_INVALID_ARGUMENT, "current device differs from the handle's device");
  qed::AbcArgs a = P->args;
  a.mom = mom;
  a.out = out;
  a.n_points = n_points;
  const long long need = (n_points + kThreads - 1) / kThreads;
  const int grid = (int)std::min<long long>(need, P->grid);
  void* params[] = {&a};
  e = cudaLaunchKernel(P->kern, dim3(grid), dim3(kThreads), params, 0, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "abc kernel launch");
  qed_internal_count_launch();
  return QED_OK;
}

qed_status abc_get_process_info(const abc_process* P, abc_process_info* info) {
  if (!P || !info) return qed_internal_fail(QED_ERR_INVALID_ARGUMENT, "NULL argument");
  info->n_b = P->N;
  long long f = 1;
  for (int i = 2; i <= P->N; ++i) f *= i;
  info->n_diagrams = (int)f;
  info->algorithm = P->algorithm;
  info->grid_blocks = P->grid;
  info->threads_per_block = kThreads;
  info->flops_per_point = P->flops;
  info->bytes_per_point = 8LL * (4 * (P->N + 1) + 1);
  return QED_OK;
}

}  // extern "C"
