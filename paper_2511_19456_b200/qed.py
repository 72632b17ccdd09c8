"""Thin Python binding of libqed's C ABI (include/qed.h).

Argument marshalling only: every step of the hot path runs in the sm_100a
kernels inside libqed.so.  There is no fallback: if the library is missing or
fails to load, importing this module raises.  torch is used only to own device
memory and to supply the current CUDA stream.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libqed.so")

QED_OK = 0
QED_SUM = -1
MC_CHUNK = 1024
HOST_ONSHELL = 1   # QED_HOST_ONSHELL (include/qed.h)
HOST_CONSERVE = 2  # QED_HOST_CONSERVE (include/qed.h)
_STATUS = {0: "QED_OK", 1: "QED_ERR_INVALID_ARGUMENT", 2: "QED_ERR_UNSUPPORTED", 3: "QED_ERR_CUDA",
           4: "QED_ERR_OUT_OF_MEMORY", 5: "QED_ERR_INTERNAL"}

EXPORTED = ["qed_process_create", "qed_process_create_ex", "qed_process_destroy", "qed_eval_msq", "qed_eval_msq_configs",
            "qed_eval_msq_host", "qed_eval_msq_host_ex", "qed_mc_sum", "qed_get_process_info", "qed_last_error", "qed_launch_count"]
EXPORTED_ABC = ["abc_process_create", "abc_process_destroy", "abc_eval_msq", "abc_get_process_info"]


class QedError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {_STATUS.get(status, status)}: {msg}")
        self.status = status


class _Spec(ctypes.Structure):
    _fields_ = [("n_photons", ctypes.c_int), ("spins", ctypes.POINTER(ctypes.c_int8))]


class _McConfig(ctypes.Structure):
    _fields_ = [("sqrt_s", ctypes.c_double), ("omega_min", ctypes.c_double), ("seed", ctypes.c_uint64),
                ("first_index", ctypes.c_uint64), ("n_points", ctypes.c_uint64)]


class _Options(ctypes.Structure):
    _fields_ = [("algorithm", ctypes.c_int), ("variant", ctypes.c_int), ("kernel_family", ctypes.c_int)]


ALGORITHMS = {"cdag": 0, "bg": 1, "berends-giele": 1}
KERNEL_FAMILIES = {"default": 0, "lane-group": 1}


class ProcessInfo(ctypes.Structure):
    _fields_ = [("n_photons", ctypes.c_int), ("n_ext", ctypes.c_int), ("n_configs", ctypes.c_int),
                ("n_diagrams", ctypes.c_int), ("lanes_per_point", ctypes.c_int), ("warps_per_block", ctypes.c_int),
                ("smem_per_block", ctypes.c_int64), ("grid_blocks", ctypes.c_int),
                ("flops_per_point", ctypes.c_int64), ("bytes_per_point", ctypes.c_int64),
                ("algorithm", ctypes.c_int), ("variant", ctypes.c_int), ("n_variants", ctypes.c_int)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class AbcProcessInfo(ctypes.Structure):
    _fields_ = [("n_b", ctypes.c_int), ("n_diagrams", ctypes.c_int), ("algorithm", ctypes.c_int),
                ("grid_blocks", ctypes.c_int), ("threads_per_block", ctypes.c_int),
                ("flops_per_point", ctypes.c_int64), ("bytes_per_point", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libqed.so not built ({LIB_PATH}); run `python -m paper_2511_19456_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    lib.qed_process_create.argtypes = [ctypes.POINTER(_Spec), ctypes.POINTER(_Spec), ctypes.c_int,
                                       ctypes.POINTER(vp)]
    lib.qed_process_create_ex.argtypes = [ctypes.POINTER(_Spec), ctypes.POINTER(_Spec), ctypes.c_int,
                                          ctypes.POINTER(_Options), ctypes.POINTER(vp)]
    lib.qed_process_destroy.argtypes = [vp]
    lib.qed_eval_msq.argtypes = [vp, vp, i64, vp, vp]
    lib.qed_eval_msq_configs.argtypes = [vp, vp, i64, vp, vp]
    lib.qed_eval_msq_host.argtypes = [vp, vp, i64, vp]
    lib.qed_eval_msq_host_ex.argtypes = [vp, vp, i64, vp, ctypes.c_uint32]
    lib.qed_mc_sum.argtypes = [vp, ctypes.POINTER(_McConfig), vp, vp]
    lib.qed_get_process_info.argtypes = [vp, ctypes.POINTER(ProcessInfo)]
    lib.abc_process_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
    lib.abc_process_destroy.argtypes = [vp]
    lib.abc_eval_msq.argtypes = [vp, vp, i64, vp, vp]
    lib.abc_get_process_info.argtypes = [vp, ctypes.POINTER(AbcProcessInfo)]
    for f in ("abc_process_create", "abc_process_destroy", "abc_eval_msq", "abc_get_process_info"):
        getattr(lib, f).restype = ctypes.c_int
    lib.qed_last_error.restype = ctypes.c_char_p
    lib.qed_launch_count.restype = ctypes.c_int64
    for f in EXPORTED:
        if f not in ("qed_last_error", "qed_launch_count"):
            getattr(lib, f).restype = ctypes.c_int
    return lib


_lib = _load()


def library() -> ctypes.CDLL:
    return _lib


def _check(st: int, where: str) -> None:
    if st != QED_OK:
        raise QedError(st, where, _lib.qed_last_error().decode())


def launch_count() -> int:
    return int(_lib.qed_launch_count())


def _stream_ptr(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _ptr(t, numel: int, name: str, device=None, shape=None) -> int:
    """Pointer of a contiguous float64 tensor with exactly ``numel`` elements (and ``shape``, when
    given), on ``device`` (a cuda device index) or on the host (device=None)."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor")
    if t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError(f"{name} must be contiguous float64")
    if device is None:
        if t.is_cuda:
            raise ValueError(f"{name} must be a host tensor for this entry point")
    elif not t.is_cuda or t.device.index != device:
        raise ValueError(f"{name} must be on cuda:{device} (the handle's device), got {t.device}")
    if shape is not None and t.dim() > 1 and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, need {tuple(shape)}")
    if t.numel() != numel:
        raise ValueError(f"{name} has {t.numel()} elements, need exactly {numel}")
    return t.data_ptr()


class Process:
    """qed_process handle.  ``in_spins`` / ``out_spins``: None (all summed) or a list
    [electron, photon...] of -1 (summed) / 0 / 1 (fixed).  ``algorithm``: "cdag" (the paper's
    node-reduced diagram DAG, default) or "bg" (Berends-Giele distributive rewrite); ``variant``:
    launch variant (None = default / QED_VARIANT)."""

    def __init__(self, n: int, n_in_photons: int = 1, in_spins=None, out_spins=None, algorithm: str = "cdag",
                 variant: int | None = None, kernel_family: str = "default"):
        self.n = n
        self.n_in_photons = n_in_photons
        self.n_out_photons = n + 1 - n_in_photons
        self.n_ext = n + 3
        self._keep = []

        def spec(nph, spins):
            s = _Spec()
            s.n_photons = nph
            if spins is None:
                s.spins = None
            else:
                arr = (ctypes.c_int8 * (nph + 1))(*[int(x) for x in spins])
                self._keep.append(arr)
                s.spins = ctypes.cast(arr, ctypes.POINTER(ctypes.c_int8))
            return s

        self._in = spec(n_in_photons, in_spins)
        self._out = spec(self.n_out_photons, out_spins)
        h = ctypes.c_void_p()
        if algorithm not in ALGORITHMS:
            raise ValueError(f"algorithm must be one of {sorted(ALGORITHMS)}")
        self.algorithm = algorithm
        if kernel_family not in KERNEL_FAMILIES:
            raise ValueError(f"kernel_family must be one of {sorted(KERNEL_FAMILIES)}")
        opt = _Options(ALGORITHMS[algorithm], -1 if variant is None else int(variant), KERNEL_FAMILIES[kernel_family])
        _check(_lib.qed_process_create_ex(ctypes.byref(self._in), ctypes.byref(self._out), n, ctypes.byref(opt),
                                          ctypes.byref(h)), "qed_process_create_ex")
        self._h = h
        import torch
        # the library binds the handle to the current device (include/qed.h "Device binding")
        self.device = torch.cuda.current_device() if torch.cuda.is_available() else None

    def close(self):
        if getattr(self, "_h", None):
            _lib.qed_process_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        inf = ProcessInfo()
        _check(_lib.qed_get_process_info(self._h, ctypes.byref(inf)), "qed_get_process_info")
        return inf.as_dict()

    def _soa(self, momenta_soa, n_points, device):
        # the kernels read row r at momenta + r * n_points: the tensor must hold exactly
        # 4 * n_ext rows of n_points (a wider batch would be read with the wrong row stride)
        return _ptr(momenta_soa, 4 * self.n_ext * n_points, "momenta", device, (4 * self.n_ext, n_points))

    def eval_msq(self, momenta_soa, out, n_points: int | None = None, stream=None) -> None:
        """momenta_soa: cuda float64 [(4*n_ext), n_points] contiguous; out: cuda float64 [n_points]."""
        n_points = out.numel() if n_points is None else n_points
        _check(_lib.qed_eval_msq(self._h, self._soa(momenta_soa, n_points, self.device), n_points,
                                 _ptr(out, n_points, "out", self.device), _stream_ptr(stream)), "qed_eval_msq")

    def eval_msq_configs(self, momenta_soa, out, n_points: int, stream=None) -> None:
        H = 1 << self.n_ext
        _check(_lib.qed_eval_msq_configs(self._h, self._soa(momenta_soa, n_points, self.device), n_points,
                                         _ptr(out, n_points * H, "out", self.device), _stream_ptr(stream)),
               "qed_eval_msq_configs")

    def eval_msq_host(self, momenta_soa_host, out_host, n_points: int | None = None, onshell: bool = False,
                      conserve: bool = False) -> None:
        """Host buffers (pinned recommended): momenta [(4*n_ext), n_points], out [n_points].
        onshell=True: qed_eval_msq_host_ex(QED_HOST_ONSHELL), only the 3-momenta are uploaded and the
        energies are restored on the device from the mass shell; conserve=True (with onshell) adds
        QED_HOST_CONSERVE, the outgoing electron is restored from momentum conservation (include/qed.h)."""
        n_points = out_host.numel() if n_points is None else n_points
        mom = self._soa(momenta_soa_host, n_points, None)
        out = _ptr(out_host, n_points, "out", None)
        if onshell or conserve:
            flags = (HOST_ONSHELL if onshell else 0) | (HOST_CONSERVE if conserve else 0)
            _check(_lib.qed_eval_msq_host_ex(self._h, mom, n_points, out, flags), "qed_eval_msq_host_ex")
        else:
            _check(_lib.qed_eval_msq_host(self._h, mom, n_points, out), "qed_eval_msq_host")

    def mc_sum(self, partials, sqrt_s: float, omega_min: float, seed: int, first_index: int, n_points: int,
               stream=None) -> None:
        """Accumulate Monte-Carlo chunk partial sums into the device tensor ``partials``
        (float64, 3 * n_chunks, zeroed by the caller)."""
        cfg = _McConfig(float(sqrt_s), float(omega_min), int(seed), int(first_index), int(n_points))
        n_chunks = (first_index + n_points + MC_CHUNK - 1) // MC_CHUNK
        if partials.numel() < 3 * n_chunks:
            raise ValueError(f"partials has {partials.numel()} elements, need >= {3 * n_chunks}")
        _check(_lib.qed_mc_sum(self._h, ctypes.byref(cfg), _ptr(partials, partials.numel(), "partials", self.device),
                               _stream_ptr(stream)), "qed_mc_sum")


# ABC model (include/abc.h): masses and coupling of the library (reading A2)
ABC_MASS_A, ABC_MASS_B, ABC_MASS_C, ABC_COUPLING = 1.0, 0.5, 1.2, 1.0


class AbcProcess:
    """abc_process handle: A + n_in B -> A + n_out B (n_in + n_out even), algorithm "cdag" or "bg"."""

    def __init__(self, n_out: int, n_in: int = 1, algorithm: str = "cdag"):
        if algorithm not in ALGORITHMS:
            raise ValueError(f"algorithm must be one of {sorted(ALGORITHMS)}")
        self.n_in, self.n_out = n_in, n_out
        self.n_ext = n_in + n_out + 2
        self.algorithm = algorithm
        h = ctypes.c_void_p()
        _check(_lib.abc_process_create(n_in, n_out, ALGORITHMS[algorithm], ctypes.byref(h)), "abc_process_create")
        self._h = h
        import torch
        self.device = torch.cuda.current_device() if torch.cuda.is_available() else None

    def close(self):
        if getattr(self, "_h", None):
            _lib.abc_process_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        inf = AbcProcessInfo()
        _check(_lib.abc_get_process_info(self._h, ctypes.byref(inf)), "abc_get_process_info")
        return inf.as_dict()

    def eval_msq(self, momenta_soa, out, n_points: int | None = None, stream=None) -> None:
        """momenta_soa: cuda float64 [(4*n_ext), n_points]; out: cuda float64 [n_points]."""
        n_points = out.numel() if n_points is None else n_points
        mp = _ptr(momenta_soa, 4 * self.n_ext * n_points, "momenta", self.device, (4 * self.n_ext, n_points))
        _check(_lib.abc_eval_msq(self._h, mp, n_points, _ptr(out, n_points, "out", self.device), _stream_ptr(stream)),
               "abc_eval_msq")
