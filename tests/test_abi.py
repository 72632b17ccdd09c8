"""CPU-side checks of the boundary: libqed.so loads and exports every symbol that
include/qed.h declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions(header="qed.h", prefix="qed"):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(rf"\b({prefix}_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    names = _declared_functions()
    for f in ("qed_process_create", "qed_eval_msq", "qed_mc_sum", "qed_process_destroy"):
        assert f in names


def test_library_exports_every_declared_symbol():
    from paper_2511_19456_b200 import qed
    lib = qed.library()
    missing = [f for f in _declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    assert set(qed.EXPORTED) <= set(_declared_functions())


def test_library_exports_every_abc_symbol():
    """include/abc.h (ABC model, App. F) is served by the same library."""
    from paper_2511_19456_b200 import qed
    names = _declared_functions("abc.h", "abc")
    assert {"abc_process_create", "abc_eval_msq", "abc_process_destroy", "abc_get_process_info"} <= set(names)
    missing = [f for f in names if not hasattr(qed.library(), f)]
    assert not missing, missing


def test_every_header_symbol_is_exported():
    import glob
    from paper_2511_19456_b200 import qed
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        for f in set(re.findall(r"^\s*(?:qed_status|const char\*|int64_t)\s+([a-z_]+)\s*\(", src, flags=re.M)):
            assert hasattr(qed.library(), f), (h, f)


def test_library_is_sm100a_only():
    """The fatbinary contains sm_100a SASS (no PTX JIT fallback, no other arch)."""
    import subprocess
    from paper_2511_19456_b200 import qed
    out = subprocess.run(["cuobjdump", "--list-elf", qed.LIB_PATH], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_errors_without_gpu_are_reported_not_raised():
    """qed_process_create fails with a status (no crash, no CPU fallback) when no device exists."""
    import torch
    if torch.cuda.is_available():
        return
    from paper_2511_19456_b200 import qed
    try:
        qed.Process(2)
    except qed.QedError as e:
        assert e.status == 3
    else:
        raise AssertionError("expected QED_ERR_CUDA without a GPU")


def test_tensor_core_joins_are_compiled():
    """The default n = 3..5 CDAG kernels join on the FP64 tensor core: the library's SASS holds DMMA
    instructions (DESIGN.md kernel 2-MMA), and the CUDA-core FP64 path (DFMA) beside them."""
    import subprocess
    from paper_2511_19456_b200 import qed
    sass = subprocess.run(["cuobjdump", "-sass", qed.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass and "DFMA" in sass
