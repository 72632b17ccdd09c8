"""B200-native batched tree-level QED |M|^2 engine (arXiv 2511.19456 hot path).

Public API: ``paper_2511_19456_b200.qed`` (ctypes binding of libqed's C ABI,
include/qed.h).  Build with ``python -m paper_2511_19456_b200.build``.
"""
