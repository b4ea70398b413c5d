"""CPU suite: the C-ABI library loads, exports every symbol include/pqrr_dev.h
declares, and fails loudly (no CPU fallback) when no GPU is present."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pqrr_dev.h")
LIB = os.path.join(ROOT, "paper_1102_3828_b200", "lib", "libpqrr_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(pqrr_dev_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    assert os.path.exists(LIB), "build the library first (__graft_entry__.build())"
    lib = ctypes.CDLL(LIB)
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    from paper_1102_3828_b200 import _lib

    assert sorted(_lib.EXPORTED) == syms


def test_sm100a_code_in_library():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu(pq):
    if pq.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(pq.DeviceUnavailable):
        pq.kernels.assign_batch(np.zeros((4, 4), np.float32), np.zeros((2, 4), np.float32))
    with pytest.raises(pq.DeviceUnavailable):
        pq.synth(2, 0, 4, 8)


def test_argument_errors_before_device(pq):
    # reference messages are raised before any device work
    with pytest.raises(ValueError, match="dimension not divisible"):
        pq.pq_train(np.zeros((300, 10), np.float32), 3)
    with pytest.raises(ValueError, match="insufficient training data"):
        pq.kmeans_train(np.zeros((3, 2), np.float32), 5)
