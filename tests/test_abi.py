"""CPU-side checks of the boundary: the C-ABI library builds for sm_100a, loads without a
GPU, and exports every symbol include/mps_b200.h declares; calls without a GPU fail
loudly (MPS_ECUDA), never fall back to the CPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "mps_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mps_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_1111_3124_b200 import _build
    _build.build()
    lib = ctypes.CDLL(_build.OUT)
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    import paper_1111_3124_b200 as m
    assert sorted(m.EXPORTS) == syms


def test_sm100a_cubin_present():
    import subprocess
    from paper_1111_3124_b200 import _build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.OUT], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1111_3124_b200 as m
    from synth import gen
    A, B, U = gen.update_batch_inputs(280, 2, 1)
    with pytest.raises(m.MpsError) as e:
        m.update_batch(280, 2, 1, A, B, U)
    assert e.value.rc == -8
    with pytest.raises(m.MpsError) as e:
        m.MPS(4, 280, 4)
    assert e.value.rc == -8


def test_record_size_and_strerror():
    import paper_1111_3124_b200 as m
    assert m.record_bytes(280) == 16 + 4 * 9
    assert m.record_bytes(512) == 16 + 4 * 16
    m.lib().mps_strerror.restype = ctypes.c_char_p
    assert m.lib().mps_strerror(-3) == b"Jacobi SVD did not converge"
