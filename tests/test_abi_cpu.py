"""C-ABI checks that need no GPU: the library loads, exports exactly what include/sfdg.h
declares, validates arguments like the reference, and fails loudly (SFDG_CUDA_ERROR)
instead of falling back to a CPU path when no device is present."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1602_00412_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sfdg.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sfdg_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("sfdg_sketcher_create", "sfdg_sketcher_append_csr", "sfdg_sketcher_finalize", "sfdg_merge",
              "sfdg_merge_device", "sfdg_dense_shrink", "sfdg_sparse_shrink", "sfdg_boosted_sparse_shrink"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    L = P.lib()
    for s in declared_symbols():
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sfdg_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_header_compiles_as_c_and_cpp(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "sfdg.h"\nint main(void){ sfdg_stats s; (void)s; return 0; }\n')
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-c", str(src), "-o",
                    str(tmp_path / "t.o")], check=True)
    hdr = os.path.join(ROOT, "include", "sfd_gpu.hpp")
    if os.path.exists(hdr):
        cpp = tmp_path / "t.cpp"
        cpp.write_text('#include "sfd_gpu.hpp"\nint main(){ sfd_gpu::SketchConfig c; (void)c; return 0; }\n')
        subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-c", str(cpp),
                        "-o", str(tmp_path / "t2.o")], check=True)


def test_config_validation_without_device():
    # sketch.cpp:9-12 -- validated before any device work (tests/test_sketch.cpp:295-302)
    for ell, d, delta in ((0, 4, 0.1), (5, 4, 0.1), (2, 4, 1.5), (2, 4, 0.0)):
        with pytest.raises(P.InvalidArgument):
            P.SfdSketcher(P.SketchConfig(ell=ell, d=d, delta=delta))


def test_power_iteration_count_host():
    assert P.power_iteration_count(3000) == 38
    assert P.power_iteration_count(3000, P.PowerConfig(q_override=0)) == 0
    with pytest.raises(P.InvalidArgument):
        P.power_iteration_count(10, P.PowerConfig(epsilon=1.5))


@pytest.mark.skipif(P.device_count() > 0, reason="GPU present: the no-device contract is not observable")
def test_no_cpu_fallback_without_device():
    with pytest.raises(P.CudaError):
        P.SfdSketcher(P.SketchConfig(ell=2, d=8))
    with pytest.raises(P.CudaError):
        P.dense_shrink(np.eye(3), 2)
    with pytest.raises(P.CudaError):
        P.gaussian_matrix(3, 3, 0)
