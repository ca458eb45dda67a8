"""The drop-in boundary in one process (VERDICT r1 "what's weak" 7, "next" 3).

oracle/_ref/bin/ref_drop_in links the UNMODIFIED reference library and libkrysp_gpu.so into
one binary and calls both with the reference's own types (krysp::CsrMatrix,
krysp::SolverConfig, krysp::CgTrace) — krysp::solve_* next to krysp::gpu::solve_*
(include/krysp_gpu_ref.hpp) — asserting bit-identical EXACT reports, SpMVs, dots and
conversions, and the same exception class and message on the error paths.  The binary is
built where the reference headers exist (oracle/Makefile refbin, from __graft_entry__.build)
and travels to the GPU box prebuilt.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "bin", "ref_drop_in")


def test_reference_types_through_the_device_bit_exact():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libkrysp_ref.so")):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    assert os.path.exists(EXE), "oracle/_ref/bin/ref_drop_in missing: run make -C oracle refbin"
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "ref drop-in ok" in out.stdout
