"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every function the
header declares, and rejects bad arguments synchronously (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2507_02754_b200 import binding
    return binding.load_library()


def header_functions():
    src = open(os.path.join(ROOT, "include", "simplicial_attn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(simplicial_attn_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    fns = header_functions()
    for f in ("simplicial_attn_fwd", "simplicial_attn_bwd", "simplicial_attn_fwd_prefixed",
              "simplicial_attn_bwd_prefixed", "simplicial_attn_bwd_workspace_bytes"):
        assert f in fns


def test_exports_every_declared_symbol(lib):
    from paper_2507_02754_b200 import binding
    for f in header_functions():
        assert hasattr(lib, f), f
    assert set(binding.EXPORTS) == set(header_functions())


def test_library_is_sm100a(lib):
    assert b"sm_100a" in lib.simplicial_attn_version()


def test_status_strings(lib):
    assert lib.simplicial_attn_status_string(0) == b"SA_OK"
    assert lib.simplicial_attn_status_string(3) == b"SA_ERR_WORKSPACE"


def test_argument_validation_without_gpu(lib):
    fake = ctypes.c_void_p(0x1000)
    null = ctypes.c_void_p(0)
    f = lib.simplicial_attn_fwd
    ok_args = lambda **kw: [kw.get(n, fake) for n in ("q", "k", "v", "k2", "v2", "o", "lse")]
    big = 1 << 40
    # null pointer
    assert f(*ok_args(q=null), fake, big, 1, 1, 8, 16, 4, 2, 0, null) == 1
    # bad sizes / windows
    assert f(*ok_args(), fake, big, 0, 1, 8, 16, 4, 2, 0, null) == 1
    assert f(*ok_args(), fake, big, 1, 1, 8, 16, 0, 2, 0, null) == 1
    assert f(*ok_args(), fake, big, 1, 1, 8, 16, 4, -1, 0, null) == 1
    # DET needs D >= 3; D > 128 unsupported; unknown flag bits rejected
    assert f(*ok_args(), fake, big, 1, 1, 8, 2, 4, 2, 1, null) == 1
    assert f(*ok_args(), fake, big, 1, 1, 8, 256, 4, 2, 0, null) == 2
    assert f(*ok_args(), fake, big, 1, 1, 8, 16, 4, 2, 1 << 9, null) == 1
    # prefixed: negative prefix
    assert lib.simplicial_attn_fwd_prefixed(*ok_args(), fake, big, 1, 1, 8, 16, 4, 2, -1, 0, null) == 1
    # bf16 inputs with no tensor-core kernel for the shape: rejected, never a silent CUDA-core run
    assert f(*ok_args(), fake, big, 1, 1, 8, 16, 4, 2, 0, null) == 2          # D = 16
    assert f(*ok_args(), fake, big, 1, 1, 512, 64, 256, 200, 0, null) == 2   # both windows > 128
    # forward workspace: the tensor-core path needs one; too small / NULL is rejected
    fws = lib.simplicial_attn_fwd_workspace_bytes(1, 2, 64, 128, 32, 8, 0)
    assert fws >= 3 * 2 * 64 * 128 * 2
    assert lib.simplicial_attn_fwd_workspace_bytes_prefixed(1, 2, 64, 128, 32, 8, 7, 0) > fws
    assert f(*ok_args(), fake, fws - 1, 1, 2, 64, 128, 32, 8, 0, null) == 3
    assert f(*ok_args(), null, fws, 1, 2, 64, 128, 32, 8, 0, null) == 3
    assert lib.simplicial_attn_fwd_workspace_bytes(1, 1, 128, 16, 32, 8, 2) == 0  # fp32 path: none
    # backward: workspace too small
    ws = lib.simplicial_attn_bwd_workspace_bytes(1, 2, 64, 16, 8, 4, 2)
    assert ws >= 4 * 2 * 64
    b = lib.simplicial_attn_bwd
    args = [fake] * 14
    assert b(*args, ws - 1, 1, 2, 64, 16, 8, 4, 2, null) == 3
    assert b(*args, 1 << 40, 1, 2, 64, 16, 8, 4, 0, null) == 2  # bf16, D = 16
    assert lib.simplicial_attn_host_step_scratch_bytes(1, 2, 64, 16, 8, 4, 2) > 0


def test_path_selection(lib):
    # fp32 inputs always take the exact CUDA-core path
    assert lib.simplicial_attn_fwd_path(1, 1, 128, 16, 32, 8, 2) == 1
    assert lib.simplicial_attn_fwd_path(1, 1, 128, 16, 32, 8, 1 << 3) == 1
    assert lib.simplicial_attn_fwd_path(1, 1, 128, 300, 32, 8, 0) == 0
    # bf16: tensor cores or nothing (SA_FORCE_SIMT is the only way onto the CUDA-core kernels)
    for fn in (lib.simplicial_attn_fwd_path, lib.simplicial_attn_bwd_path):
        assert fn(4, 16, 8192, 128, 512, 32, 0) == 2
        assert fn(2, 16, 16384, 128, 512, 32, 1) == 2
        assert fn(1, 1, 256, 128, 40, 64, 0) == 2     # folded window 40: not a power of two
        assert fn(1, 1, 256, 128, 64, 1, 0) == 2      # w2 = 1
        assert fn(1, 1, 256, 64, 200, 128, 1) == 2
        assert fn(1, 1, 256, 48, 64, 32, 0) == 0      # D = 48: no tcgen05 kernel
        assert fn(1, 1, 512, 128, 256, 200, 0) == 0   # both windows > 128
        assert fn(1, 1, 256, 48, 64, 32, 1 << 3) == 1


def test_product_path_does_not_touch_oracle():
    """The package never imports, links or loads the oracle (DESIGN.md boundary rule)."""
    pkg = os.path.join(ROOT, "paper_2507_02754_b200")
    bad = re.compile(r"(^\s*(import|from)\s+oracle\b)|liboracle|oracle\.c\b|sa_oracle_", re.M)
    for dp, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                assert not bad.search(open(os.path.join(dp, fn)).read()), fn
