"""CPU-side checks of the C-ABI library: it builds, loads, exports every symbol that
include/*.h declares, and its host-side validation returns the documented status codes
(no compute call is made -- without a GPU every valid call stops at the device check)."""
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2504_07004_b200 import _lib, build

    build.build()
    return _lib.load()


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        syms |= set(re.findall(r"^\s*(?:const\s+)?[a-zA-Z_][\w\s\*]*?\b(cy_\w+)\s*\(", txt, flags=re.M))
    return syms


def test_header_declares_all_entry_points():
    syms = declared_symbols()
    for s in ("cy_gemm", "cy_gemm_batched", "cy_dual_gemm", "cy_gemm_rowreduce", "cy_status_string"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    from paper_2504_07004_b200 import _lib

    syms = declared_symbols()
    assert syms == set(_lib.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s


def test_library_exports_exactly_the_declared_symbols(lib):
    """Every exported C symbol of the product library (nm -D, the cy_ prefix) is declared in
    include/*.h and vice versa: no undeclared entry point (e.g. a trace hook) ships."""
    import shutil
    import subprocess

    from paper_2504_07004_b200 import build

    nm = shutil.which("nm")
    if not nm:
        pytest.skip("nm not available")
    out = subprocess.run([nm, "-D", "--defined-only", build.OUT], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if ln.split() and ln.split()[-1].startswith("cy_")
                and " T " in ln}
    assert exported == declared_symbols()


def test_product_build_has_no_experiment_switches():
    """Timing-experiment switches (CY_DEBUG_MODE: invalid results) are compile-time only and the
    product build never sets them; the kernel reads no such run-time parameter."""
    from paper_2504_07004_b200 import build

    assert not any(f.startswith("-DCY_DEBUG") for f in build.FLAGS)
    with pytest.raises(ValueError):
        build.build(defines=("CY_DEBUG_MODE=1",))
    src = open(os.path.join(ROOT, "paper_2504_07004_b200", "csrc", "cy_gemm.cu")).read()
    assert "CY_DEBUG_MODE" not in src  # no getenv of it on the host side
    kern = open(os.path.join(ROOT, "paper_2504_07004_b200", "csrc", "cy_kernel.cuh")).read()
    assert "p.debug" not in kern


def test_product_build_reads_no_tuning_knobs():
    """Tile-order / L2 / scheduling / attention-variant knobs are read from the environment only in
    experiment builds (CY_TUNING_KNOBS, CY_ATTN_EXPERIMENTS): the product library carries none of
    their names, so no environment variable can change what the product path runs."""
    from paper_2504_07004_b200 import build

    data = open(build.build(), "rb").read()
    for knob in (b"CY_GROUP_M", b"CY_RASTER", b"CY_SERP", b"CY_L2_POLICY", b"CY_B4D", b"CY_SCHED", b"CY_PDL",
                 b"CY_SLEEP_NS", b"CY_A_REUSE", b"CY_L2_PROMO", b"CY_ATTN_KERNEL", b"CY_ATTN_CS", b"CY_ATTN_EMU"):
        assert knob not in data, knob


def test_library_is_sm100a_and_uses_tcgen05():
    """The cubin inside the .so is sm_100a and contains tcgen05 MMA / TMA / TMEM loads."""
    import shutil
    import subprocess

    from paper_2504_07004_b200 import build

    so = build.build()
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    lst = subprocess.run([cuobjdump, "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in lst
    sass = subprocess.run([cuobjdump, "-sass", so], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "UTMALDG", "UTMASTG", "LDTM"):
        assert mnem in sass, mnem
    assert "HMMA" not in re.sub(r"UTCHMMA", "", sass)  # no legacy mma.sync path


def test_status_strings(lib):
    for s in range(6):
        assert lib.cy_status_string(s).decode().startswith("CY_")


def test_config_menu(lib):
    import ctypes

    n = lib.cy_num_configs()
    assert n >= 4
    for i in range(n):
        v = [ctypes.c_int() for _ in range(4)]
        assert lib.cy_config_info(i, *[ctypes.byref(x) for x in v]) == 0
        cg, tm, tn, st = (x.value for x in v)
        assert cg in (1, 2) and tm in (128 * cg, 512) and tn in (64, 128, 256, 512) and st >= 2
    assert lib.cy_config_info(n, None, None, None, None) == 1
    assert lib.cy_force_config(n) == 1
    assert lib.cy_force_config(-1) == 0


# ------------------------------------------------------------------ host-side validation
P = 1 << 20  # fake, 16-B aligned "device" addresses: never dereferenced by validation


def test_invalid_values(lib):
    f = lib.cy_gemm
    assert f(0, -1, 8, 8, 1.0, P, 8, P, 8, 0.0, None, 8, P * 4, 8, None) == 1   # negative m
    assert f(0, 8, 8, 8, 1.0, P, 4, P, 8, 0.0, None, 8, P * 4, 8, None) == 1    # lda < k
    assert f(0, 8, 8, 8, 1.0, P, 8, P, 8, 0.0, None, 8, P * 4, 4, None) == 1    # ldd < n
    assert f(0, 8, 8, 8, 1.0, None, 8, P, 8, 0.0, None, 8, P * 4, 8, None) == 1  # NULL A
    assert f(0, 8, 8, 8, 1.0, P, 8, P * 2, 8, 1.0, None, 8, P * 4, 8, None) == 1  # beta != 0, NULL C
    assert f(7, 8, 8, 8, 1.0, P, 8, P * 2, 8, 0.0, None, 8, P * 4, 8, None) == 1  # bad dtype
    # D overlapping A
    assert f(0, 8, 8, 8, 1.0, P, 8, P * 2, 8, 0.0, None, 8, P + 16, 8, None) == 1
    # dual SUM with D1 given
    assert lib.cy_dual_gemm(0, 1, 8, 8, 8, 1.0, P, 8, P * 2, 8, P * 3, 8, 0.0, None, 8, None, 8,
                            P * 4, 8, P * 5, 8, None) == 1
    # rowreduce: y overlapping D
    assert lib.cy_gemm_rowreduce(0, 8, 8, 8, 1.0, P, 8, P * 2, 8, 0.0, None, 8, P * 4, 8, P * 4 + 64,
                                 None) == 1


def test_batched_zero_stride_rejected(lib):
    # broadcast (stride 0) operands are not supported: clear INVALID_VALUE, not a launch failure
    assert lib.cy_gemm_batched(0, 8, 8, 8, 2, 1.0, P, 8, 0, P * 2, 8, 64, 0.0, None, 8, 64, P * 4, 8, 64,
                               None) == 1


def test_misaligned(lib):
    f = lib.cy_gemm
    assert f(0, 8, 8, 8, 1.0, P + 2, 8, P * 2, 8, 0.0, None, 8, P * 4, 8, None) == 2  # A not 16-B aligned
    assert f(0, 8, 12, 12, 1.0, P, 12, P * 2, 12, 0.0, None, 8, P * 4, 12, None) == 2  # ld*2 % 16 != 0


def test_noop_sizes_return_ok_without_device(lib):
    f = lib.cy_gemm
    assert f(0, 0, 8, 8, 1.0, P, 8, P * 2, 8, 0.0, None, 8, P * 4, 8, None) == 0
    assert f(0, 8, 0, 8, 1.0, P, 8, P * 2, 8, 0.0, None, 8, P * 4, 8, None) == 0
    assert lib.cy_gemm_batched(0, 8, 8, 8, 0, 1.0, P, 8, 64, P * 2, 8, 64, 0.0, None, 8, 64, P * 4, 8, 64,
                               None) == 0


def test_valid_call_without_gpu_is_unsupported_device(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert lib.cy_gemm(0, 8, 8, 8, 1.0, P, 8, P * 2, 8, 0.0, None, 8, P * 4, 8, None) == 3


def test_product_package_never_imports_oracle():
    """The product path shares no code with oracle/ and never imports it."""
    pkg = os.path.join(ROOT, "paper_2504_07004_b200")
    for f in glob.glob(os.path.join(pkg, "**", "*"), recursive=True):
        if f.endswith((".py", ".cu", ".cuh", ".h", ".c")):
            txt = open(f).read()
            assert not re.search(r"\boracle\b", re.sub(r"#.*|//.*", "", txt)), f
