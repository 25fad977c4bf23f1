"""The C-ABI library: builds for sm_100a, loads without a GPU, exports every
symbol include/gcb200.h declares, and fails loudly (no CPU fallback) when
no device is present."""

import ctypes
import os
import re

import pytest

from paper_1810_08429_b200 import _native, build_native
from paper_1810_08429_b200.errors import DeviceError

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "include", "gcb200.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gc_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_loads():
    build_native.build()
    lib = _native.load()
    assert lib.gc_abi_version() == _native.ABI_VERSION


def test_every_declared_symbol_is_exported_and_bound():
    lib = ctypes.CDLL(_native.LIB_PATH)
    names = declared()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
        assert name in _native.EXPORTED, "%s has no ctypes signature" % name


def test_sm100a_code_object():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_panel_kernel_issues_all_loads_before_the_first_fma():
    """The bulk matvec kernel's streaming loop must keep PAN_UNROLL matrix
    loads in flight per thread: every LDG of the unrolled batch is issued
    before the first DFMA.  ptxas may interleave them under the 40-register
    cap (6 CTAs/SM), which cost 6 % of the C2 product in round 2 - this
    guards the SASS schedule (csrc/h2mv.cu k_panelmv)."""
    import subprocess
    src = open(os.path.join(os.path.dirname(HEADER), "..", "paper_1810_08429_b200", "csrc", "h2mv.cu")).read()
    build_native.build()
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _native.LIB_PATH],
                          capture_output=True, text=True).stdout
    for kern, macro in (("k_panelmv", "GC_PAN_UNROLL"), ("k_panel_pair", "GC_PAIR_UNROLL")):
        unroll = int(re.search(r"#define %s (\d+)" % macro, src).group(1))
        for chain in ("0", "1"):
            body = re.search(r"Function : _ZN3gcb%d%sILb%sEEEvNS_10PanelPhaseE(.*?)(Function : |\Z)"
                             % (len(kern), kern, chain), sass, re.S)
            assert body, "%s<%s> not found" % (kern, chain)
            ops = re.findall(r"\b(LDG\.E\.EF\.64|DFMA)\b", body.group(1))
            first = ops.index("DFMA")
            assert first >= unroll, "%s<%s>: only %d streaming loads before the first DFMA" % (kern, chain, first)


def test_error_mapping():
    _native.load()
    with pytest.raises(Exception) as ei:
        # invalid configuration is rejected before touching the device
        _native.call("gc_green_factor", None, 0, 54, 1, None, None, None, None, None, None,
                     None, None, None)
    assert "null" in str(ei.value)


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1810_08429_b200 import assembly, geometry
    m = geometry.build_sphere_mesh(1)
    with pytest.raises(DeviceError):
        assembly.assemble_galerkin_block("slp", m, "constant", [0, 1], [2, 3])


def test_header_compiles_as_c_and_links(tmp_path):
    """include/gcb200.h is plain C: a C11 program including it links the
    library and calls the GPU-free entry points (tests/c/abi_smoke.c)."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib_dir = os.path.dirname(build_native.LIB)
    exe = str(tmp_path / "abi_smoke")
    subprocess.run([gcc, "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(root, "include"),
                    os.path.join(root, "tests", "c", "abi_smoke.c"), "-L", lib_dir, "-l:libgcb200.so",
                    "-Wl,-rpath," + lib_dir, "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "C ABI %d ok" % _native.ABI_VERSION in out.stdout


@pytest.mark.gpu
def test_c_program_drives_the_panel_kernel(tmp_path):
    """A C program (tests/c/panel_gpu.c) runs one panel product through
    gc_panelmv and through the native executor (gc_plan_*) with cudaMalloc'd
    buffers - the C-ABI alone, no Python on the product path."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    if gcc is None or not os.path.exists(os.path.join(cuda, "include", "cuda_runtime_api.h")):
        pytest.skip("no gcc / CUDA headers")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib_dir = os.path.dirname(build_native.LIB)
    exe = str(tmp_path / "panel_gpu")
    subprocess.run([gcc, "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(root, "include"),
                    "-I", os.path.join(cuda, "include"), os.path.join(root, "tests", "c", "panel_gpu.c"),
                    "-L", lib_dir, "-l:libgcb200.so", "-L", os.path.join(cuda, "lib64"), "-lcudart", "-lm",
                    "-Wl,-rpath," + lib_dir, "-Wl,-rpath," + os.path.join(cuda, "lib64"), "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "C-ABI panel product ok" in out.stdout
