"""The C-ABI library: built for sm_100a, loads, exports every declared symbol.
No compute calls (CPU container)."""

import re
import shutil
import subprocess

import pytest

from paper_1503_07881_b200 import _native
from paper_1503_07881_b200._build import LIB_PATH, REPO, build_native


@pytest.fixture(scope="module")
def lib():
    build_native()
    return _native.load()


def declared_symbols():
    text = (REPO / "include" / "gtb200.h").read_text()
    return set(re.findall(r"^GT_API [^\n(]*?\b(gt_\w+)\(", text, flags=re.M))


def test_header_declares_the_path(lib):
    names = declared_symbols()
    for must in ("gt_build_csr", "gt_pagerank", "gt_triangles", "gt_graph_export",
                 "gt_graph_free", "gt_last_error", "gt_init"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), f"{name} missing from {LIB_PATH.name}"


def test_binding_covers_header_exactly():
    assert set(_native.SIGNATURES) == declared_symbols()


def test_no_other_exported_gt_symbols(lib):
    nm = shutil.which("nm")
    if nm is None:
        pytest.skip("nm not available")
    out = subprocess.run([nm, "-D", "--defined-only", str(LIB_PATH)], capture_output=True,
                         text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T gt_" in ln}
    assert exported == declared_symbols()


def test_cubin_targets_sm100a(lib):
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([tool, "--list-elf", str(LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_\d+a?", out.stdout))
    assert arches == {"sm_100a"}, arches


def test_init_without_gpu_fails_loudly(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    rc = lib.gt_init(0)
    assert rc == _native.GT_ENODEV
    assert b"no CUDA device" in lib.gt_last_error()
    assert lib.gt_version().startswith(b"gtb200")
