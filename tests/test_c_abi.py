"""The boundary is plain C: examples/c_abi_demo.c includes include/gtb200.h,
links libgtb200.so and runs the path without Python (build -> export ->
PageRank -> triangles) against the reference's known answers."""

import os
import subprocess
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
LIB_DIR = REPO / "paper_1503_07881_b200"


def _compile(tmp_path) -> Path:
    exe = tmp_path / "c_abi_demo"
    cmd = ["gcc", "-std=c99", "-Wall", "-Werror", str(REPO / "examples" / "c_abi_demo.c"),
           f"-I{REPO / 'include'}", f"-L{LIB_DIR}", "-lgtb200", f"-Wl,-rpath,{LIB_DIR}",
           "-lm", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_header_is_c_and_links(tmp_path):
    if not (LIB_DIR / "libgtb200.so").exists():
        pytest.skip("libgtb200.so not built")
    assert _compile(tmp_path).exists()


@pytest.mark.gpu
def test_c_program_runs_the_path(tmp_path):
    exe = _compile(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120,
                         env=dict(os.environ))
    assert out.returncode == 0, out.stdout + out.stderr
    assert "c abi demo ok" in out.stdout
    assert "triangles 4" in out.stdout
