"""The C++ drop-in (namespace bytecodec, include/bytecodec/*.hpp) as a reference
caller would use it: compiled here against the headers and libbytecodec_b200.so,
run on the GPU box."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "test_bytecodec_api.cpp"
BIN = ROOT / "build" / "test_bytecodec_api"
LIBDIR = ROOT / "paper_1709_08990_b200" / "lib"


def _build() -> Path:
    BIN.parent.mkdir(exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-I", str(ROOT / "include"), str(SRC), "-L", str(LIBDIR),
                    "-lbytecodec_b200", f"-Wl,-rpath,{LIBDIR}", "-o", str(BIN)], check=True)
    return BIN


def test_cpp_api_links():
    """CPU suite: the reference-shaped C++ caller compiles and links against the library."""
    assert _build().exists()


@pytest.mark.gpu
def test_cpp_api_runs_on_gpu():
    out = subprocess.run([str(_build())], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr + out.stdout
    assert "all checks passed" in out.stdout
