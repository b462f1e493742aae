"""The C++ drop-in headers (include/dfpca/*.hpp): they compile against the
reference's API surface here (CPU), and the C++ suite cpp_tests/test_dropin.cpp
passes on the GPU through libdfpca_cuda.so."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "cpp_tests" / "test_dropin.cpp"
LIBDIR = ROOT / "paper_1510_04439_b200"


def json_include() -> list:
    """nlohmann's json.hpp (the reference's own io.hpp dependency), if present."""
    import glob
    import site
    for sp in site.getsitepackages():
        hit = glob.glob(sp + "/include/cudnn_frontend/thirdparty/nlohmann/json.hpp")
        if hit:
            return [f"-I{Path(hit[0]).parent}"]
    return []


def build(out: Path) -> Path:
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}", *json_include(), str(SRC),
           "-o", str(out), f"-L{LIBDIR}", "-ldfpca_cuda", f"-Wl,-rpath,{LIBDIR}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out


def test_dropin_headers_compile(tmp_path):
    build(tmp_path / "test_dropin")


@pytest.mark.gpu
def test_dropin_suite_passes_on_gpu(tmp_path):
    exe = build(tmp_path / "test_dropin")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    print(r.stderr)
    assert r.returncode == 0, r.stderr
    assert "0 failures" in r.stdout
