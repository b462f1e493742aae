"""TEST HARNESS build: the reference's fit_pipeline driver (pipeline_run.cpp)
compiled (a) against this repository's drop-in headers first -- the GPU path
through libdfpca_cuda.so -- and (b) against the reference alone.  Needs the
reference sources (build container only); __graft_entry__.build() calls it,
the binaries land in tests/cpp/_bin/ (git-ignored, shipped with the tree)."""
import glob
import os
import site
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
REF_INC = Path("/root/reference/proj/include")
OUT = ROOT / "tests" / "cpp" / "_bin"


def json_dir():
    for sp in site.getsitepackages():
        hit = glob.glob(sp + "/include/cudnn_frontend/thirdparty/nlohmann/json.hpp")
        if hit:
            return str(Path(hit[0]).parent)
    return None


def openblas():
    import scipy
    libs = sorted(glob.glob(os.path.join(os.path.dirname(scipy.__file__) + ".libs", "libscipy_openblas*.so")))
    return libs[0] if libs else ""


SUITES = ["test_core", "test_fft_smoother", "test_eigensolve", "test_scores", "test_bandwidth", "test_smoother",
          "test_simulate", "test_io_pipeline", "acceptance"]


def build_suites(force=False, jobs=8):
    """The reference's own Catch2 suites (/root/reference/proj/tests), compiled
    unchanged against the Catch2 stand-in (tests/cpp/catch2): dropin_<suite>
    (drop-in headers first, GPU) and ref_<suite> (the reference alone)."""
    import concurrent.futures as cf
    ref_tests = REF_INC.parent / "tests"
    if not ref_tests.is_dir() or json_dir() is None:
        return False
    OUT.mkdir(parents=True, exist_ok=True)
    lib = ROOT / "paper_1510_04439_b200"
    shim_main = ROOT / "tests" / "cpp" / "catch2" / "shim_main.cpp"
    base = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-DDFPCA_USE_EIGEN"]
    tail = [f"-I{ROOT / 'oracle' / 'shim'}", f"-I{json_dir()}", f"-I{ROOT / 'tests' / 'cpp'}",
            str(shim_main), str(ROOT / "oracle" / "shim" / "lapack_loader.cpp"),
            f'-DDFPCA_OPENBLAS_PATH="{openblas()}"', "-ldl", "-pthread"]
    jobs_list = []
    for suite in SUITES:
        src = ref_tests / f"{suite}.cpp"
        for variant in ("dropin", "ref"):
            out = OUT / f"{variant}_{suite}"
            if not force and out.exists() and out.stat().st_mtime >= src.stat().st_mtime:
                continue
            inc = [f"-I{ROOT / 'include'}", f"-I{REF_INC}"] if variant == "dropin" else [f"-I{REF_INC}"]
            link = [f"-L{lib}", "-ldfpca_cuda", f"-Wl,-rpath,{lib}"] if variant == "dropin" else []
            t = [x for x in tail if x != str(shim_main)] if suite == "acceptance" else tail  # has its own main()
            jobs_list.append(base + inc + [str(src)] + t + link + ["-o", str(out)])
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        for r in ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs_list):
            if r.returncode != 0:
                raise RuntimeError(r.stderr[-2000:])
    return True


def build(force=False):
    if not (REF_INC / "dfpca").is_dir() or json_dir() is None:
        return False
    OUT.mkdir(parents=True, exist_ok=True)
    src = ROOT / "tests" / "cpp" / "pipeline_run.cpp"
    common = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", f"-I{ROOT / 'oracle' / 'shim'}", f"-I{json_dir()}",
              str(src), str(ROOT / "oracle" / "shim" / "lapack_loader.cpp"),
              f'-DDFPCA_OPENBLAS_PATH="{openblas()}"', "-ldl", "-pthread"]
    lib = ROOT / "paper_1510_04439_b200"
    targets = {
        "pipeline_dropin": [f"-I{ROOT / 'include'}", f"-I{REF_INC}", f"-L{lib}", "-ldfpca_cuda", f"-Wl,-rpath,{lib}"],
        "pipeline_ref": [f"-I{REF_INC}"],
    }
    for name, extra in targets.items():
        out = OUT / name
        if force or not out.exists() or out.stat().st_mtime < src.stat().st_mtime:
            subprocess.run(common[:1] + extra[:2] + common[1:] + extra[2:] + ["-o", str(out)], check=True)
    return True


if __name__ == "__main__":
    print(build(force="--force" in sys.argv), build_suites(force="--force" in sys.argv))
