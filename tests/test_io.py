"""SURVEY.md 8(f) rank 2 on the CPU: the exact number parser of the GPU
table reader (csrc/numparse.cuh, compiled here for the host) against glibc
strtod under the reference's acceptance rule (io.hpp:39-46), and the host
writers / grid-file reader against the reference's io.hpp (oracle/_ref)."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from io_corpus import error_cases, valid_cases

ROOT = Path(__file__).resolve().parent.parent


def test_number_parser_matches_strtod(tmp_path):
    exe = tmp_path / "numparse_check"
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-Werror",
                    f"-I{ROOT / 'paper_1510_04439_b200' / 'csrc'}", str(ROOT / "tests" / "cpp" / "numparse_check.cpp"),
                    "-o", str(exe)], check=True, capture_output=True, text=True)
    r = subprocess.run([str(exe), "20000"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout
    assert " 0 mismatches" in r.stdout
    n_exact = int(r.stdout.split("(")[1].split()[0])
    assert n_exact > 1000  # the big-integer halfway comparison was exercised


def test_corpus_is_pinned_by_reference(ref, tmp_path):
    """Every valid case reads and every error case raises in the reference."""
    for name, data in valid_cases().items():
        p = tmp_path / f"{name}.tsv"
        p.write_bytes(data)
        dim, off, coords, values, ids = ref.read_long_format(p)
        assert off[-1] == values.size > 0, name
    for name, data in error_cases().items():
        p = tmp_path / f"{name}.tsv"
        p.write_bytes(data)
        with pytest.raises(ref.RefError) as e:
            ref.read_long_format(p)
        assert e.value.name() == "ParseError", (name, str(e.value))


def test_write_long_format_bytes_match_reference(ref, tmp_path):
    from paper_1510_04439_b200 import api
    rng = np.random.default_rng(5)
    off = np.array([0, 3, 3, 7, 8], dtype=np.int64)
    coords = np.concatenate([rng.standard_normal(16), [0.1, -0.0, 1e-300, 5e-324]])
    values = np.concatenate([rng.standard_normal(6), [np.inf, -1e308]])
    ids = ["a", "bb", "ccc", "d d"]
    data = api.FunctionalDataset.from_csr(2, off, coords, values, ids)
    api.write_long_format(str(tmp_path / "ours.tsv"), data)
    ref.write_long_format(tmp_path / "ref.tsv", 2, off, coords, values, ids)
    assert (tmp_path / "ours.tsv").read_bytes() == (tmp_path / "ref.tsv").read_bytes()


def test_grid_files_match_reference(ref, tmp_path):
    from paper_1510_04439_b200 import api
    ax = [np.linspace(0.0, 1.0, 7), np.linspace(-2.0, 3.0, 5) ** 3]
    mask = (np.arange(35) % 3 != 0).astype(np.uint8)
    for m in (None, mask):
        g = api.EvaluationGrid(ax, m)
        api.write_grid(str(tmp_path / "ours.txt"), g)
        ref.write_grid(tmp_path / "ref.txt", (ax, m))
        assert (tmp_path / "ours.txt").read_bytes() == (tmp_path / "ref.txt").read_bytes()
        back = api.read_grid(str(tmp_path / "ref.txt"))
        raxes, rmask = ref.read_grid(tmp_path / "ours.txt")
        for k in range(2):
            assert np.array_equal(back.axis(k), raxes[k])
        assert (back.mask() is None) == (rmask is None)
        if rmask is not None:
            assert np.array_equal(back.mask(), rmask)
    bad = {"magic": "grid v1\n", "version": "dfpca-grid v2\n", "dim": "dfpca-grid v1\ndim 0\n",
           "axis": "dfpca-grid v1\ndim 1\naxis 1 3 0 1 2\n", "short": "dfpca-grid v1\ndim 1\naxis 0 3 0 1\n",
           "record": "dfpca-grid v1\ndim 1\nfoo\n", "nodim": "dfpca-grid v1\n",
           "noaxis": "dfpca-grid v1\ndim 2\naxis 0 2 0 1\n", "number": "dfpca-grid v1\ndim 1\naxis 0 2 0 x\n",
           "masklen": "dfpca-grid v1\ndim 1\naxis 0 2 0 1\nmask 101\n",
           "maskbits": "dfpca-grid v1\ndim 1\naxis 0 2 0 1\nmask 12\n", "empty": ""}
    for name, text in bad.items():
        p = tmp_path / f"bad_{name}.txt"
        p.write_text(text)
        with pytest.raises(ref.RefError) as r:
            ref.read_grid(p)
        with pytest.raises(api.Error) as o:
            api.read_grid(str(p))
        assert o.value.name() == r.value.name(), name
        assert str(r.value) == "%s: %s" % (o.value.name(), o.value.message), name
