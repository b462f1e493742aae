"""CPU tests (no GPU): the C-ABI library builds, loads and exports exactly the
entry points include/dfpca_cuda.h declares; host-side logic of the Python
mirror (grids, bandwidths, block plans, error taxonomy) behaves like the
reference's."""
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "dfpca_cuda.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"DFPCA_API\s+\w+\s+(dfpca_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("dfpca_linear_bin", "dfpca_local_linear", "dfpca_covariance", "dfpca_randomized_eig",
              "dfpca_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_1510_04439_b200 import _lib
    lib = _lib.load()  # no device needed to load
    for s in declared_symbols():
        assert hasattr(lib, s), s
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert bound == set(declared_symbols()), "ctypes prototypes out of sync with the header"


def test_exported_symbols_match_nm():
    import subprocess
    so = ROOT / "paper_1510_04439_b200" / "libdfpca_cuda.so"
    out = subprocess.run(["nm", "-D", "--defined-only", str(so)], capture_output=True, text=True).stdout
    exported = sorted(set(re.findall(r" T (dfpca_\w+)", out)))
    assert exported == declared_symbols()


def test_no_device_is_a_loud_error(monkeypatch):
    """The product path has no CPU fallback: without a device the context
    creation fails loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1510_04439_b200 import _lib
    monkeypatch.setattr(_lib, "_ctx", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.ctx()


def test_grid_construction_and_spacing():
    from paper_1510_04439_b200 import api
    g = api.EvaluationGrid.midpoint([0.0, 0.0], [1.0, 2.0], [4, 8])
    assert g.shape() == [4, 8] and g.size() == 32 and g.equispaced()
    assert abs(g.spacing(1) - 0.25) < 1e-15 and abs(g.cell_volume() - 0.0625) < 1e-15
    u = api.EvaluationGrid.uniform([0.0], [1.0], [5])
    assert u.axis(0)[-1] == 1.0
    uneven = api.EvaluationGrid([[0.0, 0.1, 0.25, 0.6, 1.0]])
    assert not uneven.equispaced()
    with pytest.raises(api.Error) as e:
        api.EvaluationGrid([[0.0, 0.0, 1.0]])
    assert e.value.name() == "InvalidArgument"
    with pytest.raises(api.Error) as e:
        api.EvaluationGrid.uniform([0.0], [0.0], [3])
    assert e.value.name() == "DegenerateAxis"


def test_bandwidth_validation():
    from paper_1510_04439_b200 import api
    g = api.EvaluationGrid.uniform([0.0], [1.0], [11])
    api.Bandwidth([0.5]).validate(g)
    for bad in ([0.0], [-1.0], [1.5], [0.1, 0.1]):
        with pytest.raises(api.Error) as e:
            api.Bandwidth(bad).validate(g)
        assert e.value.name() == "InvalidBandwidth"


def test_block_plans_mirror_reference():
    """fft_smoother.hpp:66-145 semantics (tests/test_fft_smoother.cpp:321-366)."""
    from paper_1510_04439_b200 import api
    g = api.EvaluationGrid.uniform([0.0], [1.0], [101])
    h = api.Bandwidth([0.2])  # radius 20 nodes
    one = api.single_block_plan(g, h)
    assert one.halo == [20] and one.blocks[0].lo == [0] and one.blocks[0].hi == [101]
    four = api.make_block_plan(g, h, 4)
    api.validate_block_plan(four, g, h)
    cores = [four.core(b, g.shape()) for b in range(4)]
    assert sum(c.volume() for c in cores) == 101
    short = api.make_block_plan(g, h, 2)
    short.halo[0] -= 1
    with pytest.raises(api.Error) as e:
        api.validate_block_plan(short, g, h)
    assert e.value.name() == "HaloTooSmall"
    with pytest.raises(api.Error) as e:
        api.validate_block_plan(api.make_block_plan(g, h, 6), g, h)
    assert e.value.name() == "BlockTooSmall"
    with pytest.raises(api.Error) as e:
        api.make_block_plan(g, h, 0)
    assert e.value.name() == "InvalidArgument"


def test_error_taxonomy():
    from paper_1510_04439_b200 import api
    e = api.Error(api.ErrorClass.Config, "HaloTooSmall", "x")
    assert str(e) == "HaloTooSmall: x" and e.exit_code() == 3 and e.name() == "HaloTooSmall"


def test_dataset_csr_roundtrip():
    from paper_1510_04439_b200 import api, synth
    sd = synth.random_points(2, 9, 5, 7, 0.3)
    ds = sd.dataset()
    off, c, v = ds.csr()
    assert np.array_equal(off, sd.offsets) and np.array_equal(c, sd.coords) and ds.n_obs() == 35
    ds2 = api.FunctionalDataset(2, list(ds.samples))
    off2, c2, v2 = ds2.csr()
    assert np.array_equal(off2, off) and np.array_equal(c2, c) and np.array_equal(v2, v)


def test_default_sketch_and_fve():
    from paper_1510_04439_b200 import api
    assert api.default_sketch_size(3, 1000) == 99
    assert api.default_sketch_size(60, 1000) == 130
    assert api.default_sketch_size(3, 40) == 40
    es = api.EigenSystem([4.0, 1.0, 0.5], [], [0.72, 0.9, 1.0], 5.5)
    assert api.select_components_fve(es, 0.9) == 2
    assert api.select_components_fve(es, 0.95) == 3
    with pytest.raises(api.Error):
        api.select_components_fve(es, 0.0)
