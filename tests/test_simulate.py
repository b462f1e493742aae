"""The configs' inputs: the library's restatement of the reference generator
(dfpca_simulate, csrc/simulate.cu) against the reference's own generate()
(simulate.hpp:163-245, compiled unchanged in oracle/_ref), bit for bit, and
the digests the config goldens (tests/golden/cfg*.npz) were made on.
Host-only code of libdfpca_cuda.so: no device needed."""
import hashlib
from pathlib import Path

import numpy as np
import pytest

from paper_1510_04439_b200 import synth

GOLDEN = Path(__file__).resolve().parent / "golden"
KIND = {1: synth.SIM_SIM1, 2: synth.SIM_IMAGES2, 3: synth.SIM_IMAGES2, 4: synth.SIM_SPARSE2, 5: synth.SIM_SIM2}


@pytest.mark.parametrize("cfg,n,cells", [(1, 200, None), (1, 7, 30), (2, 40, None), (3, 5, None), (4, 500, None),
                                         (4, 50, 20), (5, 2, None), (5, 3, 10)])
def test_generator_matches_reference(ref, cfg, n, cells):
    sd = synth.config(cfg, n=n, cells=cells)
    off, c, v = ref.simulate(KIND[cfg], (sd.axes, sd.mask), n, 100 if cfg == 1 else 0, 20260815)
    assert np.array_equal(off, sd.offsets)
    assert np.array_equal(c.view(np.uint64), sd.coords.view(np.uint64))
    assert np.array_equal(v.view(np.uint64), sd.values.view(np.uint64))


def test_generator_other_seed(ref):
    ax = synth.midpoint_axis(12)
    sd = synth.simulate(synth.SIM_IMAGES2, [ax, ax], None, 9, 0.2, 0, seed=99)
    off, c, v = ref.simulate(synth.SIM_IMAGES2, ([ax, ax], None), 9, 0, 99)
    assert np.array_equal(off, sd.offsets)
    assert np.array_equal(v.view(np.uint64), sd.values.view(np.uint64))
    assert np.array_equal(c.view(np.uint64), sd.coords.view(np.uint64))


def test_sparse_design_shape():
    sd = synth.config(4, n=400)
    sizes = np.diff(sd.offsets)
    assert sizes.min() >= 5 and sizes.max() <= 20
    x, y = sd.coords[0::2], sd.coords[1::2]
    assert np.all(((x - 0.5) / 0.45) ** 2 + ((y - 0.5) / 0.3) ** 2 <= 1.0)


def test_invalid_model_is_rejected():
    with pytest.raises(ValueError):
        synth.simulate(7, [synth.midpoint_axis(4)], None, 3, 0.2)
    with pytest.raises(ValueError):  # sim1 needs points per sample
        synth.simulate(synth.SIM_SIM1, [synth.midpoint_axis(4)], None, 3, 0.2, 0)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg3w", "cfg4", "cfg5"])
def test_golden_inputs_are_the_generator_outputs(name):
    p = GOLDEN / f"{name}.npz"
    if not p.exists():
        pytest.skip(f"{p.name} not generated")
    z = np.load(p)
    sd = synth.config(int(z["cfg"]), n=int(z["n"]), h=float(z["h"][0]))
    h = hashlib.sha256()
    for a in (sd.offsets, sd.coords, sd.values):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest().encode() == bytes(z["input_digest"])
