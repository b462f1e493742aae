"""GPU parity of SURVEY.md 8(f) rank 2 -- the long-format table reader
(io.hpp:115-155) parsed on the device -- against the reference's own
read_long_format (oracle/_ref).  Bar: identical sample order, ids and CSR
offsets; coordinates and values bit-identical (NaN payloads included);
rejected files rejected with the same error name and message."""
import numpy as np
import pytest

from io_corpus import error_cases, random_table, valid_cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_1510_04439_b200 import api as A
    return A


def _same(ds, want):
    dim, off, coords, values, ids = want
    got_off, got_coords, got_values = ds.csr()
    assert ds.dim == dim
    assert np.array_equal(got_off, off)
    assert np.array_equal(got_coords.view(np.uint64), coords.view(np.uint64))
    assert np.array_equal(got_values.view(np.uint64), values.view(np.uint64))
    assert [s.id.encode("utf-8", "surrogateescape") for s in ds.samples] == ids


@pytest.mark.parametrize("name", list(valid_cases()))
def test_table_matches_reference(api, ref, tmp_path, name):
    data = valid_cases()[name]
    p = tmp_path / f"{name}.tsv"
    p.write_bytes(data)
    want = ref.read_long_format(p)
    _same(api.read_long_format(str(p)), want)
    _same(api.parse_long_format(data), want)


@pytest.mark.parametrize("name", list(error_cases()))
def test_errors_match_reference(api, ref, tmp_path, name):
    p = tmp_path / f"{name}.tsv"
    p.write_bytes(error_cases()[name])
    with pytest.raises(ref.RefError) as r:
        ref.read_long_format(p)
    with pytest.raises(api.Error) as o:
        api.read_long_format(str(p))
    assert str(o.value) == str(r.value)


def test_missing_file(api, ref, tmp_path):
    p = tmp_path / "absent.tsv"
    with pytest.raises(ref.RefError) as r:
        ref.read_long_format(p)
    with pytest.raises(api.Error) as o:
        api.read_long_format(str(p))
    assert str(o.value) == str(r.value) and o.value.name() == "IoError"


def test_large_interleaved_table(api, ref, tmp_path):
    """~300k rows over 2000 interleaved samples, several upload chunks."""
    rng = np.random.default_rng(11)
    data = random_table(rng, n_samples=2000, max_obs=300, dim=2, interleave=True, id_style="long")
    assert len(data) > 2 * (8 << 20)
    p = tmp_path / "big.tsv"
    p.write_bytes(data)
    _same(api.read_long_format(str(p)), ref.read_long_format(p))


def test_decimal_token_fuzz(api, ref, tmp_path):
    """The register fast path for plain decimals (k_parse_fields) and the
    general parser it falls back to, on 60k valid tokens of many shapes:
    every value bit-equal to the reference's strtod."""
    rng = np.random.default_rng(3)
    toks = []
    for _ in range(60000):
        v = float(rng.standard_normal() * 10.0 ** rng.integers(-30, 30))
        kind = rng.integers(0, 9)
        if kind == 0:
            t = "%.17g" % v
        elif kind == 1:
            t = "%.*e" % (int(rng.integers(0, 22)), v)
        elif kind == 2:
            t = "%.*f" % (int(rng.integers(0, 12)), v / 10.0 ** rng.integers(0, 25))
        elif kind == 3:
            t = "0" * int(rng.integers(1, 6)) + "%d.%d" % (rng.integers(0, 10 ** 6), rng.integers(0, 10 ** 9))
        elif kind == 4:
            t = "+%.*g" % (int(rng.integers(1, 20)), abs(v))
        elif kind == 5:
            t = "%d." % rng.integers(0, 10 ** 15)
        elif kind == 6:
            t = ".%0*d" % (int(rng.integers(1, 25)), rng.integers(0, 10 ** 12))
        elif kind == 7:
            t = "%dE%+d" % (rng.integers(1, 10 ** 18), rng.integers(-300, 290))
        else:
            t = "".join(rng.choice(list("0123456789"), int(rng.integers(15, 24)))) + "e-" + str(rng.integers(0, 40))
        toks.append(t)
    lines = ["id\tt\ty"] + ["s%d\t%s\t%s" % (j % 7, toks[j], toks[-1 - j]) for j in range(len(toks))]
    p = tmp_path / "fuzz.tsv"
    p.write_text("\n".join(lines) + "\n")
    _same(api.read_long_format(str(p)), ref.read_long_format(p))


def test_round_trip_through_writer(api, tmp_path):
    from paper_1510_04439_b200 import synth
    sd = synth.sparse_masked(24, 300, 0.3)
    ds = sd.dataset()
    p = tmp_path / "rt.tsv"
    api.write_long_format(str(p), ds)
    back = api.read_long_format(str(p))
    a, b = ds.csr(), back.csr()
    for x, y in zip(a, b):
        assert np.array_equal(np.asarray(x).view(np.uint64) if x.dtype == np.float64 else x,
                              np.asarray(y).view(np.uint64) if y.dtype == np.float64 else y)
    assert [s.id for s in back.samples] == [s.id for s in ds.samples]


@pytest.mark.parametrize("case", ["nodes_2d", "random_2d", "random_1d", "masked"])
def test_bin_long_format_equals_host_round_trip(api, tmp_path, case):
    """bin_long_format (table parsed and binned on the device) == linear_bin
    of read_long_format's dataset, every BinnedData field bit for bit."""
    from paper_1510_04439_b200 import synth
    sd = {"nodes_2d": lambda: synth.grid_nodes(2, 12, 40, 0.2),
          "random_2d": lambda: synth.random_points(2, 13, 60, 25, 0.3),
          "random_1d": lambda: synth.random_points(1, 41, 30, 15, 0.15),
          "masked": lambda: synth.sparse_masked(20, 80, 0.2)}[case]()
    p = tmp_path / "t.tsv"
    p.write_bytes(synth.long_format_bytes(sd))
    grid = sd.grid()
    opt = api.BinOptions(True, True)
    a = api.linear_bin(api.read_long_format(str(p)), grid, opt)
    b, ids = api.bin_long_format(str(p), grid, opt)
    assert ids == ["s%d" % i for i in range(len(ids))]
    for f in ("mass", "wvalue", "wsquare", "diag_mass", "diag_value"):
        assert np.array_equal(np.asarray(getattr(a, f)).view(np.uint64), np.asarray(getattr(b, f)).view(np.uint64)), f
    assert a.sample_sizes == b.sample_sizes
    for x, y in zip(a.per_sample, b.per_sample):
        assert x.sample_index == y.sample_index and x.pair_weight == y.pair_weight
        assert np.array_equal(x.mass.view(np.uint64), y.mass.view(np.uint64))
        assert np.array_equal(x.value.view(np.uint64), y.value.view(np.uint64))


def test_bin_long_format_outside_observation(api, tmp_path):
    p = tmp_path / "bad.tsv"
    p.write_bytes(b"id\tt\ty\na\t0.5\t1\nbad id\t0.2\t1\nbad id\t1.5\t2\n")
    grid = api.EvaluationGrid.uniform([0.0], [1.0], [5])
    with pytest.raises(api.Error) as e:
        api.bin_long_format(str(p), grid)
    assert e.value.name() == "ObservationOutsideGrid"
    assert "'bad id' observation 1" in str(e.value)
