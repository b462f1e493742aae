"""Long-format table corpora for the io.hpp parity tests (test_io.py,
test_gpu_io.py): every case is file CONTENT (bytes) that the reference's
read_long_format (io.hpp:115-155) either reads or rejects with a message."""
import numpy as np

TOKENS_OK = ["1.5", "-0", "+2", ".5", "5.", "1e-5", "1E+05", "0x1.8p3", "-0X1P-3", "inf", "-Infinity", "nan",
             "-nan", "NaN(123)", "nan(0x8)", "nan(abc)", "nan()", " 7.25", "\f3", "\v 4", "2.2250738585072013e-308",
             "1.7976931348623158e308", "4503599627370496.5", "0.000000000000000000000000000000000000000000001e300",
             "100000000000000000000000000000000000000e-20", "123456789012345678901234567890",
             "0x1.fffffffffffff7p1023", "0X1P-1074"]
TOKENS_BAD = ["", "1.5 ", "abc", "1e", "1e+", "0x", "0x.p1", "1_0", "infin", "nan(1", "nan(-1)", "--1",
              "2.2250738585072012e-308", "1e309", "1e-400", "0x1p-1075", "nan(99999999999999999999)", "1,5"]


def fmt17(v: float) -> str:
    return "%.17g" % v


def random_table(rng, n_samples=20, max_obs=12, dim=2, delim="\t", crlf=False, blank_every=0, interleave=False,
                 id_style="plain", header=None, fmt=fmt17):
    ids = []
    for i in range(n_samples):
        if id_style == "plain":
            ids.append("s%d" % i)
        elif id_style == "long":
            ids.append("subject-%04d-%s" % (i, "x" * int(rng.integers(0, 20))))
        elif id_style == "unicode":
            ids.append("sujet_é%d" % i)
        else:  # numeric ids with shared prefixes of different lengths
            ids.append(str(int(rng.integers(0, 10 ** int(rng.integers(1, 12))))) + "_%d" % i)
    rows = []
    for i, sid in enumerate(ids):
        for _ in range(int(rng.integers(1, max_obs + 1))):
            vals = list(rng.random(dim)) + [float(rng.standard_normal())]
            rows.append((sid, vals))
    if interleave:
        rng.shuffle(rows)
    sep = " " * 3 if delim == " " else delim
    hdr = header if header is not None else sep.join(["id"] + ["t%d" % (k + 1) for k in range(dim)] + ["y"])
    eol = "\r\n" if crlf else "\n"
    out = [hdr]
    for j, (sid, vals) in enumerate(rows):
        out.append(sep.join([sid] + [fmt(v) for v in vals]))
        if blank_every and j % blank_every == 0:
            out.append("")
    return (eol.join(out) + eol).encode("utf-8")


def token_table(tokens, dim=1):
    """One observation per token (in the value column), ids cycling over 3."""
    lines = ["id\tt\ty"]
    for j, t in enumerate(tokens):
        lines.append("s%d\t%s\t%s" % (j % 3, fmt17(j / max(1, len(tokens))), t))
    return ("\n".join(lines) + "\n").encode()


def valid_cases():
    rng = np.random.default_rng(20261018)
    cases = {
        "tab_2d": random_table(rng),
        "comma_1d": random_table(rng, dim=1, delim=","),
        "semicolon_3d": random_table(rng, dim=3, delim=";"),
        "blanks_2d": random_table(rng, delim=" "),
        "crlf_blank_lines": random_table(rng, crlf=True, blank_every=4),
        "interleaved_ids": random_table(rng, n_samples=50, interleave=True),
        "long_ids": random_table(rng, n_samples=40, id_style="long", interleave=True),
        "numeric_ids": random_table(rng, n_samples=60, id_style="numeric", interleave=True),
        "unicode_ids": random_table(rng, id_style="unicode"),
        "short_formats": random_table(rng, fmt=lambda v: "%.3g" % v),
        "hex_floats": random_table(rng, fmt=lambda v: float(v).hex()),
        "tokens_ok": token_table(TOKENS_OK),
        "no_trailing_newline": random_table(rng).rstrip(b"\n"),
        "single_row": b"id,t,y\nA,0.5,1\n",
        "extra_header_fields_ws": b"  id   t1   t2   y  \n a 1 2 3\n\n b 4 5 6 \n a 7 8 9\n",
        "empty_fields_not_used": b"id,t,y\n,0.25,1\n,0.5,2\nx,1,3\n",
    }
    return cases


def error_cases():
    ok = "id\tt\ty\ns1\t0.1\t1\ns1\t0.2\t2\n"
    cases = {
        "empty_file": b"",
        "header_only": b"id\tt\ty\n",
        "header_blank_lines": b"id\tt\ty\n\n\r\n\n",
        "short_header": b"id\ty\ns\t1\n",
        "blank_header": b"\nid\tt\ty\n",
        "field_count": (ok + "s2\t0.3\n" + "s2\tzz\t1\n").encode(),
        "bad_coordinate": (ok + "s2\tzz\t1\n").encode(),
        "bad_value_after_bad_count": (ok + "s2\t0.1\tq\n" + "s3\t0.1\n").encode(),
        "count_and_number_same_line": (ok + "s2\tzz\t1\t5\n").encode(),
        "range_error": (ok + "s2\t0.3\t1e999\n").encode(),
        "trailing_space": (ok + "s2\t0.3\t1.0 \n").encode(),
        "crlf_field_count": b"id,t,y\r\na,1,2\r\nb,1\r\n",
    }
    for j, t in enumerate(TOKENS_BAD):
        cases["bad_token_%d" % j] = token_table(["1.0", t, "2.0"])
    return cases
