"""Long-format reader timing on the cfg-3 table:
d = 2, 64^2 nodes, n = 2000 subjects -> 8.19 M observation rows written with
the reference's format (tab, %.17g).  Times read_long_format through the
C-ABI (file -> device -> host CSR) and its device stages."""
import argparse
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1510_04439_b200 import _lib, api  # noqa: E402


def make_table(path, n=2000, cells=64, seed=7):
    rng = np.random.default_rng(seed)
    ax = (np.arange(cells) + 0.5) / cells
    t1, t2 = np.meshgrid(ax, ax, indexing="ij")
    pts = np.stack([t1.ravel(), t2.ravel()], 1)
    col = np.char.mod("%.17g", pts)
    coord_txt = np.char.add(np.char.add(col[:, 0], "\t"), col[:, 1])
    with open(path, "w") as f:
        f.write("sample_id\tt1\tt2\ty\n")
        for i in range(n):
            y = np.char.mod("%.17g", rng.standard_normal(pts.shape[0]))
            rows = np.char.add(np.char.add(np.char.add("s%d\t" % i, coord_txt), "\t"), y)
            f.write("\n".join(rows.tolist()))
            f.write("\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2000)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    d = Path(tempfile.mkdtemp())
    p = d / "cfg3.tsv"
    t0 = time.perf_counter()
    make_table(p, n=args.n)
    size = p.stat().st_size
    print(f"wrote {size / 1e6:.1f} MB in {time.perf_counter() - t0:.1f} s", flush=True)
    ds = api.read_long_format(str(p))  # warm-up (pinned slots, pool)
    rows = ds.n_obs()
    times = []
    import ctypes as C
    L = _lib.lib()
    for _ in range(args.reps):
        t0 = time.perf_counter()
        h = C.c_void_p()
        _lib.check(L.dfpca_read_long_format(_lib.ctx(), str(p).encode(), C.byref(h)))
        t1 = time.perf_counter()
        st = {k: _lib.stage_ms(k) for k in ("upload", "lines", "parse", "group", "scatter", "total")}
        ds = api._table_to_dataset(h)
        t2 = time.perf_counter()
        times.append(t2 - t0)
        st["copy_out_wall"] = 1e3 * (t2 - t1)
    med = float(np.median(times))
    print(f"rows {rows}  read_long_format median {med * 1e3:.1f} ms  ({rows / med / 1e6:.1f} M rows/s, "
          f"{size / med / 1e9:.2f} GB/s)  all {[round(t * 1e3, 1) for t in times]}")
    print("stages (ms, last rep):", {k: round(v, 2) for k, v in st.items()})
    raw = p.read_bytes()
    t0 = time.perf_counter()
    api.parse_long_format(raw)
    print(f"parse_long_format (bytes in memory) {1e3 * (time.perf_counter() - t0):.1f} ms")
    os.unlink(p)


if __name__ == "__main__":
    main()
