"""Exhaustive host check of the dynamic codec's code tables
(rsdb_dynamic_code_tables, the lookup adam8_dyn_kernel decides codes with):
for EVERY fp32 y in [-1, 1] (signed map, first moment) and [0, 1] (unsigned
map, second moment) the table lookup gives the oracle's code
(oracle/codemap.py dyn_code: nearest map value, ties to the lower code).
~5 min, numpy.  Output kept in profiles/r2/dyn_table_exhaustive.txt.  Test
infrastructure (imports the oracle); run: python tests/dyn_table_exhaustive.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import codemap as CM  # noqa: E402


def table_code(tab, y, signed):
    """The kernel's lookup (include/rsdb.h, rsdb_dynamic_code_tables), replayed."""
    mb = 6 if signed else 7
    sh = 23 - mb
    low = np.uint32((1 << sh) - 1)
    b = np.ascontiguousarray(y, np.float32).view(np.uint32)
    mag = b & np.uint32(0x7FFFFFFF)
    idx = np.maximum((mag >> np.uint32(sh)).astype(np.int64) - (100 << mb), 0)
    yl = mag & low
    if signed:
        sgn = (b >> np.uint32(31)).astype(np.int64)
        idx = idx + sgn * (28 << mb)
        yl = np.where(sgn == 1, low - yl, yl)
    e = tab[idx]
    return ((e >> np.uint32(24)) + (yl >= (e & np.uint32(0xFFFFFF)))).astype(np.uint8)


def check(tab, signed, neg):
    bad = n = 0
    one = 0x3F800000
    step = 1 << 24
    for s in range(0, one + 1, step):
        a = np.arange(s, min(s + step, one + 1), dtype=np.uint32).view(np.float32)
        y = -a if neg else a
        ok = table_code(tab, y, signed) == CM.dyn_code(y, signed)
        bad += int((~ok).sum())
        n += a.size
        if (~ok).any():
            print("BAD", signed, neg, y[np.nonzero(~ok)[0][:3]], flush=True)
    print("signed" if signed else "unsigned", "neg" if neg else "pos", n, "bad", bad, flush=True)
    return bad


if __name__ == "__main__":
    import paper_2602_22437_b200 as R
    tm, tv = (np.array(t, np.uint32) for t in R.dynamic_code_tables())
    t0 = time.time()
    bad = check(tm, True, False) + check(tm, True, True) + check(tv, False, False)
    print("time", time.time() - t0, "bad", bad)
    sys.exit(1 if bad else 0)
