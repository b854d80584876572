"""Write the rows of one flush of a BASELINE stream as a binary CSR for tools/spmm_bench.

  python tools/dump_flush.py <config> <out.bin> [flush_index]

Layout: int64 m, int64 d, int64 nnz, int64 ell, then int64 row_ptr[m+1], uint32 cols[nnz],
float64 vals[nnz]. Every flush of the five configs holds m = d rows (row trigger).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1602_00412_b200 import synthetic as S  # noqa: E402


def main():
    name, out = sys.argv[1], sys.argv[2]
    f = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    cfg = S.CONFIGS[name]
    rp, cs, vs = S.generate(name, (f * cfg.d, (f + 1) * cfg.d))
    m = rp.size - 1
    with open(out, "wb") as fh:
        np.array([m, cfg.d, int(rp[-1]), cfg.ell], np.int64).tofile(fh)
        rp.astype(np.int64).tofile(fh)
        cs.astype(np.uint32).tofile(fh)
        vs.astype(np.float64).tofile(fh)
    print(f"{name} flush {f}: m={m} d={cfg.d} nnz={int(rp[-1])} -> {out}")


if __name__ == "__main__":
    main()
