#!/usr/bin/env python
"""Generates tests/golden/config5_checksums.json: the expected checksum (sum
of fp64 bit patterns mod 2^64) of y after ONE pass of the config-4/5 region
over elements [0, n) with the bench's counter-based inputs (x seed
0x5eed01ab, y seed 0x5eed01ac, c_k = k/8), computed by the C oracle
(orc_stream_checksum, which equals orc_fill + orc_stream + orc_checksum over
the range -- tests/test_oracle_golden.py checks that identity).  bench.py
compares the all-reduced checksum of every run against this table, at every
GPU count (the element-range shards gather to the whole range).

    python tests/golden/make_config5_checksums.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

SEED_X, SEED_Y = 0x5EED01AB, 0x5EED01AC
COEF = [k / 8 for k in range(1, 9)]
SIZES = [1 << 20, 1 << 22, 1 << 24, 1 << 26, 1 << 28, 1 << 29, 1 << 31]


def main():
    cf = np.array(COEF)
    out = {"seed_x": SEED_X, "seed_y": SEED_Y, "coef": COEF, "elem": "f64",
           "generator": "oracle/ompds_oracle.c orc_stream_checksum", "checksums": {}}
    for n in SIZES:
        out["checksums"][str(n)] = "%#018x" % O.lib().orc_stream_checksum(
            1, 0, n, SEED_X, SEED_Y, O.ptr(cf), 0)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config5_checksums.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path)


if __name__ == "__main__":
    main()
