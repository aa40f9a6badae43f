#!/usr/bin/env python
"""Writes the GA frozen sets of every bench workload code in the reference's
frozen-file format (save_frozen_file, code.cpp:187-194).

bench.py's reference arm loads them with the reference's own
load_frozen_file (oracle/_ref), so it builds its codes and inputs without
this repo's library; tests/test_frozen_files.py checks that they equal the
construction the product arm runs.

  python oracle/frozen/make_frozen.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_1710_08314_b200 import polar as P  # noqa: E402
from paper_1710_08314_b200.workload import WORKLOADS, crc_width  # noqa: E402


def main():
    done = set()
    for wl in WORKLOADS.values():
        design = wl.design_db
        for n, k, crc, path in wl.code_specs():
            if path in done:
                continue
            fz = P.construct_frozen_ga(n, k + crc_width(crc), design, k / n)
            P.save_frozen_file(path, n, k + crc_width(crc), fz)
            done.add(path)
            print(os.path.relpath(path, ROOT))


if __name__ == "__main__":
    main()
