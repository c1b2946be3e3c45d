"""Known-answer vectors of the partition permutation pi_k (reading Z2) for
tests/golden/perm_kat.json.  Calls only oracle/ (the CPU reference); the GPU and the test-side
numpy re-implementation are checked against this file.

usage: python scripts/make_perm_kat.py"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

CASES = [(0, 0, 1), (0, 0, 2), (0, 0, 5), (7, 3, 64), (7, 3, 1000), (2**63 + 5, 11, 4097), (1, 0, 50000),
         (2, 0, 1000000), (4, 0, 20000000), (4, 1, 20000000)]
out = {"_citation": "pi_k(seed, k, n) of reading Z2 (DESIGN.md section 2; PAPER.md:147-151 'random disjoint "
                    "partitions', Eq.8), written by scripts/make_perm_kat.py from oracle.permutation only. "
                    "head = pi[0:16], tail = pi[n-4:n], sha256 = of the int32 little-endian array.",
       "cases": []}
for seed, k, n in CASES:
    pi = oracle.permutation(seed, k, n)
    out["cases"].append({"seed": str(seed), "k": k, "n": n, "head": pi[:16].tolist(), "tail": pi[-4:].tolist(),
                         "sha256": hashlib.sha256(pi.astype("<i4").tobytes()).hexdigest()})
    print(seed, k, n, pi[:4].tolist(), flush=True)
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "perm_kat.json"), "w"), indent=1)
